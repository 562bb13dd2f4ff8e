#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-90
python bench.py --scenario c1 --no-cpu --rollout-envs 0 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | cut -c1-90
python bench.py --scenario c1 --envs 262144 --no-cpu --rollout-envs 0 > gpurun_out/bench_c1big.log 2>&1; tail -1 gpurun_out/bench_c1big.log | cut -c1-90
python bench.py --scenario c2 --no-cpu --rollout-envs 0 > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-90
python bench.py --scenario c4 --no-cpu --rollout-envs 0 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-90
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-90
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --rollout-envs 0 --envs 65536 > gpurun_out/launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:emit_kernel -s 3 -c 1 -o gpurun_out/k2 \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rollout-envs 0 > gpurun_out/ncu_k2.log 2>&1; echo "ncu k2 rc=$?"
