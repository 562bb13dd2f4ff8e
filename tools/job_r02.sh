#!/bin/bash
# Round-2 evidence job (one gpurun call): GPU tests, smoke, the default bench
# line, the reference arm, the launch list with DRAM bytes, and ncu --set full
# captures of K2 and K1.  Outputs under gpurun_out/ (TAG prefix).
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.json | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${TAG}_bench_ref.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig > gpurun_out/${TAG}_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 bash tools/ncu_k2.sh ${TAG}_k2
timeout 600 bash tools/ncu_k1.sh ${TAG}_k1
