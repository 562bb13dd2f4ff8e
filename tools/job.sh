#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
python bench.py --scenario c1 --no-cpu --rollout-envs 0 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | cut -c1-200
python bench.py --no-cpu --rollout-envs 0 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-200
