#!/bin/bash
# ncu --set full capture of the C3 heuristic-controller pass (ctrl_kernel<1>).
TAG=${1:-k0}
ncu --set full --clock-control none --import-source on -k regex:ctrl_kernel -s 3 -c 1 -o gpurun_out/$TAG -f \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
