#!/bin/bash
# ncu --set full capture of the C4 step kernel (lane_kernel<4, 1, MODE_STEP_K0, 100, 0>).
TAG=${1:-k1c4}
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:lane_kernelILi4ELi1ELi4ELi100ELi0E -s 3 -c 1 -o gpurun_out/$TAG -f \
  python bench.py --scenario c4 --envs 32768 --steps 2 --warmup 3 --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
