#!/bin/bash
# One ncu --set full capture (source-correlated) of the C3 step kernel K1
# (lane_kernel<1, 4, MODE_STEP_K0, 20, 6>), outputs in gpurun_out/.
TAG=${1:-k1}
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:lane_kernelILi1ELi16ELi4ELi20ELi6E -s 3 -c 1 -o gpurun_out/$TAG -f \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/${TAG}*
