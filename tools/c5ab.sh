#!/bin/bash
# A/B of the C5 rollout line: tools/c5ab.sh lib1 lib2 ... (default = in-tree)
for rep in $(seq 1 ${REPS:-1}); do
for lib in "$@"; do
  if [ "$lib" = default ]; then unset TABX_LIB; else export TABX_LIB=$PWD/$lib; fi
  timeout 300 python bench.py --no-cpu --no-e2e --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig --steps 3 > gpurun_out/c5ab.log 2>&1
  printf "%-22s " "$lib"; python -c "import json; d=json.loads(open('gpurun_out/c5ab.log').read().strip().splitlines()[-1]); print(round(d['rollout_c5']['value']/1e6,2), round(d['rollout_c5']['ms_per_horizon'],2))" 2>&1 | tail -1
done
done
