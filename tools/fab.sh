#!/bin/bash
# A/B of the fused step + observation kernel variants (TABX_FUSED_VARIANT)
# against the split K1 + K2 path ("off"): tools/fab.sh off 0 1 2 ...
# prints env-steps/s (M) and per-kernel ms; REPS interleaved rounds.
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
for v in "$@"; do
  if [ "$v" = off ]; then export TABX_FUSED=0; else export TABX_FUSED=1 TABX_FUSED_VARIANT=$v; fi
  timeout 300 python bench.py --no-cpu --no-e2e --rollout-envs 0 --steps 10 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig ${BENCH_EXTRA} > gpurun_out/fab_$v.log 2>&1
  printf "%-6s " "$v"; python -c "import json; d=json.loads(open('gpurun_out/fab_$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']/1e6,2), d.get('step_path'), [(k['kernel'][:6], round(k['ms_avg'],3)) for k in r['kernels']])" 2>&1 | tail -1
done
done
