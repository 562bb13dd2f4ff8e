#!/bin/bash
# Per-kernel A/B: tools/kab.sh lib1 lib2 ... (default = in-tree build); prints
# env-steps/s (M) and per-kernel ms for each variant, REPS interleaved rounds.
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
for lib in "$@"; do
  if [ "$lib" = default ]; then unset TABX_LIB; else export TABX_LIB=$PWD/$lib; fi
  timeout 300 python bench.py --no-cpu --no-e2e --rollout-envs 0 --steps 10 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig ${BENCH_EXTRA} > gpurun_out/kab.log 2>&1
  printf "%-22s " "$lib"; python -c "import json; d=json.loads(open('gpurun_out/kab.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']/1e6,2), [(k['kernel'][:6], round(k['ms_avg'],3)) for k in r['kernels']])" 2>&1 | tail -1
done
done
