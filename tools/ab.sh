#!/bin/bash
# A/B timing of library variants: tools/ab.sh "<lib|default> <stage_bytes>" ...
# Runs each variant 3x interleaved (bench.py --no-cpu --no-e2e --rollout-envs 0 --steps 10)
# and prints the env-steps/s (millions) of each run.
mkdir -p gpurun_out
VARIANTS=("$@")
declare -A RES
for rep in 1 2 3; do
  for v in "${VARIANTS[@]}"; do
    read -r lib sb <<< "$v"
    if [ "$lib" = default ]; then unset TABX_LIB; else export TABX_LIB=$PWD/$lib; fi
    export TABX_STAGE_BYTES=$sb
    timeout 300 python bench.py --no-cpu --no-e2e --rollout-envs 0 --steps 10 ${BENCH_EXTRA} > gpurun_out/ab.log 2>&1
    val=$(python -c "import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2))" 2>/dev/null)
    RES["$v"]="${RES["$v"]} $val"
  done
done
for k in "${!RES[@]}"; do echo "$k :${RES[$k]}"; done | sort
