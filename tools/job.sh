#!/bin/bash
for w in 5 100 200 390; do printf "warmup $w: "; BENCH_EXTRA="--warmup $w" REPS=1 bash tools/kab.sh default; done
