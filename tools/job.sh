#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
REPS=2 bash tools/kab.sh variants/head.so default
