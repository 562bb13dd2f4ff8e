#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
TABX_NO_K0=1 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for r in 1 2 3; do printf "K0  "; REPS=1 bash tools/kab.sh default; done
