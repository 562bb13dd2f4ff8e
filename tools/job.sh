#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
REPS=3 bash tools/kab.sh default variants/l2pf.so
