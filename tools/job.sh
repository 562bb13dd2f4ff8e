#!/bin/bash
# Scratch job for gpurun (edited per experiment).  As committed: the round-end
# checks -- GPU tests, smoke, default bench line, reference arm.
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-100
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-100
