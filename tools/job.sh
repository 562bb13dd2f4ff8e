#!/bin/bash
python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for s in c2 c4; do timeout 300 python bench.py --scenario $s --no-cpu --no-e2e --rollout-envs 0 --steps 10 > gpurun_out/s.log 2>&1; printf "$s "; python -c "import json; d=json.loads(open('gpurun_out/s.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']/1e6,3), [(k['kernel'][:6], round(k['ms_avg'],3)) for k in r['kernels']])"; done
python tools/c5_probe.py 2>&1 | tail -1
