#!/bin/bash
# Throughput vs batch size (1 GPU), device-timed bench lines for C3 and C4.
for e in 16384 65536 262144 1048576; do
  timeout 300 python bench.py --scenario c3 --envs $e --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3', $e, round(d['value']/1e6,2), round(d['ms_per_step'],3), round(r['frac'],3), [(k['kernel'][:6], round(k['ms_avg'],3), round(k.get('frac') or 0,3)) for k in r['kernels']])"
done
for e in 16384 65536 131072; do
  timeout 300 python bench.py --scenario c4 --envs $e --no-cpu --no-e2e --rollout-envs 0 --configs "" --episode-steps 0 --host-obs-steps 0 --no-reconfig --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4', $e, round(d['value']/1e6,3), round(d['ms_per_step'],3), round(r['frac'],3), [(k['kernel'][:6], round(k['ms_avg'],3), round(k.get('frac') or 0,3)) for k in r['kernels']])"
done
