python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value']/1e6, 'e2e', d['e2e']['value']/1e6, 'c5', d['rollout_c5']['value']/1e6, 'cpu', d['cpu_baseline'])"
