python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --rollout-envs 0 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | cut -c1-300
