python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
bash tools/ab.sh "default 0" "variants/base.so 0"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --rollout-envs 0 --envs 65536"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lane_kernel|emit_kernel" -s 6 -c 2 -f -o gpurun_out/prof_k1d $CMD > gpurun_out/ncu2.log 2>&1; echo ncu=$?
