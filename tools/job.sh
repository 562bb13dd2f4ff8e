set -x
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --rollout-envs 0 --envs 65536"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv $CMD > gpurun_out/launches.csv 2> gpurun_out/launches.err; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lane_kernel|emit_kernel" -s 3 -c 2 -f -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu_full.log 2>&1; echo full=$?
