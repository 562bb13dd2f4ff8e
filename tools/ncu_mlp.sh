#!/bin/bash
# ncu --set full of the rollout's policy kernel (tcgen05 MLP + fused sampler)
# at the C5 shape; raw page to gpurun_out/mlp_ncu_raw.csv
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_policy_tma \
  -s 13 -c 1 -o gpurun_out/mlp_fused python tools/mlp_sample_time.py > gpurun_out/mlp_ncu.log 2>&1
ncu -i gpurun_out/mlp_fused.ncu-rep --page raw --csv > gpurun_out/mlp_ncu_raw.csv 2>/dev/null
tail -2 gpurun_out/mlp_ncu.log
