python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for lib in default variants/epw11.so variants/epw12.so; do
  if [ "$lib" = default ]; then unset TABX_LIB; else export TABX_LIB=$PWD/$lib; fi
  python bench.py --no-cpu --no-e2e --rollout-envs 0 --steps 10 > gpurun_out/bk.log 2>&1
  echo "$lib"; python -c "import json; d=json.loads(open('gpurun_out/bk.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']/1e6,2), [(k['kernel'][:12], round(k['ms_avg'],3), round(k.get('frac',0),3)) for k in r['kernels']])"
done
unset TABX_LIB
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --rollout-envs 0 --envs 65536"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"emit_kernel" -s 3 -c 1 -f -o gpurun_out/prof_k2g $CMD > gpurun_out/ncu2.log 2>&1; echo ncu=$?
