python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
REPS=3 bash tools/kab.sh default variants/base.so
