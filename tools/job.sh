python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -30 gpurun_out/pt.log
