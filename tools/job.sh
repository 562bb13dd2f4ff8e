python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout 600 python tools/c5_probe.py 16384 > gpurun_out/c5.log 2>&1; cat gpurun_out/c5.log | tail -6
