python -c "import sys; sys.path.insert(0,'.'); from paper_2602_01665_b200 import _native as n; n.lib()" || { echo "default lib broken"; exit 1; }
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "many_zones or two_word" > gpurun_out/pt.log 2>&1; tail -15 gpurun_out/pt.log
