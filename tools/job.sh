#!/bin/bash
python tools/c5_probe.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py -k graph_rollout -x -q 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_policy.py -x -q 2>&1 | tail -1
