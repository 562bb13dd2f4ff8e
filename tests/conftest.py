import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, ".."))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

# The heuristic-controller pass (K0) is the step's path from 4,096 lanes on;
# the tests run it at their small batch sizes too (TABX_NO_K0=1 selects the
# in-kernel controller, see test_gpu_parity.py).
os.environ.setdefault("TABX_K0_MIN_ENVS", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")
