"""How often the exact float64 fallbacks of the step run (-DTABX_COUNT_PROF).

    TABX_NVCC_EXTRA=-DTABX_COUNT_PROF TABX_BUILD_OUT=variants/count.so \\
        python -m paper_2602_01665_b200.build
    TABX_LIB=$PWD/variants/count.so python tools/count_prof.py [scenario] [envs] [warm] [steps]
"""
from __future__ import annotations

import ctypes as ct
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2602_01665_b200 import _native as nat  # noqa: E402
from paper_2602_01665_b200.rng import lane_seeds  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402

NAMES = ["exact_seen (visibility wedge/range)", "exact_box (strike box)",
         "contact exact, W=1", "contact exact, W>1 pair range", "contact exact, W>1 rows",
         "target distance sqrt (attack candidates)", "zone_exact", "f32_quot slow_div (K1+K2)",
         "closer() sqrt pair", "visibility rows (active observers)"]


def main(argv):
    name = argv[1] if len(argv) > 1 else "c3_10v10_terrain"
    envs = int(argv[2]) if len(argv) > 2 else 65536
    warm = int(argv[3]) if len(argv) > 3 else 3
    steps = int(argv[4]) if len(argv) > 4 else 10
    sc = builtin_scenario(name).scripted()
    sim = BatchSim([sc] * envs, lane_seeds(0, envs), auto_reset=True, device=0,
                   interactions=False, final_observations=False)
    L = nat.lib()
    buf = (ct.c_uint64 * 16)()
    for _ in range(warm):
        sim.step(None)
    torch.cuda.synchronize()
    L.tabx_debug_phase_cycles(buf, 1)
    for _ in range(steps):
        sim.step(None)
    torch.cuda.synchronize()
    L.tabx_debug_phase_cycles(buf, 1)
    print(f"{name}: {envs} envs, steps {warm}..{warm + steps}, calls per env-step")
    for k, p in enumerate(NAMES):
        print(f"  {p:44s} {buf[k] / envs / steps:10.4f}")
    sim.close()


if __name__ == "__main__":
    main(sys.argv)
