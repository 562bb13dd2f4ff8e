"""Per-phase SM-cycle shares of the step kernel (K1), instrumented build.

    TABX_NVCC_EXTRA=-DTABX_PHASE_PROF TABX_BUILD_OUT=variants/phase.so \
        python -m paper_2602_01665_b200.build
    TABX_LIB=$PWD/variants/phase.so python tools/phase_prof.py [scenario] [envs] [steps]

Lane 0 of every env adds clock64() deltas per phase (tabx_lane.cuh
TABX_PHASE marks); the shares are of warp-resident time, i.e. where a warp
spends its life, including the time it waits behind other warps.
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

PHASES = ["state load + masks", "action mask + controllers", "contact solve (Gauss-Seidel)",
          "boundary + rotation", "stage-8 caches", "combat, reveal, lava, deaths",
          "team ratios, rewards, termination", "outputs + stats", "state write-back",
          "  (in controllers) mask + swamp", "  integrate + contact detection (+ MODE_STEP vis/atk loads)",
          "  (in controllers) scripted_action", "  (in caches) zone_bits",
          "  (in caches) publish + build_masks",
          "    (in scripted, lowest heuristic lane) statics + target loop",
          "    (in scripted) attack / rotate-alignment check"]
MAIN = 9


def main(argv):
    name = argv[1] if len(argv) > 1 else "c3_10v10_terrain"
    envs = int(argv[2]) if len(argv) > 2 else 65536
    steps = int(argv[3]) if len(argv) > 3 else 10
    sc = builtin_scenario(name).scripted()
    sim = BatchSim([sc] * envs, lane_seeds(0, envs), auto_reset=True, device=0,
                   interactions=False, final_observations=False)
    L = nat.lib()
    buf = (ct.c_uint64 * 16)()
    for _ in range(3):
        sim.step(None)
    torch.cuda.synchronize()
    L.tabx_debug_phase_cycles(buf, 1)
    for _ in range(steps):
        sim.step(None)
    torch.cuda.synchronize()
    L.tabx_debug_phase_cycles(buf, 1)
    tot = sum(buf[k] for k in range(len(PHASES)))
    print(f"{name}: {envs} envs x {steps} steps, {tot / envs / steps:.0f} cycles/env-step")
    for k, p in enumerate(PHASES):
        print(f"  {p:36s} {buf[k] / envs / steps:9.0f} cycles/env  {100 * buf[k] / tot:5.1f}%")
    sim.close()


if __name__ == "__main__":
    main(sys.argv)
