"""Step time of the multi-word shapes (W = 2: 20v20 from the C4 roster, 40
units; W = 8: c6_75v75_terrain, 150 units) -- per-kernel CUDA events.

    [TABX_LIB=...] python tools/wprobe.py [envs_w2] [envs_w8] [steps]
"""
from __future__ import annotations

import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2602_01665_b200.rng import lane_seeds  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


def w2_scenario():
    base = builtin_scenario("c4_50v50")
    allies = [u for u in base.units if u.team == 0][:20]
    enemies = [u for u in base.units if u.team == 1][:20]
    sc = dataclasses.replace(base, units=allies + enemies, max_units=40, notes=list(base.notes))
    return sc.scripted()


def run(name, sc, envs, steps):
    sim = BatchSim([sc] * envs, lane_seeds(0, envs), auto_reset=True, device=0,
                   interactions=False, final_observations=False)
    for _ in range(3):
        sim.step(None)
    torch.cuda.synchronize()
    sim.set_profiling(True)
    for _ in range(steps):
        sim.step(None)
    kp = sim.kernel_profile()
    ms = sum(v for k, v in kp.items() if k.endswith("_ms"))
    print(f"{name:8s} envs={envs} step {ms:.3f} ms = {envs / ms / 1e3:.2f} M env-steps/s  "
          + " ".join(f"{k}={v:.3f}" for k, v in kp.items() if k.endswith("_ms")))
    sim.close()


if __name__ == "__main__":
    e2 = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    e8 = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    run("W=2", w2_scenario(), e2, steps)
    run("W=8", builtin_scenario("c6_75v75_terrain").scripted(), e8, steps)
