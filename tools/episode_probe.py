"""Per-kernel step time along the episode (C3 by default): warm W steps, then
time K steps with the per-kernel profile; prints how many of the timed steps
carried a batch refill (the next step refreshes every lane's caches).

    python tools/episode_probe.py [scenario] [envs] [warm] [steps]
"""
from __future__ import annotations

import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2602_01665_b200.rng import lane_seeds  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


def main(argv):
    name = argv[1] if len(argv) > 1 else "c3_10v10_terrain"
    envs = int(argv[2]) if len(argv) > 2 else 262144
    warm = int(argv[3]) if len(argv) > 3 else 200
    steps = int(argv[4]) if len(argv) > 4 else 20
    sc = builtin_scenario(name).scripted()
    sim = BatchSim([sc] * envs, lane_seeds(0, envs), auto_reset=True, device=0,
                   interactions=False, final_observations=True)
    for _ in range(warm):
        sim.step(None)
    torch.cuda.synchronize()
    sim.set_profiling(True)
    refills = 0
    for _ in range(steps):
        out = sim.step(None)
        refills += int(bool(out.reset_mask.any().item()))
    kp = sim.kernel_profile()
    tot = sum(v for k, v in kp.items() if k.endswith("_ms"))
    print(f"{name} envs={envs} t={warm}..{warm + steps}: {tot:.3f} ms/step = "
          f"{envs / tot / 1e3:.1f} M env-steps/s, refill steps {refills}/{steps}  "
          + " ".join(f"{k}={v:.3f}" for k, v in kp.items() if k.endswith("_ms")))
    sim.close()


if __name__ == "__main__":
    main(sys.argv)
