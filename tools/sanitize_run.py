"""Small-batch driver for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Runs every step-path kernel on small batches: K0 (heuristic-controller pass,
forced on with TABX_K0_MIN_ENVS=0), the refresh check, K1 (step), K2
(observation stream, TMA bulk stores), K3 (deferred auto-resets: episodes
of 3 steps so every lane resets), init_output, reset_env with a new config,
export/import, for the three cache-row widths the batches use: W = 1 (C3,
20 units, terrain), W = 2 (40 units) and W = 4 (C4, 100 units),
plus W = 8 (150 units, terrain).  Prints one line per case; exits non-zero on a CUDA
error.
"""
from __future__ import annotations

import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TABX_K0_MIN_ENVS", "0")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_01665_b200.reconfig import scenario_variants  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


def two_word():
    base = builtin_scenario("c4_50v50")
    allies = [u for u in base.units if u.team == 0][:20]
    enemies = [u for u in base.units if u.team == 1][:20]
    return dataclasses.replace(base, units=allies + enemies, max_units=40,
                               notes=list(base.notes))


def run(name, sc, B, steps):
    sc = dataclasses.replace(sc.scripted(), max_steps=3, notes=list(sc.notes))
    sim = BatchSim([sc] * B, np.arange(B, dtype=np.uint64) + 5, auto_reset=True, device=0)
    for _ in range(steps):
        sim.step(None)
    v = scenario_variants(sc, 1, seed=1)[0].scripted()
    v = dataclasses.replace(v, max_steps=3, notes=list(v.notes))
    sim.reset_env(1, v, seed=9)
    sim.step(None)
    st = sim.export_state()
    sim.import_state({k: st[k] for k in ("pos", "health", "heading")})
    sim.step(None)
    torch.cuda.synchronize()
    sim.close()
    print(f"{name}: B={B} N={sc.max_units} Z={sc.max_zones} steps={steps + 2} ok", flush=True)


def main() -> int:
    run("W=1 C3 terrain", builtin_scenario("c3_10v10_terrain"), 8, 5)
    run("W=1 C1", builtin_scenario("c1_3v3"), 8, 4)
    run("W=2 40 units", two_word(), 3, 4)
    run("W=4 C4", builtin_scenario("c4_50v50"), 2, 4)
    run("W=8 150 units", builtin_scenario("c6_75v75_terrain"), 1, 4)
    return 0


if __name__ == "__main__":
    sys.exit(main())
