"""Soak / determinism probe: two independent 262,144-lane C3 batches run 900
steps (two lockstep episode ends with auto-resets and batch refreshes) and
must agree bit for bit on state, observation checksums and episode stats.

    python tools/soak_probe.py
"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_01665_b200.sim import BatchSim
from paper_2602_01665_b200.scenario import builtin_scenario
from paper_2602_01665_b200.rng import lane_seeds
sc = builtin_scenario("c3_10v10_terrain").scripted()
B = 262144
hs = []
for rep in range(2):
    sim = BatchSim([sc] * B, lane_seeds(0, B), auto_reset=True, device=0, interactions=False)
    for t in range(900):
        out = sim.step(None)
    torch.cuda.synchronize()
    st = sim.export_state()
    h = (float(st["pos"].double().sum()), float(st["health"].double().sum()), int(st["episode"].sum()), float(out.observations.double().sum()))
    stats = sim.episode_stats()
    print(rep, h, {k: float(v) for k, v in list(stats.items())[:4]} if isinstance(stats, dict) else stats)
    hs.append(h)
    sim.close(); del sim; torch.cuda.empty_cache()
print("deterministic", hs[0] == hs[1])
