"""On-device reconfiguration: the latency protocol.

``reconfiguration_latency`` is the reference's gate protocol
(``pkg/src/skirmish/rollout.py:422-448``, gate "worst reset < 10 ms" in
``pkg/tests/test_acceptance.py:425-433``) on a GPU ``BatchSim``: a warm batch
cycles ``count`` distinct scenarios through ``reset_env(i % lanes, config_i,
seed=i)`` with one step after each.  Each ``reset_env`` is the reference's
O(B) operation — respawn one lane, then ``init_output`` for the whole batch
(``environment.py:490-498``) — here a config-table slot lookup (hash of the
template bytes; a slot no lane uses any more is recycled), the row staged in
pinned memory and uploaded on the stream, one spawn launch with slot and seed
as kernel arguments, and the batch-wide init kernels.  Nothing in it waits on
the device; the times reported are measured to completion (host call plus a
stream synchronise), and separately for the host call alone.

The reference draws its scenarios with ``random_scenario`` (whose zones seed
from the salted ``hash(str)``, so they do not
reproduce across processes); ``scenario_variants`` makes distinct scenarios
of one shape instead, from a numpy generator: spawn positions and headings,
heuristic parameters, zone centres and effects redrawn.
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np
import torch

from .scenario import Scenario, Team, Zone


def scenario_variants(base: Scenario, count: int, seed: int = 0) -> list[Scenario]:
    """``count`` distinct scenarios with ``base``'s unit roster and capacities."""
    g = np.random.default_rng(seed)
    f = base.field
    out = []
    for k in range(count):
        units = []
        for u in base.units:
            pos = (float(g.uniform(f.margin, f.width - f.margin)),
                   float(g.uniform(f.margin, f.height - f.margin)))
            units.append(dataclasses.replace(u, position=pos,
                                             heading_deg=float(g.integers(0, 12) * 30)))
        zones = [Zone(z.type, (float(g.uniform(f.margin, f.width - f.margin)),
                               float(g.uniform(f.margin, f.height - f.margin))), z.semi_axes,
                      0.0 if z.type == "bush" else
                      float(g.uniform(2.0, 10.0) if z.type == "lava" else g.uniform(0.2, 0.8)))
                 for z in base.zones]
        teams = tuple(Team(t.id, t.controller, float(g.uniform(0.0, 1.0)),
                           float(g.uniform(0.0, 0.7))) if t.has_heuristic else t
                      for t in base.teams)
        out.append(dataclasses.replace(base, name=f"{base.name}-v{k}", units=units, zones=zones,
                                       teams=teams, notes=list(base.notes)))
    return out


def reconfiguration_latency(base: Scenario, count: int = 100, batch: int = 8, seed: int = 0,
                            device=0) -> dict:
    """rollout.py:422-448 on the GPU.  Returns per-reset seconds measured to
    completion (``times``) and for the host call alone (``host_times``),
    plus the config-table size afterwards."""
    from .sim import BatchSim

    configs = [c.scripted() for c in scenario_variants(base, count, seed)]
    lanes = batch
    sim = BatchSim([configs[0]] * lanes, list(range(lanes)), auto_reset=True, device=device,
                   interactions=False, final_observations=False)
    dev = sim.device
    for _ in range(3):
        sim.step(None)
    sim.reset_env(0, configs[0], seed=0)  # warm the reset path too
    sim.step(None)
    torch.cuda.synchronize(dev)
    times, host_times = [], []
    for i, c in enumerate(configs):
        t0 = time.perf_counter()
        sim.reset_env(i % lanes, c, seed=i)
        t1 = time.perf_counter()
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        times.append(t2 - t0)
        host_times.append(t1 - t0)
        sim.step(None)
        torch.cuda.synchronize(dev)  # the next reset is timed from an idle stream
    rows, cap = sim.num_configs()
    sim.close()
    return {"times": times, "host_times": host_times, "config_rows": rows,
            "config_capacity": cap, "batch": lanes}
