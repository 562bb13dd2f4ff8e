"""Two C3 batches on two streams (a GPU's lanes as two shards): does the
step logic of one overlap the observation stream of the other?

    NSTREAMS=2 python tools/dual_probe.py [envs per batch] [steps]
Prints env-steps/s over both batches, device-timed (events on both streams).
(The per-SM CTA caps of the experiment in DESIGN.md §6 were env knobs of the
launchers at the time, removed since.)
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
NS = int(os.environ.get("NSTREAMS", "2"))
sc = builtin_scenario("c3_10v10_terrain")
streams = [torch.cuda.Stream() for _ in range(NS)]
sims = [BatchSim([sc] * B, np.arange(k * B, (k + 1) * B, dtype=np.uint64), auto_reset=True,
                 device=0, interactions=False, stream=streams[k]) for k in range(NS)]
for _ in range(5):
    for s in sims:
        s.step(None)
torch.cuda.synchronize()
ev0 = torch.cuda.Event(enable_timing=True)
ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(NS)]
torch.cuda.current_stream().record_event(ev0)
for st in streams:
    st.wait_event(ev0)
for _ in range(T):
    for s in sims:
        s.step(None)
for k, st in enumerate(streams):
    st.record_event(ev1[k])
torch.cuda.synchronize()
ms = max(ev0.elapsed_time(e) for e in ev1)
print(f"streams={NS} envs/batch={B}: "
      f"{NS * B * T / (ms / 1e3) / 1e6:.2f} M env-steps/s ({ms / T:.3f} ms per round)")
