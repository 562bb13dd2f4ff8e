"""On-device reconfiguration.

* Config-table slots are recycled: cycling far more distinct scenarios than
  the table's 256 rows through ``reset_env`` never fails, the table stays at
  (lanes + 1) rows, and every step still equals the oracle doing the same
  ``reset_env`` calls (``environment.py:490-498``).
* The reference's reconfiguration protocol (``rollout.py:422-448``) meets
  its gate, worst reset under 10 ms (``pkg/tests/test_acceptance.py:425-433``),
  at the reference's batch of 8 and at the 262,144-lane bench batch.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_compare import compare_outputs, compare_state  # noqa: E402
from harness import orc  # noqa: E402

from paper_2602_01665_b200.reconfig import reconfiguration_latency, scenario_variants  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


def test_slot_recycling_under_churn_matches_oracle():
    base = builtin_scenario("c3_10v10_terrain").scripted()
    variants = [v.scripted() for v in scenario_variants(base, 300, seed=5)]
    B = 8
    seeds = np.arange(B, dtype=np.uint64) + 40
    gpu = BatchSim([base] * B, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim([base] * B, seeds, auto_reset=True)
    for i, c in enumerate(variants):
        b = i % B
        gpu.reset_env(b, c, seed=1000 + i)
        ora.reset_env(b, c, seed=1000 + i)
        o = ora.step(None)
        g = gpu.step(None)
        if i % 7 == 0 or i >= len(variants) - B:
            bad = compare_outputs(g, o, f"churn {i}")
            bad += compare_state(gpu.export_state(), ora.sim, f"churn {i}")
            assert not bad, "\n".join(bad[:10])
        rows, cap = gpu.num_configs()
        assert rows <= B + 1 and cap == 256, (i, rows, cap)
    # every lane stepped once per iteration: reset_env cut episodes short,
    # their steps still count (env_steps statistic)
    assert gpu.episode_stats()["env_steps"] == len(variants) * B
    # the base row lost its last lane long ago and was recycled; every live
    # slot is held by exactly its lanes
    held = {}
    for b in range(B):
        held[int(gpu.lane_slots[b])] = held.get(int(gpu.lane_slots[b]), 0) + 1
    for slot, n in held.items():
        assert gpu.config_slot_info(slot) == (n, False)
    # same content -> same slot (content-keyed, not object identity)
    import dataclasses
    twin = dataclasses.replace(variants[-1], notes=list(variants[-1].notes))
    gpu.reset_env(0, twin, seed=3)
    assert gpu.lane_slots[0] == gpu.lane_slots[(len(variants) - 1) % B]
    # respawn_all keeps every lane on its own config (ADVICE: slot per lane)
    before = gpu.lane_slots.copy()
    gpu.respawn_all(np.arange(B, dtype=np.uint64) + 7)
    assert np.array_equal(gpu.export_state()["config"].cpu().numpy(), before)
    gpu.close()


@pytest.mark.parametrize("batch", [8, 262_144])
def test_reconfiguration_latency_gate(batch):
    r = reconfiguration_latency(builtin_scenario("c3_10v10_terrain"), count=100, batch=batch,
                                seed=0, device=0)
    worst = max(r["times"])
    assert len(r["times"]) == 100
    assert r["config_rows"] <= min(batch, 100) + 2
    assert worst < 0.010, f"worst reset {worst * 1e3:.2f} ms at batch {batch}"
