"""Parity at benchmark scale: sampled lanes of the full bench batches.

The bench steps 262,144 (C3), 1,048,576 (C3) and 131,072 (C4 per GPU) lanes;
smaller parity tests cannot reach lane indices past a few thousand, nor the
int64 offsets of a 2.2e10-float observation tensor.  Lanes are independent
(``pkg/src/skirmish/arrays.py:3-6``; the reference pins batch == sequential,
``pkg/tests/test_environment.py:347-372``) except for the batch-coupled
cache refresh after an auto-reset (``environment.py:508``), so a small oracle
batch over a lane sample, seeded with those lanes' global seeds and given the
big batch's refresh decisions, must reproduce the sampled lanes bit for bit:
observations, global state, rewards, masks, executed actions, flags, and the
full dynamic state (gathered with ``tabx_export_lanes``).  The samples
include the first and the LAST lanes of every batch.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_compare import STATE_EXACT, STATE_F64, compare_outputs  # noqa: E402
from harness import orc  # noqa: E402

from paper_2602_01665_b200.rng import lane_seeds  # noqa: E402
from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


class _Rows:
    """The sampled rows of a BatchOutput (for compare_outputs)."""

    def __init__(self, out, lanes_t):
        for k in ("observations", "global_state", "rewards", "action_mask", "terminated",
                  "truncated", "done", "dense_reward", "actions", "winner", "reason",
                  "first_kill", "episode_return", "episode_length"):
            setattr(self, k, getattr(out, k).index_select(0, lanes_t))
        self.interactions = None


def _sample_lanes(B: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(8, B - 16), size=24, replace=False)
    return np.unique(np.concatenate([np.arange(8), mid, np.arange(B - 16, B)]))


def _compare_state(st: dict, sim, where: str, caches: bool) -> list[str]:
    bad = []
    for k in STATE_F64 + STATE_EXACT:
        if k in ("vis", "atk") and not caches:
            continue
        g = st[k].cpu().numpy()
        o = np.asarray(getattr(sim, k))
        if g.shape != o.shape or not np.array_equal(g, o):
            idx = np.argwhere(g != o)[0] if g.shape == o.shape else "shape"
            bad.append(f"{where}: state {k} differs at {idx}")
    if not np.array_equal(st["seed"].cpu().numpy().view(np.uint64), sim.seed):
        bad.append(f"{where}: state seed differs")
    return bad


@pytest.mark.parametrize("scen,B,steps,warm", [
    ("c3_10v10_terrain", 262_144, 410, 0),     # the headline batch, across the t=400 reset
    ("c3_10v10_terrain", 1_048_576, 30, 0),    # 4x the headline batch
    ("c4_50v50", 131_072, 30, 0),              # C4 per-GPU shard (W = 4)
])
def test_bench_batch_sampled_lanes_match_oracle(scen, B, steps, warm):
    sc = builtin_scenario(scen).scripted()  # the bench's controllers (rollout.py:360-366)
    seeds = lane_seeds(0, B)
    gpu = BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0", interactions=False,
                   final_observations=False)
    lanes = _sample_lanes(B, B)
    lanes_t = torch.as_tensor(lanes, device="cuda:0")
    ora = orc.OracleBatchSim([sc] * len(lanes), seeds[lanes], auto_reset=True)
    bad = compare_outputs(_Rows(gpu.last, lanes_t), ora.last, f"{scen} B={B} init",
                          check_final=False)
    bad += _compare_state(gpu.export_lanes(lanes_t), ora.sim, f"{scen} init", True)
    assert not bad, "\n".join(bad[:10])
    resets = 0
    for t in range(1, steps + 1):
        g = gpu.step(None)
        any_reset = bool(g.reset_mask.any().item())
        resets += any_reset
        o = ora.step(None, refresh=any_reset)
        bad = compare_outputs(_Rows(g, lanes_t), o, f"{scen} B={B} t={t}", check_final=False)
        # after a refill the device defers the batch-wide cache refresh to
        # the next step's start: stored vis/atk rows are compared otherwise
        bad += _compare_state(gpu.export_lanes(lanes_t), ora.sim, f"{scen} t={t}",
                              not any_reset)
        assert not bad, "\n".join(bad[:10])
    if steps > 400:
        assert resets >= 1  # the lockstep truncation at t = max_steps was crossed
    gpu.close()
