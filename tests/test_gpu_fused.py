"""The fused step + observation kernel (csrc/tabx_fused.cu) against the
separate step and observation kernels (TABX_FUSED=0), and against the oracle.

The fused kernel runs the same per-environment code as K1 + K2 with a
shared-memory hand-off between step warps and emitter warps, so every output
must be bit-identical to the split path: observations, final observations
(lanes whose auto-reset is pending), global state, rewards and the state.
Every setmaxnreg variant (warp split / register redistribution) is covered.
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

from paper_2602_01665_b200.scenario import builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402

VARIANTS = (0, 1, 2, 3)


def _pair(sc, B, seeds, monkeypatch, variant=0, **kw):
    sims = []
    for flag in ("1", "0"):
        monkeypatch.setenv("TABX_FUSED", flag)
        monkeypatch.setenv("TABX_FUSED_VARIANT", str(variant))
        sims.append(BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0", **kw))
    return sims


def _same(outs, t):
    a, b = outs
    for k in ("observations", "global_state", "rewards", "final_observations",
              "final_global_state", "reset_mask", "terminated", "truncated", "dense_reward"):
        x, y = getattr(a, k, None), getattr(b, k, None)
        if x is None and y is None:
            continue
        assert torch.equal(x, y), f"{k} differs at t={t}"


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scen", ["c3_10v10_terrain", "c2_10v10"])
def test_fused_equals_split(scen, variant, monkeypatch):
    B = 8192
    sc = builtin_scenario(scen)
    fused, split = _pair(sc, B, np.arange(B, dtype=np.uint64) + 101, monkeypatch, variant,
                         interactions=False)
    for t in range(25):
        outs = (fused.step(None), split.step(None))
        assert fused.step_path() == "fused" and split.step_path() == "split"
        _same(outs, t)
    s0, s1 = fused.export_state(), split.export_state()
    for k in s0:
        assert torch.equal(s0[k], s1[k]), k


def test_fused_across_lockstep_episode_end(monkeypatch):
    """C3 lanes all truncate at t = 400 and auto-reset together: the fused
    kernel writes their terminal rows to final_observations and the next step
    refreshes every cache; 2,000 lanes over 405 steps against the split path."""
    B = 2000  # not a multiple of the SM count: ragged last items per CTA
    sc = builtin_scenario("c3_10v10_terrain")
    fused, split = _pair(sc, B, np.arange(B, dtype=np.uint64) + 7, monkeypatch, interactions=False)
    resets = 0
    for t in range(405):
        outs = (fused.step(None), split.step(None))
        resets += int(outs[0].reset_mask.sum())
        if t % 10 == 0 or t >= 395:
            _same(outs, t)
    assert resets >= B  # every lane ended an episode inside the window
    s0, s1 = fused.export_state(), split.export_state()
    for k in s0:
        assert torch.equal(s0[k], s1[k]), k


@pytest.mark.parametrize("B", [1, 3, 149, 300])
def test_fused_small_and_ragged_batches_match_oracle(B, monkeypatch):
    """Fewer environments than SMs (one item per CTA, idle emitters) and
    ragged CTA item counts, through the fused kernel, against the oracle."""
    monkeypatch.setenv("TABX_FUSED", "1")
    sc = builtin_scenario("c3_10v10_terrain")
    seeds = np.arange(B, dtype=np.uint64) * 13 + 5
    gpu = BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim([sc] * B, seeds, auto_reset=True)
    for t in range(12):
        g = gpu.step(None)
        assert gpu.step_path() == "fused"
        o = ora.step(None)
        bad = compare_outputs(g, o, f"fused B={B} t={t}")
        if t % 4 == 3:
            bad += compare_state(gpu.export_state(), ora.sim, f"fused B={B} t={t}")
        assert not bad, "\n".join(bad[:10])
    gpu.close()


def _pair_single(sc, B, seeds, monkeypatch, **kw):
    """(single-launch step, split K1 + K2 + K3), both with the in-kernel
    controller (TABX_NO_K0=1)."""
    monkeypatch.setenv("TABX_NO_K0", "1")
    sims = []
    for mx in ("4096", "0"):
        monkeypatch.setenv("TABX_SINGLE_MAX_ENVS", mx)
        sims.append(BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0", **kw))
    return sims


@pytest.mark.parametrize("scen,B,steps", [("c1_3v3", 256, 410), ("c3_10v10_terrain", 600, 40),
                                          ("c2_10v10", 37, 30)])
def test_single_launch_step_equals_split(scen, B, steps, monkeypatch):
    """The single-launch step (small batches: step, observation rows and the
    auto-resets in one kernel) against K1 + K2 + K3: every output and the
    state, across auto-resets (C1 over 410 steps crosses the lockstep
    truncation at t = 400)."""
    sc = builtin_scenario(scen).scripted()
    single, split = _pair_single(sc, B, np.arange(B, dtype=np.uint64) * 7 + 3, monkeypatch)
    resets = 0
    for t in range(steps):
        outs = (single.step(None), split.step(None))
        assert single.step_path() == "single" and split.step_path() == "split"
        resets += int(outs[0].reset_mask.sum())
        _same(outs, t)
        assert torch.equal(outs[0].action_mask, outs[1].action_mask), t
    s0, s1 = single.export_state(), split.export_state()
    for k in s0:
        assert torch.equal(s0[k], s1[k]), k
    if scen == "c1_3v3":
        assert resets > 0  # auto-resets happened inside the single kernel


@pytest.mark.parametrize("B", [1, 5, 256])
def test_single_launch_step_matches_oracle(B, monkeypatch):
    """C1 (the BASELINE parity config, 256 envs; and ragged 1 / 5 envs: one
    CTA with idle warps) through the single-launch step against the oracle
    for 120 steps, auto-resets included."""
    monkeypatch.setenv("TABX_NO_K0", "1")
    sc = builtin_scenario("c1_3v3").scripted()
    seeds = np.arange(B, dtype=np.uint64) + 900
    gpu = BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim([sc] * B, seeds, auto_reset=True)
    for t in range(120):
        g = gpu.step(None)
        assert gpu.step_path() == "single"
        o = ora.step(None)
        bad = compare_outputs(g, o, f"single t={t}")
        if t % 10 == 9:
            bad += compare_state(gpu.export_state(), ora.sim, f"single t={t}")
        assert not bad, "\n".join(bad[:10])
    gpu.close()
