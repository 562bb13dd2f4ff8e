"""Fused masked sampler of the C5 rollout loop (``tabx_masked_sample``).

Every sampled action is legal, its log-probability equals the masked
log-softmax of the logits at that action, equal logits give the uniform
distribution over the legal set (the reference's random controller,
environment.py:198-201, up to the RNG stream), and peaked logits pick their
argmax.
"""
from __future__ import annotations

import ctypes as ct

import pytest
import torch

from paper_2602_01665_b200 import _native as nat

pytestmark = pytest.mark.gpu


def sample(logits, mask, seed=1, step=0, bf16=False):
    M = mask.shape[0]
    act = torch.empty(M, dtype=torch.int64, device=mask.device)
    logp = torch.empty(M, dtype=torch.float32, device=mask.device)
    lg = logits.to(torch.bfloat16 if bf16 else torch.float32).contiguous()
    nat.check(nat.lib().tabx_masked_sample(
        ct.c_void_p(lg.data_ptr()), int(bf16), lg.shape[1], ct.c_void_p(mask.data_ptr()), M,
        ct.c_uint64(seed), None, step, ct.c_void_p(act.data_ptr()), ct.c_void_p(logp.data_ptr()),
        ct.c_void_p(torch.cuda.current_stream().cuda_stream)), "tabx_masked_sample")
    torch.cuda.synchronize()
    return act, logp


@pytest.mark.parametrize("bf16", [False, True])
def test_legal_and_logp(bf16):
    g = torch.Generator(device="cuda").manual_seed(0)
    M = 200_000
    mask = torch.rand(M, 7, device="cuda", generator=g) < 0.6
    mask[:, 6] |= ~mask.any(1)  # at least one legal action per row
    logits = torch.randn(M, 8, device="cuda", generator=g)
    act, logp = sample(logits, mask.to(torch.uint8), bf16=bf16)
    assert bool(torch.gather(mask, 1, act[:, None]).all())
    lg = logits[:, :7].to(torch.bfloat16 if bf16 else torch.float32).float()
    ref = torch.log_softmax(torch.where(mask, lg, torch.tensor(float("-inf"), device="cuda")), 1)
    want = torch.gather(ref, 1, act[:, None])[:, 0]
    assert torch.allclose(logp, want, atol=2e-5, rtol=1e-5)


def test_uniform_and_argmax():
    M = 400_000
    mask = torch.zeros(M, 7, dtype=torch.uint8, device="cuda")
    mask[:, [0, 2, 5]] = 1
    act, _ = sample(torch.zeros(M, 8, device="cuda"), mask, seed=7, step=3)
    counts = torch.bincount(act, minlength=7).float() / M
    assert set(torch.nonzero(counts).flatten().tolist()) == {0, 2, 5}
    assert torch.allclose(counts[[0, 2, 5]], torch.full((3,), 1 / 3, device="cuda"), atol=5e-3)
    peaked = torch.zeros(M, 8, device="cuda")
    peaked[:, 2] = 40.0
    act, logp = sample(peaked, mask, seed=7, step=4)
    assert bool((act == 2).all()) and float(logp.abs().max()) < 1e-6
    a1, _ = sample(torch.zeros(M, 8, device="cuda"), mask, seed=7, step=5)
    a2, _ = sample(torch.zeros(M, 8, device="cuda"), mask, seed=7, step=6)
    assert not torch.equal(a1, a2)  # the step counter changes the noise


def test_bf16_policy_feed_equals_packed_observations():
    """The emitter's bfloat16 policy feed (tabx_outputs.observations_bf16, written
    by K2 and, for auto-reset lanes, K3) equals tabx_pack_bf16 of the float32
    observation after every step, across episode boundaries."""
    from dataclasses import replace

    from paper_2602_01665_b200.rollout import Rollout
    from paper_2602_01665_b200.scenario import builtin_scenario
    sc = replace(builtin_scenario("c3_10v10_terrain"), max_steps=7)
    ro = Rollout(sc, 300, horizon=20, policy="mlp", device=0, use_graph=False)
    B, N, D, Dp = ro.B, ro.N, ro.D, ro.policy.in_dim
    ref = torch.empty(B, N, Dp, dtype=torch.bfloat16, device="cuda")
    resets = 0
    for t in range(ro.T):
        ro._step(t)
        obs = ro.buf.observations[t + 1]
        nat.check(nat.lib().tabx_pack_bf16(
            ct.c_void_p(obs.data_ptr()), B * N, D, Dp, ct.c_void_p(ref.data_ptr()),
            ct.c_void_p(torch.cuda.current_stream().cuda_stream)), "tabx_pack_bf16")
        torch.cuda.synchronize()
        assert torch.equal(ro._xin.view(torch.int16), ref.view(torch.int16)), t
        resets += int(ro.sim._buf["reset_mask"].sum())
    assert resets > 0
    ro.close()


def test_bf16_policy_feed_rejects_bad_rows():
    """The bf16 feed must be 16-byte aligned with a row stride that is a
    multiple of 8 and at least obs_dim (tabx.h): tabx_step refuses others
    with TABX_E_ALIGNMENT before launching anything."""
    import numpy as np

    from paper_2602_01665_b200.scenario import builtin_scenario
    from paper_2602_01665_b200.sim import BatchSim
    sc = builtin_scenario("c1_3v3")
    sim = BatchSim([sc] * 8, np.arange(8, dtype=np.uint64), auto_reset=True, device=0)
    D = sim.obs_dim
    Dp = (D + 7) // 8 * 8
    buf = torch.zeros(8 * sim.n_units * Dp + 16, dtype=torch.bfloat16, device="cuda")
    L = nat.lib()
    for ptr, ld in ((buf.data_ptr() + 2, Dp), (buf.data_ptr(), Dp + 4), (buf.data_ptr(), Dp - 8)):
        outs = nat.TabxOutputs.from_buffer_copy(sim._outs)
        outs.observations_bf16 = ptr
        outs.observations_bf16_ld = ld
        rc = L.tabx_step(sim.handle, None, ct.byref(outs))
        assert rc == nat.E_ALIGNMENT, (ptr - buf.data_ptr(), ld, rc)
    outs = nat.TabxOutputs.from_buffer_copy(sim._outs)
    outs.observations_bf16 = buf.data_ptr()
    outs.observations_bf16_ld = Dp
    nat.check(L.tabx_step(sim.handle, None, ct.byref(outs)), "tabx_step")
    torch.cuda.synchronize()
    sim.close()
