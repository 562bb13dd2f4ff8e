"""Host-side pieces of the C5 rollout loop that need no GPU.

The policy's fused first layer (bias + ReLU in the GEMM epilogue,
``torch._addmm_activation``) computes exactly ``l2(relu(l1(x)))``; the
torch reference sampler (``rollout.masked_sample``) only picks legal actions
and returns the masked log-softmax at the pick.
"""
from __future__ import annotations

import torch

from paper_2602_01665_b200.rollout import MLPPolicy, masked_sample


def test_fused_policy_layers_equal_unfused():
    torch.manual_seed(0)
    for dt in (torch.float32, torch.bfloat16):
        m = MLPPolicy(386, hidden=64).to(dt)
        assert m.in_dim % 8 == 0 and m.in_dim >= 386
        x = torch.randn(3, 20, m.in_dim).to(dt)
        ref = m.l2(torch.relu(m.l1(x)))
        out = m(x)
        assert out.shape == (3, 20, 8)
        assert torch.equal(out, ref), dt


def test_reference_sampler_legal_and_logp():
    torch.manual_seed(1)
    logits = torch.randn(4096, 7)
    mask = torch.rand(4096, 7) < 0.5
    mask[:, 6] |= ~mask.any(1)
    act, logp = masked_sample(logits, mask)
    assert bool(torch.gather(mask, 1, act[:, None]).all())
    want = torch.log_softmax(torch.where(mask, logits, torch.tensor(float("-inf"))), 1)
    assert torch.allclose(logp, torch.gather(want, 1, act[:, None])[:, 0], atol=1e-6)
