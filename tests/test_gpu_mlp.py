"""The tcgen05 policy MLP (csrc/tabx_mlp.cu, ``tabx_policy_mlp``) against a
plain torch fp32 reference of the same function: logits = W2 · bf16(relu(W1
· x + b1)) + b2 with bf16 inputs, fp32 accumulation and bf16 logits.

Tolerance: the kernel and the reference differ only in fp32 summation order,
which can move a hidden activation across a bf16 rounding boundary (one bf16
ulp, 2^-8 relative) and the bf16 logit by one ulp; 2e-2 absolute + 2e-2
relative on logits of magnitude ~1 covers that with margin and fails on any
layout / descriptor error (those give O(1) errors)."""
from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_01665_b200.rollout import MLPPolicy  # noqa: E402


def _ref32(pol, x):
    h = torch.relu(x.float() @ pol.l1.weight.float().t() + pol.l1.bias.float())
    return h.bfloat16().float() @ pol.l2.weight.float().t() + pol.l2.bias.float()


# K = 392 (C3 / C5 observation, 386 padded), 1704 (C4: the W1-streaming
# kernel), 8 (one 16-byte piece), 72 (ragged last TMA box); rows cover one
# partial tile, exact tiles, ragged tails and the C5 bench size
@pytest.mark.parametrize("obs_dim,rows", [(386, 1), (386, 128), (386, 129), (386, 5000),
                                          (386, 327680), (1698, 3000), (8, 300), (72, 1000)])
def test_policy_mlp_matches_fp32_reference(obs_dim, rows):
    torch.manual_seed(rows + obs_dim)
    pol = MLPPolicy(obs_dim).cuda().bfloat16()
    x = torch.randn(rows, pol.in_dim, device="cuda").bfloat16()
    out = pol(x)
    torch.cuda.synchronize()
    assert out.shape == (rows, 8) and out.dtype == torch.bfloat16
    torch.testing.assert_close(out.float(), _ref32(pol, x), rtol=2e-2, atol=2e-2)
    # and the torch / cuBLASLt module agrees with it almost everywhere bit for bit
    same = (out == pol.reference(x)).float().mean().item()
    assert same > 0.99, same


def test_policy_mlp_strided_rows_and_zero_rows():
    """Rows with a stride larger than K (a view into a wider buffer) and an
    empty batch."""
    pol = MLPPolicy(386).cuda().bfloat16()
    wide = torch.randn(777, 448, device="cuda").bfloat16()
    x = wide[:, :392]
    out = pol(x)
    torch.testing.assert_close(out.float(), _ref32(pol, x), rtol=2e-2, atol=2e-2)
    empty = pol(torch.empty(0, 392, device="cuda", dtype=torch.bfloat16))
    assert empty.shape == (0, 8)


def test_policy_mlp_rejects_bad_shapes():
    pol = MLPPolicy(386, hidden=64).cuda().bfloat16()
    with pytest.raises(ValueError):
        pol(torch.zeros(4, 392, device="cuda", dtype=torch.bfloat16))


@pytest.mark.parametrize("rows", [1, 130, 20000])
def test_fused_sampler_equals_mlp_then_sampler(rows):
    """tabx_policy_mlp_sample (sampler fused into the MLP epilogue) draws the
    same actions and log-probabilities, bit for bit, as the MLP kernel
    followed by the stand-alone tabx_masked_sample on its bf16 logits."""
    import ctypes as ct

    from paper_2602_01665_b200 import _native as nat
    torch.manual_seed(rows)
    pol = MLPPolicy(386).cuda().bfloat16()
    x = torch.randn(rows, pol.in_dim, device="cuda").bfloat16()
    mask = (torch.rand(rows, 7, device="cuda") < 0.6).to(torch.uint8)
    mask[:, 0] = 1  # at least one legal action per row
    ctr = torch.tensor([5], dtype=torch.int64, device="cuda")
    L, s = nat.lib(), ct.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: ct.c_void_p(t.data_ptr())  # noqa: E731
    a1 = torch.empty(rows, dtype=torch.int64, device="cuda")
    l1 = torch.empty(rows, device="cuda")
    logits = pol(x)
    nat.check(L.tabx_masked_sample(p(logits), 1, 8, p(mask), rows, ct.c_uint64(77), p(ctr), 3,
                                   p(a1), p(l1), s), "sample")
    a2, l2 = torch.empty_like(a1), torch.empty_like(l1)
    lg2 = torch.empty_like(logits)
    nat.check(L.tabx_policy_mlp_sample(
        p(x), rows, pol.in_dim, pol.in_dim, p(pol.l1.weight), p(pol.l1.bias), p(pol.l2.weight),
        p(pol.l2.bias), p(lg2), p(mask), ct.c_uint64(77), p(ctr), 3, p(a2), p(l2), s), "fused")
    a3, l3 = torch.empty_like(a1), torch.empty_like(l1)
    nat.check(L.tabx_policy_mlp_sample(
        p(x), rows, pol.in_dim, pol.in_dim, p(pol.l1.weight), p(pol.l1.bias), p(pol.l2.weight),
        p(pol.l2.bias), None, p(mask), ct.c_uint64(77), p(ctr), 3, p(a3), p(l3), s), "fused")
    torch.cuda.synchronize()
    assert torch.equal(lg2, logits)
    assert torch.equal(a1, a2) and torch.equal(a1, a3)
    assert torch.equal(l1, l2) and torch.equal(l1, l3)
    assert bool((mask.gather(1, a1[:, None]) == 1).all())  # only legal actions
