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
