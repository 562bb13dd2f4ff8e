"""tcgen05 policy MLP (tabx_policy_mlp) vs the torch / cuBLASLt module:
numerics against an fp32 reference, and time at the C5 shape
(16,384 envs x 20 agents = 327,680 rows, K = 392)."""
import ctypes as ct
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_01665_b200 import _native as nat  # noqa: E402
from paper_2602_01665_b200.rollout import MLPPolicy  # noqa: E402


def run(x, pol, out):
    s = torch.cuda.current_stream().cuda_stream
    nat.check(nat.lib().tabx_policy_mlp(
        ct.c_void_p(x.data_ptr()), x.shape[0], pol.in_dim, x.stride(0),
        ct.c_void_p(pol.l1.weight.data_ptr()), ct.c_void_p(pol.l1.bias.data_ptr()),
        ct.c_void_p(pol.l2.weight.data_ptr()), ct.c_void_p(pol.l2.bias.data_ptr()),
        ct.c_void_p(out.data_ptr()), ct.c_void_p(s)), "tabx_policy_mlp")


def ref(x, pol):
    h = torch.relu(x.float() @ pol.l1.weight.float().t() + pol.l1.bias.float())
    h = h.bfloat16().float()
    return h @ pol.l2.weight.float().t() + pol.l2.bias.float()


torch.manual_seed(0)
for rows, D in [(1, 386), (129, 386), (5000, 386), (3000, 1698), (327680, 386)]:
    pol = MLPPolicy(D).cuda().bfloat16()
    x = torch.randn(rows, pol.in_dim, device="cuda").bfloat16()
    out = torch.empty(rows, 8, device="cuda", dtype=torch.bfloat16)
    run(x, pol, out)
    torch.cuda.synchronize()
    r = ref(x, pol)
    c = pol(x).float()
    e_k = (out.float() - r).abs().max().item()
    e_c = (c - r).abs().max().item()
    print(f"rows {rows} K {pol.in_dim}: max|kernel-ref| {e_k:.4g}  max|cublas-ref| {e_c:.4g}  "
          f"max|ref| {r.abs().max().item():.3g}  exact-vs-cublas {(out.float() == c).float().mean().item():.4f}")

rows, D = 327680, 386
pol = MLPPolicy(D).cuda().bfloat16()
x = torch.randn(rows, pol.in_dim, device="cuda").bfloat16()
out = torch.empty(rows, 8, device="cuda", dtype=torch.bfloat16)
for name, fn in [("tcgen05", lambda: run(x, pol, out)), ("cublas", lambda: pol(x))]:
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    gb = rows * pol.in_dim * 2 / ms / 1e6
    print(f"{name}: {ms * 1e3:.1f} us  ({gb:.0f} GB/s of x)")
