"""C5 shape: policy MLP alone, MLP + stand-alone sampler, and the fused
MLP + sampler kernel (tabx_policy_mlp_sample), CUDA-event timed."""
import ctypes as ct
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_01665_b200 import _native as nat  # noqa: E402
from paper_2602_01665_b200.rollout import MLPPolicy  # noqa: E402

rows = 327680
pol = MLPPolicy(386).cuda().bfloat16()
x = torch.randn(rows, pol.in_dim, device="cuda").bfloat16()
mask = (torch.rand(rows, 7, device="cuda") < 0.6).to(torch.uint8)
mask[:, 0] = 1
ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
act = torch.empty(rows, dtype=torch.int64, device="cuda")
logp = torch.empty(rows, device="cuda")
logits = torch.empty(rows, 8, device="cuda", dtype=torch.bfloat16)
L, s = nat.lib(), ct.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: ct.c_void_p(t.data_ptr())  # noqa: E731
w = [p(pol.l1.weight), p(pol.l1.bias), p(pol.l2.weight), p(pol.l2.bias)]


def mlp():
    L.tabx_policy_mlp(p(x), rows, 392, 392, *w, p(logits), s)


def sample():
    L.tabx_masked_sample(p(logits), 1, 8, p(mask), rows, ct.c_uint64(1), p(ctr), 0, p(act), p(logp), s)


def fused():
    L.tabx_policy_mlp_sample(p(x), rows, 392, 392, *w, None, p(mask), ct.c_uint64(1), p(ctr), 0,
                             p(act), p(logp), s)


def t(fn, n=50):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000


print(f"mlp {t(mlp):.1f} us  sampler {t(sample):.1f} us  mlp+sampler {t(lambda: (mlp(), sample())):.1f} us  fused {t(fused):.1f} us")
