"""Time tabx_policy_mlp at the C5 shape (for A/B of probe builds via TABX_LIB)."""
import ctypes as ct
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_01665_b200 import _native as nat  # noqa: E402
from paper_2602_01665_b200.rollout import MLPPolicy  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 327680
ld = int(sys.argv[2]) if len(sys.argv) > 2 else 392
pol = MLPPolicy(386).cuda().bfloat16()
x = torch.randn(rows, ld, device="cuda").bfloat16()
out = torch.empty(rows, 8, device="cuda", dtype=torch.bfloat16)
L = nat.lib()
args = [ct.c_void_p(x.data_ptr()), rows, pol.in_dim, x.stride(0),
        ct.c_void_p(pol.l1.weight.data_ptr()), ct.c_void_p(pol.l1.bias.data_ptr()),
        ct.c_void_p(pol.l2.weight.data_ptr()), ct.c_void_p(pol.l2.bias.data_ptr()),
        ct.c_void_p(out.data_ptr()), ct.c_void_p(torch.cuda.current_stream().cuda_stream)]
for _ in range(5):
    nat.check(L.tabx_policy_mlp(*args), "mlp")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    L.tabx_policy_mlp(*args)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
print(f"ld {ld}: {ms * 1e3:.1f} us  {rows * pol.in_dim * 2 / ms / 1e6:.0f} GB/s")
