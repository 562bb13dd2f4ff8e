"""Time the pieces of one C5 rollout step (16,384 envs, C3 shape)."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_01665_b200.rollout import Rollout, masked_sample
from paper_2602_01665_b200.scenario import builtin_scenario
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ro = Rollout(builtin_scenario("c3_10v10_terrain"), B, horizon=16, policy="mlp", device=0)
obs = ro._current_obs(0); mask = ro.sim._buf["action_mask"]
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
import ctypes as ct
from paper_2602_01665_b200 import _native as nat
def pack():
    nat.lib().tabx_pack_bf16(ct.c_void_p(obs.data_ptr()), B * ro.N, ro.D, ro.policy.in_dim,
                             ct.c_void_p(ro._xin.data_ptr()), ct.c_void_p(torch.cuda.current_stream().cuda_stream))
print("pack bf16    ", round(t(pack), 4), "ms")
print("mlp forward  ", round(t(lambda: ro.policy(ro._xin)), 4), "ms")
print("one step     ", round(t(lambda: ro._step(0)), 4), "ms")
ro.run()
print("horizon/16   ", round(t(lambda: ro.run(), 3) / 16, 4), "ms (graph replay)")
logits = ro.policy(ro._xin).reshape(B * ro.N, -1)
L = nat.lib()
def sample():
    L.tabx_masked_sample(ct.c_void_p(logits.data_ptr()), 1, 8, ct.c_void_p(mask.data_ptr()), B * ro.N,
                         ct.c_uint64(0), None, 0, ct.c_void_p(ro.buf.actions[0].data_ptr()),
                         ct.c_void_p(ro.buf.logp[0].data_ptr()), ct.c_void_p(torch.cuda.current_stream().cuda_stream))
print("sampler      ", round(t(sample), 4), "ms")
def envstep():
    L.tabx_step(ro.sim.handle, ct.c_void_p(ro.buf.actions[0].data_ptr()), ct.byref(ro._outs[0]))
print("env step     ", round(t(envstep), 4), "ms")
