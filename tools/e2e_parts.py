import os, sys, time
import numpy as np, torch, ctypes as ct
sys.path.insert(0, '.')
from paper_2602_01665_b200 import bindings, _native as nat
from paper_2602_01665_b200.scenario import builtin_scenario, save_scenario
B, T = 262144, 12
base = builtin_scenario("c3_10v10_terrain")
h = bindings.make_batch(save_scenario(base).encode(), B, 0, device=0, interactions=False, final_observations=True, strict=False)
N = h.agents
gen = np.random.default_rng(1)
pinned = [torch.from_numpy(gen.integers(0, 5, size=(B, N), dtype=np.int64)).pin_memory() for _ in range(2)]
dev = [p.to(0) for p in pinned]
sim = h.sim
rew = torch.empty(B, N, device=0); fl = torch.empty(2, B, dtype=torch.bool, device=0)
def timed(fn):
    fn(3); torch.cuda.synchronize(); t0 = time.perf_counter(); fn(T); torch.cuda.synchronize()
    return B * T / (time.perf_counter() - t0) / 1e6
def b(n):
    for k in range(n): sim.step(dev[k % 2], strict=False)
def b_d2d(n):
    for k in range(n):
        o = sim.step(dev[k % 2], strict=False)
        rew.copy_(o.rewards, non_blocking=True); fl[0].copy_(o.terminated, non_blocking=True); fl[1].copy_(o.truncated, non_blocking=True)
up = torch.cuda.Stream()
def b_h2d(n):
    for k in range(n):
        with torch.cuda.stream(up):
            dev[k % 2].copy_(pinned[k % 2], non_blocking=True)
        torch.cuda.current_stream().wait_stream(up)
        sim.step(dev[k % 2], strict=False)
print("b  device actions   ", round(timed(b), 2))
print("b + D2D copies      ", round(timed(b_d2d), 2))
print("b + H2D (waited)    ", round(timed(b_h2d), 2))
st = bindings.HostStepper(h)
def a(n):
    prev = None
    for k in range(n):
        t = st.submit(pinned[k % 2])
        if prev is not None: st.result(prev)
        prev = t
    if prev is not None: st.result(prev)
print("a HostStepper       ", round(timed(a), 2))
# isolate the copies: actions resident (no H2D) but the results copied out,
# and the converse
down = torch.cuda.Stream()
rh = torch.empty(B, N).pin_memory(); fh = torch.empty(2, B, dtype=torch.bool).pin_memory()
def b_d2h(n):
    for k in range(n):
        o = sim.step(dev[k % 2], strict=False)
        ev = torch.cuda.Event(); ev.record()
        down.wait_event(ev)
        with torch.cuda.stream(down):
            rh.copy_(o.rewards, non_blocking=True); fh[0].copy_(o.terminated, non_blocking=True)
print("b + D2H (async)     ", round(timed(b_d2h), 2))
def b_h2d_async(n):
    for k in range(n):
        with torch.cuda.stream(up):
            dev[(k + 1) % 2].copy_(pinned[(k + 1) % 2], non_blocking=True)
        sim.step(dev[k % 2], strict=False)
        torch.cuda.current_stream().wait_stream(up)
print("b + H2D (ahead)     ", round(timed(b_h2d_async), 2))
