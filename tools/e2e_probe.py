"""Where does the e2e gap come from?  Times, at C3 / 262,144 envs:
(a) HostStepper (host actions in, host results out, overlapped copies),
(b) bindings.step with device-resident actions (no copies),
(c) the device-value configuration (ally on the random controller, no actions)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_01665_b200 import bindings
from paper_2602_01665_b200.scenario import builtin_scenario, save_scenario

B, T = 262144, 12
base = builtin_scenario("c3_10v10_terrain")
h = bindings.make_batch(save_scenario(base).encode(), B, 0, device=0, interactions=False,
                        final_observations=True, strict=False)
N = h.agents
gen = np.random.default_rng(1)
pinned = [torch.from_numpy(gen.integers(0, 5, size=(B, N), dtype=np.int64)).pin_memory() for _ in range(4)]
devact = [p.to(0) for p in pinned]
st = bindings.HostStepper(h)
def timed(fn):
    fn(3); torch.cuda.synchronize(); t0 = time.perf_counter(); fn(T); torch.cuda.synchronize()
    return B * T / (time.perf_counter() - t0) / 1e6
def a(n):
    prev = None
    for k in range(n):
        t = st.submit(pinned[k % 4])
        if prev is not None: st.result(prev)
        prev = t
    if prev is not None: st.result(prev)
def b(n):
    for k in range(n): bindings.step(h, devact[k % 4])
print("a HostStepper      ", round(timed(a), 2))
print("b device actions   ", round(timed(b), 2))
h.sim.set_profiling(True)
b(T)
print("b kernel profile   ", h.sim.kernel_profile())
h.sim.set_profiling(False)
from paper_2602_01665_b200.sim import BatchSim
from paper_2602_01665_b200.rng import lane_seeds
sc = base.scripted()
sim = BatchSim([sc] * B, lane_seeds(0, B), auto_reset=True, device=0, interactions=False)
def c(n):
    for k in range(n): sim.step(None)
print("c scripted, no acts", round(timed(c), 2))
sim.set_profiling(True); c(T); print("c kernel profile   ", sim.kernel_profile())
