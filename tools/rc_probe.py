import gc, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_01665_b200.reconfig import reconfiguration_latency
from paper_2602_01665_b200.scenario import builtin_scenario
base = builtin_scenario("c3_10v10_terrain")
for label in ("plain", "plain", "freeze", "nogc"):
    if label == "freeze":
        gc.collect(); gc.freeze()
    if label == "nogc":
        gc.disable()
    for batch in (8, 262144):
        r = reconfiguration_latency(base, 100, batch, 0, 0)
        t = np.array(r["times"]) * 1e3; h = np.array(r["host_times"]) * 1e3
        print(label, batch, "worst %.2f mean %.2f | host worst %.2f mean %.2f | argmax %d" % (t.max(), t.mean(), h.max(), h.mean(), t.argmax()), np.sort(t)[-4:].round(2))
