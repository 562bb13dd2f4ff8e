"""Shared test plumbing: drive the oracle through a golden case."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, ".."))
for p in (ROOT, os.path.join(ROOT, "oracle"), HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import tabx_oracle as orc  # noqa: E402
from golden_cases import (CASES, GOLDEN_DIR, case_seeds, case_text, legal_pick,  # noqa: E402
                          step_record)

from paper_2602_01665_b200.scenario import load_scenario  # noqa: E402


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN_DIR, f"{name}.json"), encoding="utf-8") as fh:
        return json.load(fh)


def case_scenario(name: str):
    return load_scenario(case_text(CASES[name]))


def oracle_records(name: str, steps: int | None = None):
    """Yield (t, record) for the oracle replaying golden case ``name``."""
    case = CASES[name]
    sc = case_scenario(name)
    sim = orc.OracleBatchSim([sc] * case["batch"], np.array(case_seeds(case), np.uint64),
                             auto_reset=case["auto_reset"])
    gen = np.random.default_rng(case["external"]) if "external" in case else None
    yield 0, step_record(sim.last, sim.sim)
    resets = {int(k): v for k, v in case.get("resets", {}).items()}
    n = case["steps"] if steps is None else min(steps, case["steps"])
    for t in range(1, n + 1):
        acts = legal_pick(sim.last["action_mask"], gen) if gen is not None else None
        out = sim.step(acts)
        rec = step_record(out, sim.sim)
        for lane, seed in resets.get(t, []):
            sim.reset_env(lane, seed=seed)
            rec["after_reset"] = step_record(sim.last, sim.sim)
        yield t, rec
