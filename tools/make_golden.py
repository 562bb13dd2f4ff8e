"""Generate tests/golden/*.json from the reference engine itself.

Run in the build container only (imports /root/reference read-only):

    PYTHONPATH=/root/reference/pkg/src:tests python tools/make_golden.py

For every case in tests/golden_cases.py this drives the reference
``BatchSim`` (``pkg/src/skirmish/environment.py:463-519``) and records, per
step, a digest of every ``BatchOutput`` field and of the dynamic
``SimArrays`` state (float64 bytes, so the oracle must match bit for bit).
It also re-derives the reference's 100 FoV boundary verdicts
(``frontend/tests/fixtures/fov_samples.json``, generator
``frontend/scripts/make_fixtures.py:138-205``) by calling the reference
``perception.in_fov`` on each sample, and writes them with the verdicts.
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "tests"))

from golden_cases import (CASES, GOLDEN_DIR, case_seeds, case_text, legal_pick,  # noqa: E402
                          step_record)
from skirmish import BatchSim, load_scenario  # noqa: E402
from skirmish.core import UnitSpec, UnitState  # noqa: E402
from skirmish.perception import in_fov  # noqa: E402


def out_dict(out) -> dict:
    return {f.name: getattr(out, f.name) for f in dataclasses.fields(out)}


def run_case(name: str, case: dict) -> dict:
    cfg = load_scenario(case_text(case))
    seeds = np.array(case_seeds(case), dtype=np.uint64)
    sim = BatchSim([cfg] * case["batch"], seeds, auto_reset=case["auto_reset"])
    gen = np.random.default_rng(case["external"]) if "external" in case else None
    steps = [step_record(out_dict(sim.last), sim.sim)]
    resets = {int(k): v for k, v in case.get("resets", {}).items()}
    for t in range(1, case["steps"] + 1):
        acts = legal_pick(sim.last.action_mask, gen) if gen is not None else None
        out = sim.step(acts)
        steps.append(step_record(out_dict(out), sim.sim))
        for lane, seed in resets.get(t, []):
            sim.reset_env(lane, seed=seed)
            steps[-1]["after_reset"] = step_record(out_dict(sim.last), sim.sim)
    return {"case": name, "definition": case, "records": steps}


def fov_fixture() -> list:
    src = "/root/reference/pkg/frontend/tests/fixtures/fov_samples.json"
    with open(src, encoding="utf-8") as fh:
        samples = json.load(fh)
    out = []
    for smp in samples:
        spec = UnitSpec(max_health=100.0, body_radius=1.0, body_mass=1.0, speed=1.0,
                        attack_damage=1.0, attack_range=1.0, attack_cooldown=1.0,
                        sight_angle=smp["sight_angle"], sight_range=smp["sight_range"])
        obs = UnitState(spec=spec, team=0, position=np.array(smp["position"]),
                        heading=smp["heading"], velocity=np.zeros(2), health=100.0)
        verdict = bool(in_fov(obs, np.array(smp["point"])))
        assert verdict == smp["inside"]
        out.append({k: smp[k] for k in ("position", "heading", "sight_angle", "sight_range",
                                        "point")} | {"inside": verdict})
    return out


def main(argv) -> int:
    os.makedirs(GOLDEN_DIR, exist_ok=True)
    only = set(argv[1:])
    for name, case in CASES.items():
        if only and name not in only:
            continue
        rec = run_case(name, case)
        with open(os.path.join(GOLDEN_DIR, f"{name}.json"), "w", encoding="utf-8") as fh:
            json.dump(rec, fh, separators=(",", ":"))
        print(name, len(rec["records"]), "steps")
    with open(os.path.join(GOLDEN_DIR, "fov_samples.json"), "w", encoding="utf-8") as fh:
        json.dump(fov_fixture(), fh, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
