"""Golden-trajectory case definitions shared by tools/make_golden.py (which runs
the reference engine) and the tests (which run the oracle / the CUDA path).

A case is a scenario document (one of the shipped JSON files plus JSON-level
edits), a batch of lanes seeded like the trainer bindings
(``derive_seed(run_seed, b, TAG_EPISODE)``, ``bindings/.../__init__.py:51-55``),
an auto-reset flag, a step count, and optionally

* ``external``: seed of a host RNG that picks a uniformly random *legal*
  action for every unit from the previous step's action mask (exercises the
  external-controller path),
* ``resets``: ``{step: [(lane, seed), ...]}`` — ``reset_env`` calls made
  after that step (the rollout driver pattern, ``rollout.py:280-283``).
"""
from __future__ import annotations

import copy
import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_DIR = os.path.join(HERE, "golden")
SCEN_DIR = os.path.join(HERE, "..", "paper_2602_01665_b200", "scenarios")

MASK64 = (1 << 64) - 1


def _mix(x):
    x &= MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def derive_seed(seed, index, tag):
    h = _mix(seed + 0x9E3779B97F4A7C15 * tag)
    h = _mix(h + index * 0xC2B2AE3D27D4EB4F)
    return _mix(h)


def load_doc(name: str) -> dict:
    with open(os.path.join(SCEN_DIR, f"{name}.json"), encoding="utf-8") as fh:
        return json.load(fh)


def _teams(doc, ally, enemy):
    tiers = {"medium": (0.2, 0.3), "expert": (0.01, 0.7), "novice": (0.5, 0.1),
             "advanced": (0.1, 0.5), "random": (1.0, 0.0)}
    out = []
    for tid, spec in ((0, ally), (1, enemy)):
        if spec.startswith("heuristic:"):
            e, x = tiers[spec.split(":")[1]]
            out.append({"id": tid, "controller": "heuristic",
                        "heuristic": {"epsilon": e, "aggressive_threshold": x}})
        else:
            out.append({"id": tid, "controller": spec})
    doc["teams"] = out


def case_doc(case: dict) -> dict:
    doc = copy.deepcopy(load_doc(case["scenario"]))
    _teams(doc, case.get("ally", "random"), case.get("enemy", "heuristic:medium"))
    for path, value in case.get("edits", []):
        node = doc
        for key in path[:-1]:
            node = node[key]
        node[path[-1]] = value
    return doc


def case_text(case: dict) -> str:
    return json.dumps(case_doc(case), sort_keys=True, indent=2) + "\n"


def case_seeds(case: dict) -> list[int]:
    return [derive_seed(case.get("run_seed", 0), b, 1) for b in range(case["batch"])]


CASES = {
    # C1 shape, bench controllers (random vs heuristic-medium), crosses the
    # t=400 truncation so every lane auto-resets.
    "c1_bench": dict(scenario="c1_3v3", batch=16, steps=410, auto_reset=True),
    # C3 shape with terrain (lava, bush, swamp), heuristic enemy.
    "c3_bench": dict(scenario="c3_10v10_terrain", batch=6, steps=405, auto_reset=True),
    # C2 shape, short.
    "c2_short": dict(scenario="c2_10v10", batch=4, steps=80, auto_reset=True, run_seed=3),
    # C4 shape (N=100, multi-warp path), short.
    "c4_short": dict(scenario="c4_50v50", batch=2, steps=25, auto_reset=True, run_seed=5),
    # Both teams expert heuristics on terrain: eliminations, reveals, bush play,
    # out-of-lockstep auto-resets (batch-coupled cache refresh).
    "duel_expert": dict(scenario="duel_terrain", batch=24, steps=260, auto_reset=True,
                        ally="heuristic:expert", enemy="heuristic:expert", run_seed=7,
                        edits=[(("max_steps",), 120)]),
    # External ally driven by legal random actions; big bodies (mammoth, king).
    "kings_external": dict(scenario="mixed_kings", batch=8, steps=150, auto_reset=True,
                           ally="external", external=11, run_seed=2,
                           edits=[(("max_steps",), 90)]),
    # No auto-reset; rollout-style reset_env of finished lanes, noop enabled,
    # a kinematic unit, a negative heading, and a unit spawned on the border.
    "rollout_resets": dict(
        scenario="duel_terrain", batch=5, steps=140, auto_reset=False,
        ally="heuristic:novice", enemy="random", run_seed=9,
        edits=[(("max_steps",), 60), (("physics", "enable_noop"), True),
               (("units", 0, "overrides"), {"kinematic": True}),
               (("units", 1, "heading_deg"), -75.0),
               (("units", 2, "position"), [0.0, 40.0])],
        resets={60: [(0, 101), (3, 103)], 61: [(1, 102)], 121: [(2, 104), (4, 105)]}),
    # N = 150 on terrain: the W = 8 path (5 words per cache row) and
    # numpy's recursive pairwise split (n > 128) in the team-health sums;
    # short episodes so truncations, ties / wins and auto-resets all occur.
    "w8_terrain": dict(scenario="c6_75v75_terrain", batch=3, steps=45, auto_reset=True,
                       run_seed=12, edits=[(("max_steps",), 20)]),
    # Two units spawned on the same point (coincident-centre contact normal),
    # random vs random.
    "coincident": dict(scenario="mixed_kings", batch=3, steps=40, auto_reset=True,
                       ally="random", enemy="random", run_seed=4,
                       edits=[(("units", 1, "position"), [10.0, 12.5]),
                              (("units", 0, "position"), [10.0, 12.5])]),
}


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha1()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()[:16]


OUTPUT_KEYS = ("observations", "global_state", "rewards", "action_mask", "terminated",
               "truncated", "done", "dense_reward", "actions", "interactions", "winner",
               "reason", "first_kill", "episode_return", "episode_length")
STATE_KEYS = ("seed", "episode", "t", "pos", "heading", "vel", "imp_dv", "health",
              "cooldown", "reveal", "alive", "prev_gap", "ep_return", "done", "terminated",
              "truncated", "winner", "reason", "first_kill", "mem_pos", "mem_valid",
              "vis", "atk")


def step_record(out: dict, sim) -> dict:
    rec = {k: digest(np.asarray(out[k])) for k in OUTPUT_KEYS}
    if out.get("final_observations") is not None:
        rec["final_observations"] = digest(out["final_observations"])
        rec["final_global_state"] = digest(out["final_global_state"])
    rec["state"] = digest(np.concatenate(
        [np.ascontiguousarray(getattr(sim, k)).view(np.uint8).ravel() for k in STATE_KEYS]))
    return rec


def legal_pick(mask: np.ndarray, gen: np.random.Generator) -> np.ndarray:
    """Uniform legal action per unit from a [B,N,7] mask."""
    u = gen.random(mask.shape[:2])
    n = mask.sum(axis=-1)
    k = np.minimum((u * n).astype(np.int64), n - 1)
    return np.argmax(np.cumsum(mask, axis=-1) > k[..., None], axis=-1).astype(np.int64)
