"""Generate tests/golden/traces.json from the reference rollout driver.

Run in the build container only (imports /root/reference read-only):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tools/make_traces.py

Each case runs the reference ``run_rollouts`` (``pkg/src/skirmish/rollout.py:271-319``)
on a schema-v1 scenario document and records the SHA-256, size and line
count of the JSONL trace it writes, its first and last record, and the
summary.  The duel case is the reference tests' ``small_run`` scenario
(``pkg/tests/test_rollout.py:33-39``, ``conftest.duel_config``).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

from conftest import duel_config  # reference pkg/tests
from skirmish.rollout import run_rollouts
from skirmish.scenario import load_scenario, save_scenario

HERE = os.path.dirname(os.path.abspath(__file__))
SCEN = os.path.join(HERE, "..", "paper_2602_01665_b200", "scenarios")
OUT = os.path.join(HERE, "..", "tests", "golden", "traces.json")


def scen(name: str) -> str:
    with open(os.path.join(SCEN, f"{name}.json"), encoding="utf-8") as fh:
        return fh.read()


CASES = {
    # test_rollout.small_run: medium vs novice duel, batch 1
    "duel_small_run": dict(text=lambda: save_scenario(duel_config(enemy_controller="external")),
                           ally="heuristic:medium", enemy="heuristic:novice", episodes=3,
                           seed=17, threads=1, batch=1),
    # random ally vs medium, 3 lanes pulling 4 episodes (reset_env mid-batch)
    "c1_random_medium_b3": dict(text=lambda: scen("c1_3v3"), ally="random",
                                enemy="heuristic:medium", episodes=4, seed=5, threads=1,
                                batch=3),
    # test_rollout.test_bytes_stable_across_threads_and_batch shape
    "kings_t2_b3": dict(text=lambda: scen("mixed_kings"), ally="heuristic:medium",
                        enemy="heuristic:medium", episodes=5, seed=99, threads=2, batch=3),
    # terrain, expert vs random, 2 lanes
    "duel_terrain_b2": dict(text=lambda: scen("duel_terrain"), ally="heuristic:expert",
                            enemy="random", episodes=3, seed=3, threads=1, batch=2),
}


def main() -> int:
    out = {}
    for name, c in CASES.items():
        text = c["text"]()
        cfg = load_scenario(text)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "trace.jsonl")
            summary = run_rollouts(cfg, c["ally"], c["enemy"], episodes=c["episodes"],
                                   seed=c["seed"], trace=path, threads=c["threads"],
                                   batch=c["batch"])
            data = open(path, "rb").read()
        lines = data.decode().splitlines()
        out[name] = {
            "scenario": text,
            "args": {k: c[k] for k in ("ally", "enemy", "episodes", "seed", "threads", "batch")},
            "sha256": hashlib.sha256(data).hexdigest(),
            "bytes": len(data),
            "lines": len(lines),
            "first": lines[0],
            "last": lines[-1],
            "summary": summary,
        }
        print(name, len(lines), "records", out[name]["sha256"][:16], summary)
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
