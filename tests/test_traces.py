"""Trace emission / replay, CPU side.

The rollout driver of ``paper_2602_01665_b200.traces`` runs here on the CPU
oracle (through its ``engine_factory`` hook) and must write byte-identical
JSONL traces to the reference ``run_rollouts`` (``tests/golden/traces.json``,
made by ``tools/make_traces.py`` from ``pkg/src/skirmish/rollout.py``).  The
trace-format and replay properties follow ``pkg/tests/test_rollout.py``.
The GPU engine runs the same cases in ``test_gpu_traces.py``.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import harness  # noqa: F401  (sys.path for the oracle)
import tabx_oracle as orc
from paper_2602_01665_b200 import traces
from paper_2602_01665_b200.scenario import load_scenario

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "traces.json")
with open(GOLDEN, encoding="utf-8") as _fh:
    CASES = json.load(_fh)

RECORD_KEYS = {"t", "units", "reward", "terminated", "truncated"}
UNIT_KEYS = {"id", "team", "position", "heading", "health", "alive", "action",
             "cooldown_timer", "reveal_timer"}


class OracleEngine:
    """traces' engine protocol over the CPU oracle (test infrastructure)."""

    def __init__(self, configs, seeds):
        self.sim = orc.OracleBatchSim(configs, seeds, auto_reset=False)

    def step(self, actions):
        out = self.sim.step(actions)
        s = self.sim.sim
        st = {"pos": s.pos, "heading": s.heading, "health": s.health, "alive": s.alive,
              "cooldown": s.cooldown, "reveal": s.reveal, "t": s.t, "done": s.done,
              "winner": s.winner, "reason": s.reason, "first_kill": s.first_kill}
        return {k: out[k] for k in traces.OUT_FIELDS}, {k: np.copy(v) for k, v in st.items()}

    def reset_env(self, b, seed):
        self.sim.reset_env(b, seed=seed)

    def close(self):
        pass


def run_case(name, tmp_path, **over):
    c = CASES[name]
    args = dict(c["args"]) | over
    path = tmp_path / f"{name}.jsonl"
    summary = traces.run_rollouts(load_scenario(c["scenario"]), args["ally"], args["enemy"],
                                  episodes=args["episodes"], seed=args["seed"], trace=path,
                                  threads=args["threads"], batch=args["batch"],
                                  engine_factory=OracleEngine)
    return path, summary


@pytest.mark.parametrize("name", ["duel_small_run", "c1_random_medium_b3", "duel_terrain_b2"])
def test_trace_bytes_match_reference(name, tmp_path):
    c = CASES[name]
    path, summary = run_case(name, tmp_path)
    data = path.read_bytes()
    lines = data.decode().splitlines()
    assert lines[0] == c["first"]
    assert lines[-1] == c["last"]
    assert len(data) == c["bytes"] and len(lines) == c["lines"]
    assert hashlib.sha256(data).hexdigest() == c["sha256"]
    assert summary == c["summary"]


@pytest.mark.slow
def test_threads_and_batch_chunking_match_reference(tmp_path):
    c = CASES["kings_t2_b3"]
    path, summary = run_case("kings_t2_b3", tmp_path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == c["sha256"]
    assert summary == c["summary"]


def test_record_format(tmp_path):
    path, _ = run_case("duel_small_run", tmp_path, episodes=1)
    lines = path.read_text().splitlines()
    first, last = json.loads(lines[0]), json.loads(lines[-1])
    assert set(first) == RECORD_KEYS and set(last) == RECORD_KEYS | {"outcome"}
    assert set(first["units"][0]) == UNIT_KEYS
    for line in lines:
        rec = json.loads(line)
        assert list(rec) == sorted(rec)
        assert ("outcome" in rec) == (rec["terminated"] or rec["truncated"])
        for u in rec["units"]:
            assert list(u) == sorted(u)
            assert 0 <= u["action"] < 7
            assert 0.0 <= u["heading"] < 360.0


def test_summary_from_trace_recomputes_exactly(tmp_path):
    path, summary = run_case("duel_small_run", tmp_path)
    assert traces.summary_from_trace(path) == summary


def test_two_sided_replay_reproduces_bytes(tmp_path):
    c = CASES["duel_small_run"]
    path, summary = run_case("duel_small_run", tmp_path)
    again = tmp_path / "again.jsonl"
    s2 = traces.run_rollouts(load_scenario(c["scenario"]), f"replay:{path}", f"replay:{path}",
                             episodes=3, seed=17, trace=again, engine_factory=OracleEngine)
    assert s2 == summary
    assert again.read_bytes() == path.read_bytes()


def test_one_sided_replay_matches_live(tmp_path):
    c = CASES["duel_small_run"]
    path, summary = run_case("duel_small_run", tmp_path)
    s2 = traces.run_rollouts(load_scenario(c["scenario"]), f"replay:{path}", "heuristic:novice",
                             episodes=3, seed=17, engine_factory=OracleEngine)
    assert s2 == summary


def test_replay_errors_and_book(tmp_path):
    c = CASES["duel_small_run"]
    path, _ = run_case("duel_small_run", tmp_path, episodes=2)
    with pytest.raises(ValueError, match="replay holds 2 episodes"):
        traces.run_rollouts(load_scenario(c["scenario"]), f"replay:{path}", "heuristic:novice",
                            episodes=5, seed=17, engine_factory=OracleEngine)
    book = traces.ReplayBook.load(str(path))
    assert len(book.episodes) == 2
    assert book.actions(0, 1).shape == (2,)
    with pytest.raises(ValueError, match="ends at step"):
        book.actions(0, len(book.episodes[0]) + 1)


def test_policy_parsing():
    assert traces.parse_policy("random") == ("random", None)
    assert traces.parse_policy("heuristic:expert")[0] == "heuristic"
    assert traces.parse_policy("replay:/tmp/x.jsonl") == ("replay", "/tmp/x.jsonl")
    with pytest.raises(ValueError, match="unknown heuristic tier"):
        traces.parse_policy("heuristic:grandmaster")
    with pytest.raises(ValueError, match="unknown policy"):
        traces.parse_policy("greedy")


def test_empty_run(tmp_path):
    c = CASES["duel_small_run"]
    path = tmp_path / "empty.jsonl"
    s = traces.run_rollouts(load_scenario(c["scenario"]), "random", "random", episodes=0,
                            trace=path, engine_factory=OracleEngine)
    assert s == traces.summarize([]) and path.read_bytes() == b""
