"""Trace emission / replay on the GPU engine.

The device run loop (``traces.GpuEngine``: ``BatchSim`` + the
``tabx_export_lanes`` gather) must write the reference's trace bytes
(``tests/golden/traces.json`` from ``tools/make_traces.py``), and the sampled
lane stream (``TraceStream``) must reproduce the same records.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2602_01665_b200 import traces
from paper_2602_01665_b200.rng import lane_seeds
from paper_2602_01665_b200.scenario import load_scenario

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "traces.json")
with open(GOLDEN, encoding="utf-8") as _fh:
    CASES = json.load(_fh)


def run_case(name, tmp_path, **over):
    c = CASES[name]
    args = dict(c["args"]) | over
    path = tmp_path / f"{name}.jsonl"
    summary = traces.run_rollouts(load_scenario(c["scenario"]), args["ally"], args["enemy"],
                                  episodes=args["episodes"], seed=args["seed"], trace=path,
                                  threads=args["threads"], batch=args["batch"], device=0)
    return path, summary


@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_trace_bytes_match_reference(name, tmp_path):
    c = CASES[name]
    path, summary = run_case(name, tmp_path)
    data = path.read_bytes()
    lines = data.decode().splitlines()
    assert lines[0] == c["first"]
    assert lines[-1] == c["last"]
    assert hashlib.sha256(data).hexdigest() == c["sha256"]
    assert summary == c["summary"]


def test_gpu_two_sided_replay_reproduces_bytes(tmp_path):
    c = CASES["duel_small_run"]
    path, summary = run_case("duel_small_run", tmp_path)
    again = tmp_path / "again.jsonl"
    s2 = traces.run_rollouts(load_scenario(c["scenario"]), f"replay:{path}", f"replay:{path}",
                             episodes=3, seed=17, trace=again, device=0)
    assert s2 == summary
    assert again.read_bytes() == path.read_bytes()


def test_trace_stream_matches_full_gather():
    """Sampled lanes of an auto-reset batch: the pinned double-buffered stream
    yields the same records as a synchronous gather of the same lanes."""
    import torch

    from paper_2602_01665_b200.sim import BatchSim
    c = CASES["c1_random_medium_b3"]
    sc = load_scenario(c["scenario"]).with_controllers(ally="random")
    B = 64
    sim = BatchSim([sc] * B, lane_seeds(7, B), auto_reset=True, device=0,
                   interactions=False, final_observations=False)
    lanes = [0, 5, 17, 63]
    stream = traces.TraceStream(sim, lanes, sc)
    builder = traces.RecordBuilder(sc)
    lanes_t = torch.tensor(lanes, device=sim.device)
    pending = []
    for step in range(12):
        sim.step(None)
        slot = stream.capture()
        st = {k: v.cpu().numpy() for k, v in sim.export_lanes(lanes_t, traces.TRACE_FIELDS).items()}
        out = {k: getattr(sim.last, k).cpu().numpy()[lanes] for k in traces.OUT_FIELDS}
        want = [builder.record(st, out, k, k) for k in range(len(lanes))]
        if pending:
            prev_slot, prev_want = pending.pop()
            assert stream.records(prev_slot) == prev_want
        pending.append((slot, want))
    slot, want = pending.pop()
    assert stream.records(slot) == want
    assert all(r["t"] == 12 for r in want)
    sim.close()
