"""Device level generation against the host restatement.

``DeviceLevels`` (``tabx_levels``: one warp per level, numpy-exact PCG64
streams) must write config-table rows byte-equal to
``build_config(sample_level / mutate_level(...))`` of ``oracle/levels_oracle.py``
and advance the numpy generators to the same states; that restatement is
pinned to the reference generator by ``test_levels.py``.  Lanes respawned on device-made
rows (``tabx_respawn_lanes``) must then step exactly like the CPU oracle on
the host-made scenarios.
"""
from __future__ import annotations

import ctypes as ct
import json
import os

import numpy as np
import pytest

import harness  # noqa: F401  (puts oracle/ on sys.path)
import levels_oracle as host
from paper_2602_01665_b200 import levels
from paper_2602_01665_b200.rng import lane_seeds
from paper_2602_01665_b200.scenario import load_scenario
from paper_2602_01665_b200.template import build_config

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "levels.json")
with open(GOLDEN, encoding="utf-8") as _fh:
    CASES = json.load(_fh)


# golden-case spec keys (the reference's LevelGenSpec) -> LevelRanges keys
_RENAME = {"categories": "open", "unit_ranges": "units", "zone_types": "zone_types",
           "zone_center_box": "center_box", "zone_axis_range": "zone_axes",
           "zone_effect_ranges": "zone_effects", "epsilon_range": "epsilon",
           "aggressive_range": "aggressive"}


def make_spec(case):
    """(base, host spec, device ranges) of a golden case."""
    base = load_scenario(case["base"])
    if case["spec"] is None:
        return base, host.default_level_spec(base), levels.LevelRanges.broad(base)
    kw = dict(case["spec"])
    for k in ("categories", "zone_types"):
        if k in kw:
            kw[k] = tuple(kw[k])
    dkw = {_RENAME[k]: v for k, v in kw.items()}
    for k in ("units", "zone_effects"):
        if k in dkw:
            dkw[k] = dict(dkw[k])
    if "center_box" in dkw:
        dkw["center_box"] = tuple(tuple(r) for r in dkw["center_box"])
    return base, host.LevelGenSpec(base=base, **kw), levels.LevelRanges(base, **dkw)


def cfg_bytes(c) -> bytes:
    return bytes(memoryview(c))


def new_sim(sc, lanes=1):
    from paper_2602_01665_b200.sim import BatchSim
    return BatchSim([sc] * lanes, lane_seeds(0, lanes), device=0, interactions=False,
                    final_observations=False)


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_chain_matches_host(name):
    case = CASES[name]
    base, spec, ranges = make_spec(case)
    sim = new_sim(base)
    dl = levels.DeviceLevels(sim)
    g_dev = np.random.default_rng(case["seed"])
    g_host = np.random.default_rng(case["seed"])
    cur, row = base, 0
    for step in case["steps"]:
        op = step["op"]
        if op == "sample":
            cur = host.sample_level(spec, g_host)
            (row,) = dl.sample(ranges, [g_dev], base_slot=0)
        else:
            _, mop, delta, spec_from = op
            use = None if spec_from == "none" else spec
            cur = host.mutate_level(cur, mop, g_host, spec=use, delta=delta)
            # mutate_level(spec=None) uses the default spec over the level's
            # field, which levels never change
            dranges = levels.LevelRanges.broad(base) if use is None else ranges
            (row,) = dl.mutate(mop, [g_dev], [row], dranges, delta=delta)
        assert cfg_bytes(dl.config(row)) == cfg_bytes(build_config(cur, validate=False)), step
        assert g_dev.bit_generator.state == g_host.bit_generator.state
    sim.close()


def test_batch_of_levels_and_respawn_match_oracle():
    import harness  # noqa: F401
    import tabx_oracle as orc
    base = load_scenario(CASES["c3_default_sample_then_mutate"]["base"])
    spec = host.default_level_spec(base)
    ranges = levels.LevelRanges.broad(base)
    B, K = 64, 48
    sim = new_sim(base, B)
    dl = levels.DeviceLevels(sim)
    seeds = list(range(1000, 1000 + K))
    gens = [np.random.default_rng(s) for s in seeds]
    rows = dl.sample(ranges, gens, base_slot=0)
    mgens = [np.random.default_rng(s + 7) for s in seeds]
    rows2 = dl.mutate("perturb", mgens, rows, ranges, delta=0.15)
    host1 = [host.sample_level(spec, np.random.default_rng(s)) for s in seeds]
    host2 = [host.mutate_level(h, "perturb", np.random.default_rng(s + 7), spec=spec,
                               delta=0.15) for h, s in zip(host1, seeds)]
    for k in range(K):
        assert cfg_bytes(dl.config(rows2[k])) == cfg_bytes(build_config(host2[k], validate=False))
    # lanes 0..K-1 restart on the mutated levels with fresh seeds; the rest keep the base
    lane_seed = lane_seeds(77, K)
    dl.respawn(list(range(K)), rows2, lane_seed)
    scen = host2 + [base] * (B - K)
    seeds_all = np.concatenate([lane_seed, lane_seeds(0, B)[K:]])
    ref = orc.OracleBatchSim(scen, seeds_all, auto_reset=False)
    for t in range(6):
        out = sim.step(None)
        r = ref.step(None)
        np.testing.assert_array_equal(out.dense_reward.cpu().numpy(), r["dense_reward"])
        np.testing.assert_array_equal(out.actions.cpu().numpy(), r["actions"])
        np.testing.assert_array_equal(out.observations.cpu().numpy(),
                                      r["observations"].astype(np.float32))
    st = sim.export_state()
    np.testing.assert_array_equal(st["health"].cpu().numpy(), ref.sim.health)
    np.testing.assert_array_equal(st["pos"].cpu().numpy(), ref.sim.pos)
    sim.close()


def test_table_growth_and_errors():
    base = load_scenario(CASES["duel_default_samples"]["base"])
    spec = levels.LevelRanges.broad(base)
    sim = new_sim(base)
    dl = levels.DeviceLevels(sim)
    n0, cap0 = dl.counts()
    gens = [np.random.default_rng(s) for s in range(cap0 + 10)]
    rows = dl.sample(spec, gens)
    n1, cap1 = dl.counts()
    assert rows[0] == n0 and n1 == n0 + len(gens) and cap1 >= n1 > cap0
    with pytest.raises(ValueError, match="unknown mutation op"):
        dl.mutate("transpose", gens[:1], [0], spec)
    sim.close()
