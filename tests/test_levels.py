"""Level sampling / mutation, host restatement.

``oracle/levels_oracle.py`` (the checker of the device batch) must reproduce the reference generator draw
for draw: the canonical JSON of every level and the numpy generator state
after every call equal ``tests/golden/levels.json`` (``tools/make_levels.py``
over ``pkg/src/skirmish/scenario.py:696-826``).  Spec validation follows
``pkg/tests/test_scenario.py:275-312``.  The device batch
(``DeviceLevels``) is checked against this mirror in ``test_gpu_levels.py``.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import harness  # noqa: F401  (puts oracle/ on sys.path)
import levels_oracle as levels
from paper_2602_01665_b200.scenario import load_scenario, save_scenario

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "levels.json")
with open(GOLDEN, encoding="utf-8") as _fh:
    CASES = json.load(_fh)


def make_spec(case):
    base = load_scenario(case["base"])
    if case["spec"] is None:
        return base, levels.default_level_spec(base)
    kw = dict(case["spec"])
    for k in ("categories", "zone_types"):
        if k in kw:
            kw[k] = tuple(kw[k])
    return base, levels.LevelGenSpec(base=base, **kw)


def gen_state(g):
    st = g.bit_generator.state
    return {"state": str(st["state"]["state"]), "inc": str(st["state"]["inc"]),
            "has_uint32": int(st["has_uint32"]), "uinteger": int(st["uinteger"])}


def replay(case):
    """Yield (step record, produced scenario, generator state) along a case."""
    base, spec = make_spec(case)
    g = np.random.default_rng(case["seed"])
    cur = base
    for step in case["steps"]:
        op = step["op"]
        if op == "sample":
            cur = levels.sample_level(spec, g)
        else:
            _, mop, delta, spec_from = op
            cur = levels.mutate_level(cur, mop, g, spec=None if spec_from == "none" else spec,
                                      delta=delta)
        yield step, cur, gen_state(g)


@pytest.mark.parametrize("name", sorted(CASES))
def test_levels_match_reference(name):
    for step, cur, st in replay(CASES[name]):
        text = save_scenario(cur)
        if step["text"] is not None:
            assert text == step["text"]
        assert hashlib.sha256(text.encode()).hexdigest() == step["sha256"]
        assert st == step["rng"]


def test_spec_validation():
    base = load_scenario(CASES["duel_default_samples"]["base"])
    with pytest.raises(ValueError, match="unknown category"):
        levels.LevelGenSpec(base=base, categories=("units",))
    with pytest.raises(ValueError, match="unknown unit range field"):
        levels.LevelGenSpec(base=base, unit_ranges={"body_mass": (1, 2)})
    with pytest.raises(ValueError, match="bush"):
        levels.LevelGenSpec(base=base, zone_effect_ranges={"bush": (0.0, 1.0)})
    with pytest.raises(ValueError, match="min > max"):
        levels.LevelGenSpec(base=base, unit_ranges={"speed": (2.0, 1.0)})
    with pytest.raises(ValueError, match="unknown zone type"):
        levels.LevelGenSpec(base=base, zone_types=("mud",))
    with pytest.raises(ValueError, match="unknown mutation op"):
        levels.mutate_level(base, "transpose", np.random.default_rng(0))
    spec = levels.LevelGenSpec(base=base, unit_ranges={"max_health": (-50.0, 900.0)},
                               zone_effect_ranges={"swamp": (0.0, 3.0)}, epsilon_range=(-1.0, 2.0))
    assert dict(spec.unit_ranges)["max_health"][0] == 1.0
    assert dict(spec.zone_effect_ranges)["swamp"] == (0.01, 1.0)
    assert spec.epsilon_range == (0.0, 1.0)
    assert levels.LevelGenSpec(base=base).center_box() == ((2.0, 38.0), (2.0, 38.0))


def test_closed_spec_and_zero_delta_keep_the_base():
    case = CASES["duel_mutation_chain"]
    base = load_scenario(case["base"])
    out = levels.sample_level(levels.LevelGenSpec(base=base, categories=()),
                              np.random.default_rng(1))
    assert save_scenario(out) == save_scenario(base)
    out = levels.mutate_level(base, "perturb", np.random.default_rng(2), delta=0.0)
    for ub, um in zip(base.units, out.units):
        assert um.resolved_spec() == ub.resolved_spec()
    assert out.zones == base.zones and out.teams == base.teams


def test_device_ranges_resolve_like_the_reference_spec():
    """The product's LevelRanges (what DeviceLevels reads) resolves every
    range exactly as the reference's LevelGenSpec does, and rejects the same
    inputs (scenario.py:581-663)."""
    from paper_2602_01665_b200.levels import LevelRanges, level_spec_struct
    base = load_scenario(CASES["duel_default_samples"]["base"])
    for bad in (dict(open=("units",)), dict(units={"body_mass": (1, 2)}),
                dict(zone_effects={"bush": (0.0, 1.0)}), dict(units={"speed": (2.0, 1.0)}),
                dict(zone_types=("mud",))):
        with pytest.raises(ValueError):
            LevelRanges(base, **bad)
    r = LevelRanges(base, units={"max_health": (-50.0, 900.0)}, zone_effects={"swamp": (0.0, 3.0)},
                    epsilon=(-1.0, 2.0), zone_axes=(-1.0, 0.05), aggressive=(-2.0, 0.5))
    h = levels.LevelGenSpec(base=base, unit_ranges={"max_health": (-50.0, 900.0)},
                            zone_effect_ranges={"swamp": (0.0, 3.0)}, epsilon_range=(-1.0, 2.0),
                            zone_axis_range=(-1.0, 0.05), aggressive_range=(-2.0, 0.5))
    assert r.units == dict(h.unit_ranges)
    assert r.zone_effects == dict(h.zone_effect_ranges)
    assert (r.epsilon, r.zone_axes, r.aggressive) == (h.epsilon_range, h.zone_axis_range,
                                                      h.aggressive_range)
    assert r.center_box == h.center_box() == ((2.0, 38.0), (2.0, 38.0))
    b, d = LevelRanges.broad(base), levels.default_level_spec(base)
    assert b.units == dict(d.unit_ranges) and b.zone_effects == dict(d.zone_effect_ranges)
    assert (b.epsilon, b.zone_axes, b.aggressive) == (d.epsilon_range, d.zone_axis_range,
                                                      d.aggressive_range)
    s = level_spec_struct(b)
    assert (s.open_units, s.open_zones, s.open_heuristic, s.n_zone_types) == (1, 1, 1, 3)
    assert list(s.unit_open) == [1, 1, 1] and (s.unit_lo[1], s.unit_hi[1]) == (20.0, 800.0)
