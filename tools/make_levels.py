"""Generate tests/golden/levels.json from the reference level generator.

Run in the build container only (imports /root/reference read-only):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tools/make_levels.py

Each case starts a ``numpy.random.default_rng(seed)``, applies a sequence of
``sample_level`` / ``mutate_level`` calls (``pkg/src/skirmish/scenario.py:696-826``)
and records the canonical JSON of every produced level plus the generator
state after each call.  The duel bases are the reference tests' own
(``pkg/tests/test_scenario.py:317-420``).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
from conftest import duel_config  # reference pkg/tests
from skirmish.core import Zone
from skirmish.scenario import (LevelGenSpec, default_level_spec, load_scenario, mutate_level,
                               sample_level, save_scenario)

HERE = os.path.dirname(os.path.abspath(__file__))
SCEN = os.path.join(HERE, "..", "paper_2602_01665_b200", "scenarios")
OUT = os.path.join(HERE, "..", "tests", "golden", "levels.json")


def scen(name):
    with open(os.path.join(SCEN, f"{name}.json"), encoding="utf-8") as fh:
        return load_scenario(fh.read())


def duel_lava_bush():
    return duel_config(zones=[Zone("lava", (20.0, 12.0), (4.0, 2.0), 5.0),
                              Zone("bush", (20.0, 28.0), (3.0, 3.0), 0.0)])


def duel_lava_swamp():
    return duel_config(zones=[Zone("lava", (20.0, 12.0), (4.0, 2.0), 5.0),
                              Zone("swamp", (20.0, 28.0), (3.0, 2.0), 0.5)])


def narrow_spec(base):
    # unit health only, two zone types, no axis range, lava range only (a
    # retyped swamp falls back to the default range), epsilon only
    return dict(categories=("unit_spec", "zones", "heuristic"),
                unit_ranges={"max_health": (50.0, 300.0)}, zone_types=("lava", "swamp"),
                zone_effect_ranges={"lava": (1.0, 4.0)}, epsilon_range=(0.05, 0.5))


# (base factory, spec kwargs or None = default_level_spec, seed, ops)
# ops: "sample" | ("mutate", op, delta, spec_from: "none" | "spec")
CASES = {
    "duel_default_samples": (duel_lava_bush, None, 0xA11CE, ["sample"] * 6),
    "duel_mutation_chain": (duel_lava_swamp, None, 3,
                            [("mutate", "perturb", 0.1, "none"), ("mutate", "swap_axes", 0.1, "none"),
                             ("mutate", "retype", 0.1, "none"), ("mutate", "perturb", 0.05, "none"),
                             ("mutate", "retype", 0.1, "none"), ("mutate", "swap_axes", 0.1, "none")]),
    "c3_default_sample_then_mutate": (lambda: scen("c3_10v10_terrain"), None, 42,
                                      ["sample", "sample", ("mutate", "perturb", 0.2, "spec"),
                                       ("mutate", "retype", 0.1, "spec"),
                                       ("mutate", "swap_axes", 0.1, "spec")]),
    "c3_narrow_spec": (lambda: scen("c3_10v10_terrain"), narrow_spec, 7,
                       ["sample", "sample", "sample", ("mutate", "perturb", 0.1, "spec"),
                        ("mutate", "retype", 0.1, "spec")]),
    "kings_no_zones": (lambda: scen("mixed_kings"), None, 11,
                       ["sample", ("mutate", "swap_axes", 0.1, "none"),
                        ("mutate", "retype", 0.1, "none"), ("mutate", "perturb", 0.3, "none")]),
    "closed_spec": (duel_lava_bush, lambda b: dict(categories=()), 5, ["sample", "sample"]),
}


def gen_state(g):
    st = g.bit_generator.state
    return {"state": str(st["state"]["state"]), "inc": str(st["state"]["inc"]),
            "has_uint32": int(st["has_uint32"]), "uinteger": int(st["uinteger"])}


def main() -> int:
    out = {}
    for name, (base_f, spec_f, seed, ops) in CASES.items():
        base = base_f()
        spec = default_level_spec(base) if spec_f is None else LevelGenSpec(base=base,
                                                                            **spec_f(base))
        g = np.random.default_rng(seed)
        cur = base
        steps = []
        for op in ops:
            if op == "sample":
                cur = sample_level(spec, g)
            else:
                _, mop, delta, spec_from = op
                cur = mutate_level(cur, mop, g, spec=None if spec_from == "none" else spec,
                                   delta=delta)
            text = save_scenario(cur)
            steps.append({"op": op if isinstance(op, str) else list(op),
                          "sha256": hashlib.sha256(text.encode()).hexdigest(),
                          "text": text if len(cur.units) <= 8 else None,
                          "rng": gen_state(g)})
        out[name] = {"base": save_scenario(base), "seed": seed,
                     "spec": None if spec_f is None else spec_f(base), "steps": steps}
        print(name, [s["sha256"][:8] for s in steps])
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
