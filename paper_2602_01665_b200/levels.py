"""Level sampling and mutation on the device.

``DeviceLevels`` runs the reference's ``sample_level`` / ``mutate_level``
(``pkg/src/skirmish/scenario.py:696-826``) for a whole batch of levels on the
GPU, one warp per level (``tabx_levels``), writing ``tabx_config`` rows
straight into a simulator's config table, so a curriculum can resample or
mutate thousands of levels and respawn lanes on them
(``tabx_respawn_lanes``) without building configs on the host.  Each level
draws from its own PCG64 stream whose state is the numpy bit generator's
(128-bit LCG, XSL-RR output, the buffered 32-bit half used by bounded
integers), so a device level equals the reference's level built from the
same ``Generator(PCG64(...))`` and the generators' states advance
identically (checked against a host restatement in ``oracle/`` by
``tests/test_gpu_levels.py``).

``LevelRanges`` describes the free parameters: which categories are open
and the ranges draws come from, resolved (clipped to each field's
invariants, ``scenario.py:581-663``) into the ``tabx_level_spec`` the
kernel reads.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np

from .scenario import ZONE_TYPES, Scenario

# unit fields a level may redraw, in the kernel's (sorted-name) order, with
# the (floor, ceiling) each drawn range is clipped to
UNIT_FIELDS = {"attack_damage": (None, None), "max_health": (1.0, None), "speed": (0.0, None)}
EFFECT_BOUNDS = {"lava": (0.01, None), "swamp": (0.01, 1.0)}
AXIS_FLOOR = 0.1
OPEN_ALL = ("unit_spec", "zones", "heuristic")
MUTATION_OPS = ("perturb", "swap_axes", "retype")


def _resolve(rng, floor, ceil):
    lo, hi = float(rng[0]), float(rng[1])
    if lo > hi:
        raise ValueError(f"range ({rng[0]}, {rng[1]}) has min > max")
    if floor is not None:
        lo, hi = max(lo, floor), max(hi, floor)
    if ceil is not None:
        lo, hi = min(lo, ceil), min(hi, ceil)
    return lo, hi


@dataclass(frozen=True)
class LevelRanges:
    """Free-parameter ranges around a base scenario.  ``None`` for a range
    keeps the base value; an empty ``open`` freezes everything."""

    base: Scenario
    open: tuple = OPEN_ALL
    units: dict = field(default_factory=dict)        # field -> (lo, hi)
    zone_types: tuple = ZONE_TYPES
    center_box: tuple | None = None                  # ((x0, x1), (y0, y1))
    zone_axes: tuple | None = None
    zone_effects: dict = field(default_factory=dict)  # "lava" / "swamp" -> (lo, hi)
    epsilon: tuple | None = None
    aggressive: tuple | None = None

    def __post_init__(self):
        bad = [c for c in self.open if c not in OPEN_ALL]
        if bad:
            raise ValueError(f"unknown category {bad[0]!r}")
        units = {}
        for name, rng in self.units.items():
            if name not in UNIT_FIELDS:
                raise ValueError(f"unknown unit range field {name!r}")
            units[name] = _resolve(rng, *UNIT_FIELDS[name])
        effects = {}
        for name, rng in self.zone_effects.items():
            if name not in EFFECT_BOUNDS:
                raise ValueError(f"{name} zones have no effect range")
            effects[name] = _resolve(rng, *EFFECT_BOUNDS[name])
        for t in self.zone_types:
            if t not in ZONE_TYPES:
                raise ValueError(f"unknown zone type {t!r}")
        set_ = object.__setattr__
        set_(self, "units", units)
        set_(self, "zone_effects", effects)
        if self.zone_axes is not None:
            set_(self, "zone_axes", _resolve(self.zone_axes, AXIS_FLOOR, None))
        if self.epsilon is not None:
            set_(self, "epsilon", _resolve(self.epsilon, 0.0, 1.0))
        if self.aggressive is not None:
            set_(self, "aggressive", _resolve(self.aggressive, 0.0, None))
        if self.center_box is None:
            f = self.base.field
            set_(self, "center_box", ((f.margin, f.width - f.margin),
                                      (f.margin, f.height - f.margin)))

    @classmethod
    def broad(cls, base: Scenario) -> "LevelRanges":
        """Every category open with the reference's default ranges
        (``default_level_spec``, scenario.py:666-679)."""
        return cls(base, units={"max_health": (20.0, 800.0), "speed": (0.5, 1.5),
                                "attack_damage": (-10.0, 80.0)},
                   zone_axes=(1.5, 6.0), zone_effects={"lava": (2.0, 10.0), "swamp": (0.2, 0.8)},
                   epsilon=(0.0, 1.0), aggressive=(0.0, 0.7))

# ------------------------------------------------------------- device batch --

_ZONE_CODE = {"lava": 1, "bush": 2, "swamp": 3}
_M64 = (1 << 64) - 1


def level_spec_struct(r: LevelRanges):
    """The tabx_level_spec of resolved ranges (include/tabx.h)."""
    from . import _native as nat
    s = nat.TabxLevelSpec()
    s.open_units = int("unit_spec" in r.open)
    s.open_zones = int("zones" in r.open)
    s.open_heuristic = int("heuristic" in r.open)
    for f, name in enumerate(UNIT_FIELDS):
        if name in r.units:
            s.unit_open[f] = 1
            s.unit_lo[f], s.unit_hi[f] = r.units[name]
    s.n_zone_types = len(r.zone_types)
    for k, t in enumerate(r.zone_types):
        s.zone_types[k] = _ZONE_CODE[t]
    (s.box_x0, s.box_x1), (s.box_y0, s.box_y1) = r.center_box
    if r.zone_axes is not None:
        s.axis_open = 1
        s.axis_lo, s.axis_hi = r.zone_axes
    for name, (lo, hi) in r.zone_effects.items():
        c = _ZONE_CODE[name]
        s.effect_open[c] = 1
        s.effect_lo[c], s.effect_hi[c] = lo, hi
    if r.epsilon is not None:
        s.eps_open = 1
        s.eps_lo, s.eps_hi = r.epsilon
    if r.aggressive is not None:
        s.agg_open = 1
        s.agg_lo, s.agg_hi = r.aggressive
    return s


def pcg_states(gens) -> np.ndarray:
    """numpy PCG64 generators -> packed tabx_pcg64 records (uint64 [n, 5])."""
    out = np.zeros((len(gens), 5), np.uint64)
    for k, g in enumerate(gens):
        st = g.bit_generator.state
        if st["bit_generator"] != "PCG64":
            raise ValueError(f"device levels need PCG64 generators, got {st['bit_generator']}")
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        out[k, 0], out[k, 1] = s >> 64, s & _M64
        out[k, 2], out[k, 3] = inc >> 64, inc & _M64
        out[k, 4] = (int(st["uinteger"]) << 32) | int(st["has_uint32"])
    return out


def set_pcg_states(gens, packed: np.ndarray) -> None:
    """Write device-advanced states back into the numpy generators."""
    for g, r in zip(gens, packed):
        st = g.bit_generator.state
        st["state"]["state"] = (int(r[0]) << 64) | int(r[1])
        st["has_uint32"] = int(r[4]) & 0xFFFFFFFF
        st["uinteger"] = int(r[4]) >> 32
        g.bit_generator.state = st


class DeviceLevels:
    """The reference's sample_level / mutate_level for a batch of levels on the device.

    Levels live in the rows of ``sim``'s config table; ``sample`` and
    ``mutate`` write rows with one warp per level (``tabx_levels``) and
    advance the given numpy generators exactly as the host functions would;
    ``respawn`` starts lanes on chosen rows (``tabx_respawn_lanes`` +
    ``init_output``, i.e. ``reset_env`` for many lanes at once).
    """

    def __init__(self, sim):
        self.sim = sim

    def _lib(self):
        from . import _native as nat
        return nat, nat.lib()

    def counts(self) -> tuple[int, int]:
        nat, L = self._lib()
        n, cap = ct.c_int32(), ct.c_int32()
        nat.check(L.tabx_num_configs(self.sim.handle, ct.byref(n), ct.byref(cap)),
                  "tabx_num_configs")
        return n.value, cap.value

    def reserve(self, capacity: int) -> None:
        nat, L = self._lib()
        nat.check(L.tabx_reserve_configs(self.sim.handle, int(capacity)), "tabx_reserve_configs")

    def config(self, slot: int):
        nat, L = self._lib()
        c = nat.TabxConfig()
        nat.check(L.tabx_get_config(self.sim.handle, int(slot), ct.byref(c)), "tabx_get_config")
        return c

    def _run(self, op: int, spec: LevelRanges, gens, src, dst_first, delta: float):
        import torch
        nat, L = self._lib()
        count = len(gens)
        n, cap = self.counts()
        if dst_first is None:
            dst_first = n
        if dst_first + count > cap:
            self.reserve(max(dst_first + count, 2 * cap))
        dev = self.sim.device
        rng_t = torch.from_numpy(pcg_states(gens).view(np.int64)).to(dev)
        src_t = None
        if src is not None:
            src_t = torch.as_tensor(np.broadcast_to(np.asarray(src, np.int32), (count,)).copy(),
                                    device=dev)
        sp = level_spec_struct(spec)
        self.sim._consume(rng_t, src_t)
        with torch.cuda.device(dev):
            nat.check(L.tabx_levels(self.sim.handle, op, ct.byref(sp), float(delta),
                                    None if src_t is None else ct.c_void_p(src_t.data_ptr()),
                                    int(dst_first), count, ct.c_void_p(rng_t.data_ptr())),
                      "tabx_levels")
        self.sim._publish()  # the generator states are read back on this stream
        set_pcg_states(gens, rng_t.cpu().numpy().view(np.uint64))
        return list(range(dst_first, dst_first + count))

    def sample(self, spec: LevelRanges, gens, base_slot=0, dst_first=None) -> list[int]:
        """Row per generator: a level sampled from ``spec`` over the base row(s)
        (scenario.py:696-747)."""
        return self._run(nat_op("sample"), spec, gens, base_slot, dst_first, 0.0)

    def mutate(self, op: str, gens, slots, spec: LevelRanges, delta: float = 0.1,
               dst_first=None) -> list[int]:
        """Row per generator: row ``slots[k]`` mutated by ``op``
        (scenario.py:753-826); ``slots=None`` mutates rows dst_first.. in place."""
        if op not in MUTATION_OPS:
            raise ValueError(f"unknown mutation op {op!r}; expected one of {MUTATION_OPS}")
        return self._run(nat_op(op), spec, gens, slots, dst_first, delta)

    def respawn(self, lanes, slots=None, seeds=None) -> None:
        """Lanes restart on the given rows / seeds, then init_output."""
        import torch
        nat, L = self._lib()
        dev = self.sim.device
        lanes_t = torch.as_tensor(np.asarray(lanes, np.int64), device=dev)
        slots_t = None if slots is None else torch.as_tensor(np.asarray(slots, np.int32),
                                                             device=dev)
        seeds_t = None if seeds is None else torch.as_tensor(
            np.asarray(seeds, np.uint64).view(np.int64), device=dev)
        p = lambda t: None if t is None else ct.c_void_p(t.data_ptr())  # noqa: E731
        self.sim._consume(lanes_t, slots_t, seeds_t)
        with torch.cuda.device(dev):
            nat.check(L.tabx_respawn_lanes(self.sim.handle, p(lanes_t), p(slots_t), p(seeds_t),
                                           lanes_t.numel()), "tabx_respawn_lanes")
        if slots is not None:
            self.sim.lane_slots[np.asarray(lanes, np.int64)] = np.asarray(slots, np.int32)
        self.sim._init_output()
        self.sim._stream.synchronize()


def nat_op(name: str) -> int:
    return {"sample": 0, "perturb": 1, "swap_axes": 2, "retype": 3}[name]
