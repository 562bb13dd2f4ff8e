"""Level sampling and mutation, host API + device batch.

Host functions mirror ``pkg/src/skirmish/scenario.py:563-826`` draw for draw
on a ``numpy.random.Generator``:

* ``LevelGenSpec`` (``:581-663``) with the same validation messages and
  invariant clipping, ``default_level_spec`` (``:666-679``);
* ``sample_level(spec, rng)`` (``:696-747``);
* ``mutate_level(config, op, rng, spec=None, delta=0.1)`` (``:753-826``).

``DeviceLevels`` runs the same two functions for a whole batch of levels on
the GPU, one warp per level, writing the resulting ``tabx_config`` rows
straight into a simulator's config table (``tabx_levels``), so a curriculum
can resample or mutate thousands of levels and respawn lanes on them
(``tabx_respawn_lanes``) without building configs on the host.  Each level
draws from its own PCG64 stream whose state is the numpy bit generator's
(128-bit LCG, XSL-RR output, the buffered 32-bit half used by bounded
integers), so a device level equals ``build_config(sample_level(spec,
Generator(PCG64(...))))`` and the generators' states advance identically.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, replace

import numpy as np

from .scenario import ZONE_TYPES, Scenario, Team, Unit, Zone

UNIT_FREE_FIELDS = ("attack_damage", "max_health", "speed")
LAVA_DAMAGE_RANGE = (2.0, 10.0)   # scenario.py:41
SWAMP_MULT_RANGE = (0.2, 0.8)     # scenario.py:42
ZONE_AXIS_RANGE = (1.5, 6.0)      # scenario.py:43
_MIN_HEALTH = 1.0
_MIN_AXIS = 0.1
_MIN_EFFECT = 0.01
MUTATION_OPS = ("perturb", "swap_axes", "retype")
CATEGORIES = ("unit_spec", "zones", "heuristic")


def _clip_range(lo: float, hi: float, floor: float | None, ceil: float | None):
    if lo > hi:
        raise ValueError(f"range ({lo}, {hi}) has min > max")
    if floor is not None:
        lo, hi = max(lo, floor), max(hi, floor)
    if ceil is not None:
        lo, hi = min(lo, ceil), min(hi, ceil)
    return (float(lo), float(hi))


@dataclass(frozen=True)
class LevelGenSpec:
    """Free-parameter ranges around a base scenario (scenario.py:581-663)."""

    base: Scenario
    categories: tuple = CATEGORIES
    unit_ranges: tuple | dict = ()
    zone_types: tuple = ZONE_TYPES
    zone_center_box: tuple | None = None
    zone_axis_range: tuple | None = None
    zone_effect_ranges: tuple | dict = ()
    epsilon_range: tuple | None = None
    aggressive_range: tuple | None = None

    def __post_init__(self):
        for cat in self.categories:
            if cat not in CATEGORIES:
                raise ValueError(f"unknown category {cat!r}")
        ur = dict(self.unit_ranges)
        for name in ur:
            if name not in UNIT_FREE_FIELDS:
                raise ValueError(f"unknown unit range field {name!r}")
        if "max_health" in ur:
            ur["max_health"] = _clip_range(*ur["max_health"], _MIN_HEALTH, None)
        if "speed" in ur:
            ur["speed"] = _clip_range(*ur["speed"], 0.0, None)
        if "attack_damage" in ur:
            ur["attack_damage"] = _clip_range(*ur["attack_damage"], None, None)
        object.__setattr__(self, "unit_ranges", tuple(sorted((k, v) for k, v in ur.items())))
        er = dict(self.zone_effect_ranges)
        if "lava" in er:
            er["lava"] = _clip_range(*er["lava"], _MIN_EFFECT, None)
        if "swamp" in er:
            er["swamp"] = _clip_range(*er["swamp"], _MIN_EFFECT, 1.0)
        if "bush" in er:
            raise ValueError("bush zones have no effect range")
        object.__setattr__(self, "zone_effect_ranges",
                           tuple(sorted((k, v) for k, v in er.items())))
        if self.zone_axis_range is not None:
            object.__setattr__(self, "zone_axis_range",
                               _clip_range(*self.zone_axis_range, _MIN_AXIS, None))
        if self.epsilon_range is not None:
            object.__setattr__(self, "epsilon_range", _clip_range(*self.epsilon_range, 0.0, 1.0))
        if self.aggressive_range is not None:
            object.__setattr__(self, "aggressive_range",
                               _clip_range(*self.aggressive_range, 0.0, None))
        for t in self.zone_types:
            if t not in ZONE_TYPES:
                raise ValueError(f"unknown zone type {t!r}")

    def center_box(self):
        if self.zone_center_box is not None:
            return self.zone_center_box
        f = self.base.field
        return ((f.margin, f.width - f.margin), (f.margin, f.height - f.margin))

    def effect_range(self, ztype: str):
        for name, rng in self.zone_effect_ranges:
            if name == ztype:
                return rng
        return None


def default_level_spec(base: Scenario) -> LevelGenSpec:
    """All three categories open with broad but safe ranges (scenario.py:666-679)."""
    return LevelGenSpec(
        base=base,
        unit_ranges={"max_health": (20.0, 800.0), "speed": (0.5, 1.5),
                     "attack_damage": (-10.0, 80.0)},
        zone_axis_range=ZONE_AXIS_RANGE,
        zone_effect_ranges={"lava": LAVA_DAMAGE_RANGE, "swamp": SWAMP_MULT_RANGE},
        epsilon_range=(0.0, 1.0),
        aggressive_range=(0.0, 0.7),
    )


def _with_unit_fields(u: Unit, fields: dict) -> Unit:
    if not fields:
        return u
    if u.preset is not None:
        merged = dict(u.overrides)
        merged.update(fields)
        return replace(u, overrides=tuple(sorted(merged.items())))
    return replace(u, spec=replace(u.spec, **fields))


def _unit_value(u: Unit, name: str) -> float:
    return float(getattr(u.resolved_spec(), name))


def _copy(sc: Scenario, **kw) -> Scenario:
    return replace(sc, units=list(sc.units), zones=list(sc.zones), notes=list(sc.notes), **kw)


def sample_level(spec: LevelGenSpec, rng: np.random.Generator) -> Scenario:
    """Base config with every open free parameter redrawn uniformly."""
    out = _copy(spec.base)
    if "unit_spec" in spec.categories and spec.unit_ranges:
        for i, u in enumerate(out.units):
            drawn = {name: float(rng.uniform(lo, hi)) for name, (lo, hi) in spec.unit_ranges}
            out.units[i] = _with_unit_fields(u, drawn)
    if "zones" in spec.categories:
        (x0, x1), (y0, y1) = spec.center_box()
        for i, z in enumerate(out.zones):
            ztype = str(rng.choice(spec.zone_types))
            center = (float(rng.uniform(x0, x1)), float(rng.uniform(y0, y1)))
            if spec.zone_axis_range is not None:
                axes = (float(rng.uniform(*spec.zone_axis_range)),
                        float(rng.uniform(*spec.zone_axis_range)))
            else:
                axes = z.semi_axes
            er = spec.effect_range(ztype)
            if ztype == "bush":
                effect = 0.0
            elif er is not None:
                effect = float(rng.uniform(*er))
            elif ztype == z.type:
                effect = z.effect
            else:
                lo, hi = LAVA_DAMAGE_RANGE if ztype == "lava" else SWAMP_MULT_RANGE
                effect = float(rng.uniform(lo, hi))
            out.zones[i] = Zone(ztype, center, axes, effect)
    if "heuristic" in spec.categories:
        out.teams = tuple(_redraw_team(t, spec, rng) for t in out.teams)
    return out


def _redraw_team(t: Team, spec: LevelGenSpec, rng) -> Team:
    if t.controller != "heuristic" or not t.has_heuristic:
        return t
    eps, agg = t.epsilon, t.aggressive_threshold
    if spec.epsilon_range is not None:
        eps = float(rng.uniform(*spec.epsilon_range))
    if spec.aggressive_range is not None:
        agg = float(rng.uniform(*spec.aggressive_range))
    return replace(t, epsilon=eps, aggressive_threshold=agg)


def mutate_level(config: Scenario, op: str, rng: np.random.Generator,
                 spec: LevelGenSpec | None = None, delta: float = 0.1) -> Scenario:
    """One mutation: noise on all free parameters, or a single zone edit."""
    if op not in MUTATION_OPS:
        raise ValueError(f"unknown mutation op {op!r}; expected one of {MUTATION_OPS}")
    if spec is None:
        spec = default_level_spec(config)
    out = _copy(config)
    if op == "perturb":
        def bump(value: float, lo: float, hi: float) -> float:
            width = hi - lo
            nudged = value + float(rng.uniform(-delta * width, delta * width))
            return float(min(max(nudged, lo), hi))

        if "unit_spec" in spec.categories:
            for i, u in enumerate(out.units):
                nudged = {name: bump(_unit_value(u, name), lo, hi)
                          for name, (lo, hi) in spec.unit_ranges}
                out.units[i] = _with_unit_fields(u, nudged)
        if "zones" in spec.categories:
            (x0, x1), (y0, y1) = spec.center_box()
            for i, z in enumerate(out.zones):
                cx = bump(z.center[0], x0, x1)
                cy = bump(z.center[1], y0, y1)
                if spec.zone_axis_range is not None:
                    lo, hi = spec.zone_axis_range
                    axes = (bump(z.semi_axes[0], lo, hi), bump(z.semi_axes[1], lo, hi))
                else:
                    axes = z.semi_axes
                er = spec.effect_range(z.type)
                effect = bump(z.effect, *er) if er is not None else z.effect
                out.zones[i] = Zone(z.type, (cx, cy), axes, effect)
        if "heuristic" in spec.categories:
            teams = []
            for t in out.teams:
                if t.controller == "heuristic" and t.has_heuristic:
                    eps, agg = t.epsilon, t.aggressive_threshold
                    if spec.epsilon_range is not None:
                        eps = bump(eps, *spec.epsilon_range)
                    if spec.aggressive_range is not None:
                        agg = bump(agg, *spec.aggressive_range)
                    t = replace(t, epsilon=eps, aggressive_threshold=agg)
                teams.append(t)
            out.teams = tuple(teams)
        return out
    if not out.zones:
        return out
    idx = int(rng.integers(len(out.zones)))
    z = out.zones[idx]
    if op == "swap_axes":
        out.zones[idx] = replace(z, semi_axes=(z.semi_axes[1], z.semi_axes[0]))
    else:
        new_type = str(rng.choice(spec.zone_types))
        if new_type == "bush":
            effect = 0.0
        else:
            er = spec.effect_range(new_type)
            if er is None:
                er = LAVA_DAMAGE_RANGE if new_type == "lava" else SWAMP_MULT_RANGE
            effect = float(rng.uniform(*er))
        out.zones[idx] = replace(z, type=new_type, effect=effect)
    return out


# ------------------------------------------------------------- device batch --

_ZONE_CODE = {"lava": 1, "bush": 2, "swamp": 3}
_M64 = (1 << 64) - 1


def level_spec_struct(spec: LevelGenSpec):
    """The tabx_level_spec of a LevelGenSpec (include/tabx.h)."""
    from . import _native as nat
    s = nat.TabxLevelSpec()
    s.open_units = int("unit_spec" in spec.categories)
    s.open_zones = int("zones" in spec.categories)
    s.open_heuristic = int("heuristic" in spec.categories)
    ranges = dict(spec.unit_ranges)
    for f, name in enumerate(UNIT_FREE_FIELDS):  # sorted-name order
        if name in ranges:
            s.unit_open[f] = 1
            s.unit_lo[f], s.unit_hi[f] = ranges[name]
    s.n_zone_types = len(spec.zone_types)
    for k, t in enumerate(spec.zone_types):
        s.zone_types[k] = _ZONE_CODE[t]
    (s.box_x0, s.box_x1), (s.box_y0, s.box_y1) = spec.center_box()
    if spec.zone_axis_range is not None:
        s.axis_open = 1
        s.axis_lo, s.axis_hi = spec.zone_axis_range
    for name, (lo, hi) in spec.zone_effect_ranges:
        c = _ZONE_CODE[name]
        s.effect_open[c] = 1
        s.effect_lo[c], s.effect_hi[c] = lo, hi
    if spec.epsilon_range is not None:
        s.eps_open = 1
        s.eps_lo, s.eps_hi = spec.epsilon_range
    if spec.aggressive_range is not None:
        s.agg_open = 1
        s.agg_lo, s.agg_hi = spec.aggressive_range
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
    """sample_level / mutate_level for a batch of levels on the device.

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

    def _run(self, op: int, spec: LevelGenSpec, gens, src, dst_first, delta: float):
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
        with torch.cuda.device(dev):
            nat.check(L.tabx_levels(self.sim.handle, op, ct.byref(sp), float(delta),
                                    None if src_t is None else ct.c_void_p(src_t.data_ptr()),
                                    int(dst_first), count, ct.c_void_p(rng_t.data_ptr())),
                      "tabx_levels")
        set_pcg_states(gens, rng_t.cpu().numpy().view(np.uint64))
        return list(range(dst_first, dst_first + count))

    def sample(self, spec: LevelGenSpec, gens, base_slot=0, dst_first=None) -> list[int]:
        """Row per generator: sample_level(spec, g) over the base row(s)."""
        return self._run(nat_op("sample"), spec, gens, base_slot, dst_first, 0.0)

    def mutate(self, op: str, gens, slots, spec: LevelGenSpec, delta: float = 0.1,
               dst_first=None) -> list[int]:
        """Row per generator: mutate_level(row slots[k], op, g, spec, delta);
        ``slots=None`` mutates rows dst_first.. in place."""
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
        with torch.cuda.device(dev):
            nat.check(L.tabx_respawn_lanes(self.sim.handle, p(lanes_t), p(slots_t), p(seeds_t),
                                           lanes_t.numel()), "tabx_respawn_lanes")
        self.sim._init_output()
        torch.cuda.current_stream(dev).synchronize()


def nat_op(name: str) -> int:
    return {"sample": 0, "perturb": 1, "swap_axes": 2, "retype": 3}[name]
