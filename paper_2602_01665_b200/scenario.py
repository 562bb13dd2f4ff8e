"""Scenario documents for the batched step: parse, validate, serialise.

Host-side configuration only.  The document format is the reference's
schema-v1 JSON (reader: ``pkg/src/skirmish/scenario.py:143-401``; writer
``:60-131``; invariants ``pkg/src/skirmish/core.py:316-420``).  A scenario is
read once on the host and turned into a device template by
``paper_2602_01665_b200.template``; nothing here runs per step.

Error behaviour mirrors the reference: malformed documents raise
``ScenarioFormatError`` with a ``$.path: message`` text, structurally valid
but inconsistent scenarios are reported by :func:`validate_scenario`, and the
simulator refuses them with ``ScenarioFormatError("invalid scenario ...")``
(``environment.py:139-144``).
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
from dataclasses import dataclass, field as dc_field

TEAM_ALLY = 0
TEAM_ENEMY = 1

# Action ids (core.py:15-22).
ACTION_MOVE_POS_Y = 0
ACTION_MOVE_NEG_Y = 1
ACTION_MOVE_POS_X = 2
ACTION_MOVE_NEG_X = 3
ACTION_ROTATE = 4
ACTION_ATTACK = 5
ACTION_NOOP = 6
NUM_ACTIONS = 7

CONTROLLERS = ("external", "heuristic", "random")  # core.py:138
ZONE_TYPES = ("lava", "bush", "swamp")  # core.py:12; device ids are index+1

SCHEMA_VERSION = 1


class ScenarioFormatError(ValueError):
    """Malformed scenario document or invalid scenario (core.py:30)."""


class ActionMaskError(ValueError):
    """External action outside the current action mask (core.py:34)."""


@dataclass(frozen=True)
class UnitSpec:
    """Per-kind combat statistics (core.py:38-57)."""

    max_health: float
    body_radius: float
    body_mass: float
    speed: float
    attack_damage: float
    attack_range: float
    attack_cooldown: float
    sight_angle: float = 2.0 * math.pi / 3.0
    sight_range: float = 20.0
    space_occupied: int = 1
    kinematic: bool = False


SPEC_KEYS = tuple(f.name for f in dataclasses.fields(UnitSpec))

# Preset table (core.py:60-70): max_health, radius, mass, speed, damage,
# range, cooldown.
UNIT_PRESETS: dict[str, UnitSpec] = {
    "farmer": UnitSpec(60.0, 1.0, 1.0, 1.1, 14.0, 2.5, 2.5),
    "assassin": UnitSpec(70.0, 1.0, 1.0, 1.4, 22.0, 2.5, 1.5),
    "king": UnitSpec(346.0, 1.47, 10.0, 1.2, 46.0, 3.2, 2.5),
    "mammoth": UnitSpec(685.0, 4.25, 50.0, 1.2, 20.0, 3.0, 6.5, space_occupied=4),
    "archer": UnitSpec(40.0, 1.0, 1.0, 1.0, 28.0, 27.0, 8.0),
    "cannon": UnitSpec(100.0, 1.0, 5.2, 0.5, 80.0, 40.0, 10.0),
    "deadeye": UnitSpec(40.0, 1.0, 1.0, 1.1, 25.0, 20.0, 8.0),
    "healer": UnitSpec(25.0, 1.0, 1.0, 1.0, -7.0, 10.0, 2.0),
    "paladin": UnitSpec(220.0, 1.32, 8.5, 1.2, -6.0, 7.5, 2.0),
}

# Heuristic tiers (core.py:130-136): (epsilon, aggressive_threshold).
HEURISTIC_TIERS: dict[str, tuple[float, float]] = {
    "random": (1.0, 0.0),
    "novice": (0.5, 0.1),
    "medium": (0.2, 0.3),
    "advanced": (0.1, 0.5),
    "expert": (0.01, 0.7),
}


@dataclass(frozen=True)
class Field:
    width: float = 40.0
    height: float = 40.0
    margin: float = 2.0


@dataclass(frozen=True)
class Physics:
    """Integrator / contact constants (core.py:99-118); angles in degrees."""

    dt: float = 0.1
    restitution: float = 0.5
    penetration_slop: float = 0.01
    correction_percent: float = 0.8
    rotation_step_deg: float = 30.0
    boundary_damage_coeff: float = 0.1
    reveal_duration: float = 1.0
    enable_noop: bool = False


PHYSICS_KEYS = tuple(f.name for f in dataclasses.fields(Physics))


@dataclass(frozen=True)
class Team:
    id: int
    controller: str = "external"
    epsilon: float | None = None  # None <=> no heuristic block
    aggressive_threshold: float | None = None

    @property
    def has_heuristic(self) -> bool:
        return self.epsilon is not None


@dataclass(frozen=True)
class Zone:
    type: str
    center: tuple[float, float]
    semi_axes: tuple[float, float]
    effect: float = 0.0


@dataclass(frozen=True)
class Unit:
    team: int
    position: tuple[float, float]
    heading_deg: float = 0.0
    preset: str | None = None
    spec: UnitSpec | None = None
    overrides: tuple[tuple[str, object], ...] = ()

    def resolved_spec(self) -> UnitSpec:
        base = self.spec if self.spec is not None else UNIT_PRESETS[self.preset]
        if not self.overrides:
            return base
        kw = {}
        for key, value in self.overrides:
            if key == "space_occupied":
                kw[key] = int(value)
            elif key == "kinematic":
                kw[key] = bool(value)
            else:
                kw[key] = float(value)
        return dataclasses.replace(base, **kw)


def _default_teams() -> tuple[Team, Team]:
    eps, xi = HEURISTIC_TIERS["medium"]
    return (Team(TEAM_ALLY, "external"), Team(TEAM_ENEMY, "heuristic", eps, xi))


@dataclass
class Scenario:
    name: str
    units: list[Unit]
    field: Field = Field()
    physics: Physics = Physics()
    max_steps: int = 400
    teams: tuple[Team, Team] = dc_field(default_factory=_default_teams)
    zones: list[Zone] = dc_field(default_factory=list)
    max_units: int = 0
    max_zones: int = 0
    notes: list[str] = dc_field(default_factory=list, compare=False, repr=False)

    def __post_init__(self) -> None:
        if self.max_units == 0:
            self.max_units = max(len(self.units), 1)
        if self.max_zones == 0:
            self.max_zones = len(self.zones)

    def team_by_id(self, tid: int) -> Team | None:
        for t in self.teams:
            if t.id == tid:
                return t
        return None

    @property
    def obs_dim(self) -> int:
        """perception.py:40-45."""
        return 15 + (self.max_units - 1) * 17 + self.max_zones * 8

    @property
    def global_dim(self) -> int:
        """perception.py:47-49."""
        return self.max_units * 15 + self.max_zones * 8

    def with_controllers(self, ally: str | None = None, enemy: str | None = None) -> "Scenario":
        """Copy with team controllers replaced.

        Each spec is ``external``, ``random`` or ``heuristic:<tier>`` (the
        policy grammar of ``rollout.py:37-51``).
        """
        teams = list(sorted(self.teams, key=lambda t: t.id))
        for tid, spec in ((TEAM_ALLY, ally), (TEAM_ENEMY, enemy)):
            if spec is None:
                continue
            if spec in ("external", "random"):
                teams[tid] = Team(tid, spec)
            elif spec.startswith("heuristic:"):
                tier = spec.split(":", 1)[1]
                if tier not in HEURISTIC_TIERS:
                    raise ValueError(f"unknown heuristic tier {tier!r}")
                eps, xi = HEURISTIC_TIERS[tier]
                teams[tid] = Team(tid, "heuristic", eps, xi)
            else:
                raise ValueError(f"unknown policy {spec!r}")
        return dataclasses.replace(self, teams=tuple(teams), notes=list(self.notes))

    def scripted(self) -> "Scenario":
        """External teams become ``random`` (the bench rule, rollout.py:360-366)."""
        teams = tuple(
            Team(t.id, "random") if t.controller == "external" else t for t in self.teams
        )
        return dataclasses.replace(self, teams=teams, notes=list(self.notes))


# ---------------------------------------------------------------- parsing --

def _bad(path: str, msg: str):
    raise ScenarioFormatError(f"{path}: {msg}")


def _obj(v, path: str, allowed: frozenset) -> dict:
    if not isinstance(v, dict):
        _bad(path, f"expected object, got {type(v).__name__}")
    extra = set(v) - allowed
    if extra:
        _bad(path, f"unknown keys {sorted(extra)}")
    return v


def _num(v, path: str) -> float:
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        _bad(path, f"expected number, got {type(v).__name__}")
    return float(v)


def _int(v, path: str) -> int:
    if isinstance(v, bool) or not isinstance(v, int):
        _bad(path, f"expected integer, got {type(v).__name__}")
    return v


def _xy(v, path: str) -> tuple[float, float]:
    if not isinstance(v, list) or len(v) != 2:
        _bad(path, "expected [x, y]")
    return (_num(v[0], f"{path}[0]"), _num(v[1], f"{path}[1]"))


def _bool(v, path: str) -> bool:
    if not isinstance(v, bool):
        _bad(path, "expected boolean")
    return v


_TOP = frozenset({"version", "name", "field", "physics", "max_steps", "max_units",
                  "max_zones", "teams", "units", "zones"})


def scenario_from_dict(doc: dict) -> Scenario:
    """Build a Scenario from a parsed document (scenario.py:143-401)."""
    notes: list[str] = []
    root = _obj(doc, "$", _TOP)
    if "version" not in root or root["version"] is None:
        notes.append("version missing, assumed 1")
    elif _int(root["version"], "$.version") != SCHEMA_VERSION:
        _bad("$.version", f"unsupported version {root['version']}")
    if not isinstance(root.get("name"), str):
        _bad("$.name", "required string")

    if "field" in root:
        f = _obj(root["field"], "$.field", frozenset({"width", "height", "margin"}))
        fld = Field(_num(f.get("width", 40.0), "$.field.width"),
                    _num(f.get("height", 40.0), "$.field.height"),
                    _num(f.get("margin", 2.0), "$.field.margin"))
    else:
        fld = Field()
        notes.append("field missing, defaults applied")

    if "physics" in root:
        p = _obj(root["physics"], "$.physics", frozenset(PHYSICS_KEYS))
        base = Physics()
        kw = {}
        for key in PHYSICS_KEYS:
            if key not in p:
                kw[key] = getattr(base, key)
                notes.append(f"physics.{key} missing, default applied")
            elif key == "enable_noop":
                kw[key] = _bool(p[key], "$.physics.enable_noop")
            else:
                kw[key] = _num(p[key], f"$.physics.{key}")
        phys = Physics(**kw)
    else:
        phys = Physics()
        notes.append("physics missing, defaults applied")

    if "teams" in root:
        if not isinstance(root["teams"], list):
            _bad("$.teams", "expected array")
        teams = []
        for k, raw in enumerate(root["teams"]):
            path = f"$.teams[{k}]"
            t = _obj(raw, path, frozenset({"id", "controller", "heuristic"}))
            tid = _int(t.get("id", k), f"{path}.id")
            ctrl = t.get("controller", "external")
            if not isinstance(ctrl, str):
                _bad(f"{path}.controller", "expected string")
            eps = xi = None
            if "heuristic" in t:
                h = _obj(t["heuristic"], f"{path}.heuristic",
                         frozenset({"epsilon", "aggressive_threshold"}))
                eps = _num(h.get("epsilon", 0.2), f"{path}.heuristic.epsilon")
                xi = _num(h.get("aggressive_threshold", 0.3),
                          f"{path}.heuristic.aggressive_threshold")
            elif ctrl == "heuristic":
                eps, xi = HEURISTIC_TIERS["medium"]
                notes.append(f"teams[{k}].heuristic missing, medium tier applied")
            teams.append(Team(tid, ctrl, eps, xi))
        team_t = tuple(teams)
    else:
        team_t = _default_teams()
        notes.append("teams missing, defaults applied")
    if len(team_t) != 2:
        _bad("$.teams", f"expected exactly 2 teams, got {len(team_t)}")

    if not isinstance(root.get("units"), list):
        _bad("$.units", "required array")
    units = []
    for k, raw in enumerate(root["units"]):
        path = f"$.units[{k}]"
        u = _obj(raw, path, frozenset({"team", "position", "heading_deg", "preset",
                                       "overrides", "spec"}))
        if "position" not in u:
            _bad(f"{path}.position", "required")
        heading = u.get("heading_deg")
        if heading is None:
            heading = 0.0
            notes.append(f"units[{k}].heading_deg missing, 0 applied")
        else:
            heading = _num(heading, f"{path}.heading_deg")
        preset = u.get("preset")
        spec = None
        overrides: tuple = ()
        if preset is not None:
            if not isinstance(preset, str):
                _bad(f"{path}.preset", "expected string")
            if "spec" in u:
                _bad(path, "preset and spec are mutually exclusive")
            ov = u.get("overrides", {})
            if not isinstance(ov, dict):
                _bad(f"{path}.overrides", "expected object")
            items = []
            for key in sorted(ov):
                val = ov[key]
                if key == "kinematic":
                    items.append((key, _bool(val, f"{path}.overrides.kinematic")))
                elif key == "space_occupied":
                    items.append((key, _int(val, f"{path}.overrides.{key}")))
                else:
                    items.append((key, _num(val, f"{path}.overrides.{key}")))
            overrides = tuple(items)
        elif "spec" in u:
            spec = _spec_from_dict(u["spec"], f"{path}.spec")
            if "overrides" in u:
                _bad(f"{path}.overrides", "not allowed with spec")
        else:
            _bad(path, "needs preset or spec")
        units.append(Unit(team=_int(u.get("team", 0), f"{path}.team"),
                          position=_xy(u["position"], f"{path}.position"),
                          heading_deg=heading, preset=preset, spec=spec,
                          overrides=overrides))

    zones = []
    if "zones" in root:
        if not isinstance(root["zones"], list):
            _bad("$.zones", "expected array")
        for k, raw in enumerate(root["zones"]):
            path = f"$.zones[{k}]"
            z = _obj(raw, path, frozenset({"type", "center", "semi_axes", "effect"}))
            if not isinstance(z.get("type"), str):
                _bad(f"{path}.type", "required string")
            zones.append(Zone(z["type"], _xy(z.get("center", [0, 0]), f"{path}.center"),
                              _xy(z.get("semi_axes", [1, 1]), f"{path}.semi_axes"),
                              _num(z.get("effect", 0.0), f"{path}.effect")))
    else:
        notes.append("zones missing, none applied")

    def _cap(key, default, what):
        v = root.get(key)
        if v is None:
            notes.append(what)
            return default
        return _int(v, f"$.{key}")

    max_units = _cap("max_units", max(len(units), 1), "max_units missing, derived from units")
    max_zones = _cap("max_zones", len(zones), "max_zones missing, derived from zones")
    max_steps = _cap("max_steps", 400, "max_steps missing, 400 applied")
    return Scenario(name=root["name"], units=units, field=fld, physics=phys,
                    max_steps=max_steps, teams=team_t, zones=zones,
                    max_units=max_units, max_zones=max_zones, notes=notes)


def _spec_from_dict(v, path: str) -> UnitSpec:
    obj = _obj(v, path, frozenset(SPEC_KEYS))
    kw = {}
    for key in SPEC_KEYS:
        if key not in obj:
            _bad(path, f"missing key {key!r}")
        if key == "space_occupied":
            kw[key] = _int(obj[key], f"{path}.{key}")
        elif key == "kinematic":
            if not isinstance(obj[key], bool):
                _bad(f"{path}.{key}", "expected boolean")
            kw[key] = obj[key]
        else:
            kw[key] = _num(obj[key], f"{path}.{key}")
    return UnitSpec(**kw)


def load_scenario(text: str | bytes) -> Scenario:
    """Parse a document (scenario.py:387-397)."""
    if isinstance(text, (bytes, bytearray)):
        text = bytes(text).decode("utf-8")
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ScenarioFormatError(
            f"malformed JSON at line {e.lineno}, column {e.colno}: {e.msg}"
        ) from None
    return scenario_from_dict(doc)


def load_scenario_file(path) -> Scenario:
    with open(os.fspath(path), "rb") as fh:
        return load_scenario(fh.read())


SCENARIO_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios")


def builtin_scenario(name: str) -> Scenario:
    """One of the shipped benchmark scenarios (``scenarios/<name>.json``)."""
    path = os.path.join(SCENARIO_DIR, f"{name}.json")
    if not os.path.isfile(path):
        raise KeyError(f"unknown scenario {name!r}")
    return load_scenario_file(path)


def scenario_to_dict(sc: Scenario) -> dict:
    """Canonical document (scenario.py:60-131 key set)."""
    units = []
    for u in sc.units:
        d: dict = {"team": int(u.team), "position": [float(u.position[0]), float(u.position[1])],
                   "heading_deg": float(u.heading_deg)}
        if u.preset is not None:
            d["preset"] = u.preset
            if u.overrides:
                d["overrides"] = {k: (v if isinstance(v, (bool, int)) else float(v))
                                  for k, v in u.overrides}
        else:
            d["spec"] = {k: getattr(u.spec, k) for k in SPEC_KEYS}
        units.append(d)
    teams = []
    for t in sorted(sc.teams, key=lambda t: t.id):
        d = {"id": int(t.id), "controller": t.controller}
        if t.has_heuristic:
            d["heuristic"] = {"epsilon": float(t.epsilon),
                              "aggressive_threshold": float(t.aggressive_threshold)}
        teams.append(d)
    return {
        "version": SCHEMA_VERSION,
        "name": sc.name,
        "field": {"width": float(sc.field.width), "height": float(sc.field.height),
                  "margin": float(sc.field.margin)},
        "physics": {k: getattr(sc.physics, k) for k in PHYSICS_KEYS},
        "max_steps": int(sc.max_steps),
        "max_units": int(sc.max_units),
        "max_zones": int(sc.max_zones),
        "teams": teams,
        "units": units,
        "zones": [{"type": z.type, "center": list(z.center), "semi_axes": list(z.semi_axes),
                   "effect": float(z.effect)} for z in sc.zones],
    }


def save_scenario(sc: Scenario) -> str:
    return json.dumps(scenario_to_dict(sc), sort_keys=True, indent=2) + "\n"


# ------------------------------------------------------------- validation --

def _spec_violations(sp: UnitSpec, path: str, out: list[str]) -> None:
    checks = (
        (sp.max_health <= 0, f"{path}.max_health must be > 0, got {sp.max_health}"),
        (sp.body_radius <= 0, f"{path}.body_radius must be > 0, got {sp.body_radius}"),
        (sp.body_mass <= 0, f"{path}.body_mass must be > 0, got {sp.body_mass}"),
        (sp.speed < 0, f"{path}.speed must be >= 0, got {sp.speed}"),
        (sp.attack_range < 0, f"{path}.attack_range must be >= 0, got {sp.attack_range}"),
        (sp.attack_cooldown < 0,
         f"{path}.attack_cooldown must be >= 0, got {sp.attack_cooldown}"),
        (not 0.0 < sp.sight_angle <= 2.0 * math.pi + 1e-12,
         f"{path}.sight_angle must be in (0, 2*pi], got {sp.sight_angle}"),
        (sp.sight_range < 0, f"{path}.sight_range must be >= 0, got {sp.sight_range}"),
        (sp.space_occupied < 1,
         f"{path}.space_occupied must be >= 1, got {sp.space_occupied}"),
    )
    out.extend(msg for bad, msg in checks if bad)


def validate_scenario(sc: Scenario) -> list[str]:
    """All violated invariants (core.py:316-420); empty means valid."""
    v: list[str] = []
    f = sc.field
    if f.width <= 0 or f.height <= 0:
        v.append(f"field dimensions must be > 0, got {f.width}x{f.height}")
    if f.margin < 0:
        v.append(f"field.margin must be >= 0, got {f.margin}")
    elif f.width > 0 and f.height > 0 and 2 * f.margin >= min(f.width, f.height):
        v.append(f"field.margin {f.margin} leaves no interior")
    p = sc.physics
    if p.dt <= 0:
        v.append(f"physics.dt must be > 0, got {p.dt}")
    if not 0.0 <= p.restitution <= 1.0:
        v.append(f"physics.restitution must be in [0, 1], got {p.restitution}")
    if p.penetration_slop < 0:
        v.append(f"physics.penetration_slop must be >= 0, got {p.penetration_slop}")
    if not 0.0 <= p.correction_percent <= 1.0:
        v.append(f"physics.correction_percent must be in [0, 1], got {p.correction_percent}")
    if not 0.0 < p.rotation_step_deg <= 360.0:
        v.append(f"physics.rotation_step_deg must be in (0, 360], got {p.rotation_step_deg}")
    if p.boundary_damage_coeff < 0:
        v.append(f"physics.boundary_damage_coeff must be >= 0, got {p.boundary_damage_coeff}")
    if p.reveal_duration < 0:
        v.append(f"physics.reveal_duration must be >= 0, got {p.reveal_duration}")
    if sc.max_steps < 1:
        v.append(f"max_steps must be >= 1, got {sc.max_steps}")
    ids = sorted(t.id for t in sc.teams)
    if len(sc.teams) != 2 or ids != [TEAM_ALLY, TEAM_ENEMY]:
        v.append(f"exactly two teams with ids 0 and 1 required, got ids {ids}")
    for t in sc.teams:
        path = f"teams[{t.id}]"
        if t.controller not in CONTROLLERS:
            v.append(f"{path}.controller must be one of {CONTROLLERS}, got {t.controller!r}")
        if t.controller == "heuristic" and not t.has_heuristic:
            v.append(f"{path}.heuristic params required for heuristic controller")
        if t.has_heuristic:
            if not 0.0 <= t.epsilon <= 1.0:
                v.append(f"{path}.heuristic.epsilon must be in [0, 1], got {t.epsilon}")
            if not 0.0 <= t.aggressive_threshold <= 1.0:
                v.append(f"{path}.heuristic.aggressive_threshold must be in [0, 1],"
                         f" got {t.aggressive_threshold}")
    if sc.max_units < 1:
        v.append(f"max_units must be >= 1, got {sc.max_units}")
    if len(sc.units) > sc.max_units:
        v.append(f"{len(sc.units)} units exceed max_units {sc.max_units}")
    if sc.max_zones < 0:
        v.append(f"max_zones must be >= 0, got {sc.max_zones}")
    if len(sc.zones) > sc.max_zones:
        v.append(f"{len(sc.zones)} zones exceed max_zones {sc.max_zones}")
    for tid in (TEAM_ALLY, TEAM_ENEMY):
        if not any(u.team == tid for u in sc.units):
            v.append(f"team {tid} has no units")
    for i, u in enumerate(sc.units):
        path = f"units[{i}]"
        if u.team not in (TEAM_ALLY, TEAM_ENEMY):
            v.append(f"{path}.team must be 0 or 1, got {u.team}")
        if (u.preset is None) == (u.spec is None):
            v.append(f"{path} must set exactly one of preset or spec")
            continue
        if u.preset is not None and u.preset not in UNIT_PRESETS:
            v.append(f"{path}.preset unknown: {u.preset!r}")
            continue
        if u.spec is not None and u.overrides:
            v.append(f"{path}.overrides only apply to presets")
        unknown = [k for k, _ in u.overrides if k not in SPEC_KEYS]
        if unknown:
            v.append(f"{path}.overrides has unknown keys {unknown}")
            continue
        _spec_violations(u.resolved_spec(), path, v)
        x, y = u.position
        if not (0.0 <= x <= f.width and 0.0 <= y <= f.height):
            v.append(f"{path}.position ({x}, {y}) outside field")
    for i, z in enumerate(sc.zones):
        path = f"zones[{i}]"
        if z.type not in ZONE_TYPES:
            v.append(f"{path}.type must be one of {ZONE_TYPES}, got {z.type!r}")
            continue
        a, b = z.semi_axes
        if a <= 0 or b <= 0:
            v.append(f"{path}.semi_axes must be > 0 componentwise, got ({a}, {b})")
        if z.type == "lava" and z.effect <= 0:
            v.append(f"{path}.effect must be > 0 for lava, got {z.effect}")
        if z.type == "swamp" and not 0.0 < z.effect <= 1.0:
            v.append(f"{path}.effect must be in (0, 1] for swamp, got {z.effect}")
        if z.type == "bush" and z.effect != 0.0:
            v.append(f"{path}.effect must be 0 for bush, got {z.effect}")
    return v


def ensure_valid(sc: Scenario) -> None:
    """Raise like ``environment._ensure_valid`` (environment.py:139-144)."""
    bad = validate_scenario(sc)
    if bad:
        raise ScenarioFormatError(f"invalid scenario {sc.name!r}: " + "; ".join(bad[:5]))
