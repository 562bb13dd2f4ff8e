"""Scenario -> device template (``tabx_config``).

Host-side restatement of ``fill_env``'s static columns
(``pkg/src/skirmish/arrays.py:244-351``).  Radians and ``cos(sight/2)`` are
computed with numpy here, exactly as the reference computes them, so the
spawn state on the device is bit-identical by construction; the device only
copies these values.
"""
from __future__ import annotations

import numpy as np

from ._native import MAX_UNITS, MAX_ZONES, TabxConfig
from .scenario import CONTROLLERS, Scenario, ensure_valid

ZONE_IDS = {"lava": 1, "bush": 2, "swamp": 3}
ASSASSIN_SPEED = 1.4  # arrays.py:31
RANGER_RANGE = 10.0  # arrays.py:32


def build_config(sc: Scenario, validate: bool = True) -> TabxConfig:
    if validate:
        ensure_valid(sc)
    N, Z = sc.max_units, sc.max_zones
    if not 1 <= N <= MAX_UNITS:
        raise ValueError(f"max_units {N} outside 1..{MAX_UNITS}")
    if not 0 <= Z <= MAX_ZONES:
        raise ValueError(f"max_zones {Z} outside 0..{MAX_ZONES}")
    c = TabxConfig()
    c.n_units, c.n_zones, c.max_steps = N, Z, int(sc.max_steps)
    ph = sc.physics
    c.enable_noop = 1 if ph.enable_noop else 0
    for t in sc.teams:
        c.controller[t.id] = CONTROLLERS.index(t.controller)
        c.epsilon[t.id] = float(t.epsilon) if t.has_heuristic else 0.0
        c.aggressive[t.id] = float(t.aggressive_threshold) if t.has_heuristic else 0.0
    c.dt = ph.dt
    c.restitution = ph.restitution
    c.slop = ph.penetration_slop
    c.correction = ph.correction_percent
    c.rot_step = float(np.radians(ph.rotation_step_deg))
    c.boundary_coeff = ph.boundary_damage_coeff
    c.reveal_duration = ph.reveal_duration
    c.field_w = sc.field.width
    c.field_h = sc.field.height
    # padding defaults (arrays.py:320-326); other columns stay zero
    for i in range(N):
        c.max_health[i] = 1.0
        c.mass[i] = 1.0
        c.inv_mass[i] = 1.0
        c.sight_cos_half[i] = 1.0
    for i, u in enumerate(sc.units):
        sp = u.resolved_spec()
        c.active[i] = 1
        c.team[i] = int(u.team)
        c.kinematic[i] = 1 if sp.kinematic else 0
        c.role_assassin[i] = 1 if sp.speed >= ASSASSIN_SPEED else 0
        c.role_ranger[i] = 1 if (sp.attack_range >= RANGER_RANGE and sp.attack_damage > 0) else 0
        c.role_healer[i] = 1 if sp.attack_damage < 0 else 0
        c.max_health[i] = sp.max_health
        c.radius[i] = sp.body_radius
        c.mass[i] = sp.body_mass
        c.inv_mass[i] = 0.0 if sp.kinematic else 1.0 / sp.body_mass
        c.speed[i] = sp.speed
        c.damage[i] = sp.attack_damage
        c.attack_range[i] = sp.attack_range
        c.cooldown[i] = sp.attack_cooldown
        c.sight_angle[i] = sp.sight_angle
        c.sight_cos_half[i] = float(np.cos(sp.sight_angle / 2.0))
        c.sight_range[i] = sp.sight_range
        c.spawn_x[i] = float(u.position[0])
        c.spawn_y[i] = float(u.position[1])
        c.spawn_heading[i] = float(np.radians(u.heading_deg))
    for z in range(Z):
        c.zone_ax[z] = 1.0
        c.zone_ay[z] = 1.0
    for z, zn in enumerate(sc.zones):
        c.zone_type[z] = ZONE_IDS[zn.type]
        c.zone_cx[z], c.zone_cy[z] = float(zn.center[0]), float(zn.center[1])
        c.zone_ax[z], c.zone_ay[z] = float(zn.semi_axes[0]), float(zn.semi_axes[1])
        c.zone_effect[z] = float(zn.effect)
    return c
