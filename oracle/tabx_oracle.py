"""CPU oracle for the TABX batched environment step — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference engine's step path
(``/root/reference/pkg/src/skirmish``: ``environment.py:147-519``,
``arrays.py:244-400``, ``physics.py:27-120``, ``combat.py:16-113``,
``perception.py:52-201``, ``heuristics.py:70-243``, ``rng.py:25-48``).  It is
the checker for the CUDA path and the ``cpu_baseline`` / ``--impl reference``
arm of ``bench.py``; nothing in ``paper_2602_01665_b200`` imports it, and the
product path never falls back to it.

Parity pin: ``tests/test_oracle_golden.py`` replays the golden trajectories
in ``tests/golden/`` (written by ``tools/make_golden.py`` from the reference
itself, imported read-only in the build container) and requires bit-identical
float64 state and outputs at every step.

Every array op below is chosen to round exactly like the reference's numpy
expression it cites: no FMA, numpy's pairwise ``add.reduce`` for last-axis
sums, sequential middle-axis sums, first-index argmin/argmax.
"""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

# ----------------------------------------------------------------- consts --
ALLY, ENEMY = 0, 1
A_ROTATE, A_ATTACK, A_NOOP = 4, 5, 6
N_ACTIONS = 7
CTRL_EXTERNAL, CTRL_HEURISTIC, CTRL_RANDOM = 0, 1, 2
CONTROLLER_IDS = {"external": 0, "heuristic": 1, "random": 2}
Z_NONE, Z_LAVA, Z_BUSH, Z_SWAMP = 0, 1, 2, 3
ZONE_IDS = {"lava": 1, "bush": 2, "swamp": 3}
R_NONE, R_ELIM, R_TRUNC, R_TIE = 0, 1, 2, 3
REASON_NAMES = {1: "elimination", 2: "truncation", 3: "truncation_tie"}
STEP_DIRS = np.array([[0.0, 1.0], [0.0, -1.0], [1.0, 0.0], [-1.0, 0.0]])  # core.py:25
ASSASSIN_MIN_SPEED = 1.4  # arrays.py:31
RANGER_MIN_RANGE = 10.0  # arrays.py:32
BUFFER = 0.5  # heuristics.py:42
STANDOFF = 0.8  # heuristics.py:44
HEALTH_NORM = 1000.0  # perception.py:22
TWO_PI = 2.0 * np.pi

U64 = np.uint64
_K_GOLD = U64(0x9E3779B97F4A7C15)
_K_STEP = U64(0xC2B2AE3D27D4EB4F)
_K_LANE = U64(0x165667B19E3779F9)
TAG_EPISODE, TAG_RESEED, TAG_EXPLORE, TAG_PICK, TAG_RANDOM = 1, 2, 3, 4, 5


class OracleActionMaskError(ValueError):
    pass


# --------------------------------------------------------------------- rng --
def _finalize(x):
    x = (x ^ (x >> U64(30))) * U64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> U64(27))) * U64(0x94D049BB133111EB)
    return x ^ (x >> U64(31))


def keyed_hash(seed, step=0, tag=0, lane=0):
    """rng.py:31-37 (wrapping uint64)."""
    with np.errstate(over="ignore"):
        h = _finalize(np.asarray(seed, dtype=U64) + _K_GOLD * U64(int(tag)))
        h = _finalize(h + np.asarray(step, dtype=U64) * _K_STEP)
        return _finalize(h + np.asarray(lane, dtype=U64) * _K_LANE)


def unit_uniform(seed, step, tag, lane):
    """rng.py:40-43."""
    return (keyed_hash(seed, step, tag, lane) >> U64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ------------------------------------------------------------------- state --
_F64_BN = ("u_max_health", "u_radius", "u_mass", "u_inv_mass", "u_speed", "u_damage",
           "u_range", "u_cooldown", "u_sight_angle", "u_sight_cos_half", "u_sight_range",
           "heading", "health", "cooldown", "reveal")
_BOOL_BN = ("u_active", "u_kinematic", "role_assassin", "role_ranger", "role_healer",
            "alive", "mem_valid")
_F64_B = ("dt", "restitution", "slop", "correction", "rot_step", "boundary_coeff",
          "reveal_duration", "field_w", "field_h", "prev_gap", "ep_return")
_BOOL_B = ("enable_noop", "done", "terminated", "truncated")


def blank_state(B: int, N: int, Z: int) -> SimpleNamespace:
    """Zeroed batch state with the reference field names (arrays.py:155-223)."""
    s = SimpleNamespace(batch=B, n_units=N, n_zones=Z)
    for k in _F64_BN:
        setattr(s, k, np.zeros((B, N)))
    for k in _BOOL_BN:
        setattr(s, k, np.zeros((B, N), bool))
    for k in _F64_B:
        setattr(s, k, np.zeros(B))
    for k in _BOOL_B:
        setattr(s, k, np.zeros(B, bool))
    s.seed = np.zeros(B, U64)
    s.episode = np.zeros(B, np.int64)
    s.u_team = np.zeros((B, N), np.int64)
    s.t_controller = np.zeros((B, 2), np.int64)
    s.t_epsilon = np.zeros((B, 2))
    s.t_aggressive = np.zeros((B, 2))
    s.max_steps = np.zeros(B, np.int64)
    s.z_type = np.zeros((B, Z), np.int64)
    s.z_center = np.zeros((B, Z, 2))
    s.z_axes = np.ones((B, Z, 2))
    s.z_effect = np.zeros((B, Z))
    s.t = np.zeros(B, np.int64)
    s.pos = np.zeros((B, N, 2))
    s.vel = np.zeros((B, N, 2))
    s.imp_dv = np.zeros((B, N, 2))
    s.mem_pos = np.zeros((B, N, 2))
    s.winner = np.full(B, -1, np.int64)
    s.reason = np.zeros(B, np.int64)
    s.first_kill = np.full(B, -1, np.int64)
    s.vis = np.zeros((B, N, N), bool)
    s.atk = np.zeros((B, N, N), bool)
    return s


def copy_state(s: SimpleNamespace) -> SimpleNamespace:
    return SimpleNamespace(**{k: (v.copy() if isinstance(v, np.ndarray) else v)
                              for k, v in vars(s).items()})


def respawn(s: SimpleNamespace, b: int, sc) -> None:
    """Write lane b's static columns and spawn state (arrays.py:244-321)."""
    s.u_active[b] = False
    s.alive[b] = False
    s.z_type[b] = Z_NONE
    for i, u in enumerate(sc.units):
        sp = u.resolved_spec()
        s.u_active[b, i] = True
        s.u_team[b, i] = u.team
        s.u_max_health[b, i] = sp.max_health
        s.u_radius[b, i] = sp.body_radius
        s.u_mass[b, i] = sp.body_mass
        s.u_inv_mass[b, i] = 0.0 if sp.kinematic else 1.0 / sp.body_mass
        s.u_speed[b, i] = sp.speed
        s.u_damage[b, i] = sp.attack_damage
        s.u_range[b, i] = sp.attack_range
        s.u_cooldown[b, i] = sp.attack_cooldown
        s.u_sight_angle[b, i] = sp.sight_angle
        s.u_sight_cos_half[b, i] = np.cos(sp.sight_angle / 2.0)
        s.u_sight_range[b, i] = sp.sight_range
        s.u_kinematic[b, i] = sp.kinematic
        s.role_assassin[b, i] = sp.speed >= ASSASSIN_MIN_SPEED
        s.role_ranger[b, i] = sp.attack_range >= RANGER_MIN_RANGE and sp.attack_damage > 0
        s.role_healer[b, i] = sp.attack_damage < 0
        s.pos[b, i] = u.position
        s.heading[b, i] = np.radians(u.heading_deg)
        s.health[b, i] = sp.max_health
        s.alive[b, i] = True
    pad = ~s.u_active[b]
    s.u_max_health[b, pad] = 1.0
    s.u_radius[b, pad] = 0.0
    s.u_mass[b, pad] = 1.0
    s.u_inv_mass[b, pad] = 1.0
    s.u_sight_cos_half[b, pad] = 1.0
    for tm in sc.teams:
        s.t_controller[b, tm.id] = CONTROLLER_IDS[tm.controller]
        s.t_epsilon[b, tm.id] = tm.epsilon if tm.has_heuristic else 0.0
        s.t_aggressive[b, tm.id] = tm.aggressive_threshold if tm.has_heuristic else 0.0
    ph = sc.physics
    s.dt[b] = ph.dt
    s.restitution[b] = ph.restitution
    s.slop[b] = ph.penetration_slop
    s.correction[b] = ph.correction_percent
    s.rot_step[b] = np.radians(ph.rotation_step_deg)
    s.boundary_coeff[b] = ph.boundary_damage_coeff
    s.reveal_duration[b] = ph.reveal_duration
    s.enable_noop[b] = ph.enable_noop
    s.max_steps[b] = sc.max_steps
    s.field_w[b] = sc.field.width
    s.field_h[b] = sc.field.height
    for z, zn in enumerate(sc.zones):
        s.z_type[b, z] = ZONE_IDS[zn.type]
        s.z_center[b, z] = zn.center
        s.z_axes[b, z] = zn.semi_axes
        s.z_effect[b, z] = zn.effect
    s.t[b] = 0
    for k in ("vel", "imp_dv", "cooldown", "reveal", "mem_pos"):
        getattr(s, k)[b] = 0.0
    s.prev_gap[b] = 0.0
    s.ep_return[b] = 0.0
    for k in ("done", "terminated", "truncated", "mem_valid", "vis", "atk"):
        getattr(s, k)[b] = False
    s.winner[b] = -1
    s.reason[b] = R_NONE
    s.first_kill[b] = -1


def build_state(scenarios, seeds) -> SimpleNamespace:
    B = len(scenarios)
    N, Z = scenarios[0].max_units, scenarios[0].max_zones
    s = blank_state(B, N, Z)
    s.seed = np.asarray(seeds, dtype=U64).reshape(B).copy()
    for b, sc in enumerate(scenarios):
        respawn(s, b, sc)
    return s


# ------------------------------------------------------------ array kernels --
def inside_zones(s):
    """[B,N,Z] ellipse membership (arrays.py:329-335)."""
    rel = s.pos[:, :, None, :] - s.z_center[:, None, :, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        q = rel / s.z_axes[:, None, :, :]
    return ((q[..., 0] ** 2 + q[..., 1] ** 2) <= 1.0) & (s.z_type[:, None, :] != Z_NONE)


def swamp_speed(s):
    """Speed after swamp multipliers, sequential product over z (arrays.py:338-343)."""
    hit = inside_zones(s) & (s.z_type == Z_SWAMP)[:, None, :]
    return s.u_speed * np.where(hit, s.z_effect[:, None, :], 1.0).prod(axis=2)


def all_dists(pos):
    """[B,N,N] with d = p_j - p_i (arrays.py:346-349)."""
    d = pos[:, None, :, :] - pos[:, :, None, :]
    return np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)


def legal_actions(alive, active, cooldown, enable_noop):
    """[B,N,7] mask (arrays.py:373-387)."""
    ok = alive & active
    m = np.zeros(ok.shape + (N_ACTIONS,), bool)
    m[..., 0:5] = ok[..., None]
    m[..., 5] = ok & (cooldown <= 0.0)
    m[..., 6] = (ok & enable_noop[:, None]) | ~ok
    return m


def team_ratio(s, team):
    """Masked mean health ratio, numpy pairwise sum (arrays.py:390-395)."""
    member = s.u_active & (s.u_team == team)
    r = np.where(member, s.health / s.u_max_health, 0.0)
    return r.sum(axis=1) / np.maximum(member.sum(axis=1), 1)


def ratio_gap(s):
    return team_ratio(s, ALLY) - team_ratio(s, ENEMY)


def sees(s):
    """Visibility = FoV wedge minus bush concealment (perception.py:52-96)."""
    d = s.pos[:, None, :, :] - s.pos[:, :, None, :]
    dist = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)
    along = d[..., 0] * np.cos(s.heading)[:, :, None] + d[..., 1] * np.sin(s.heading)[:, :, None]
    with np.errstate(invalid="ignore", divide="ignore"):
        cdev = np.where(dist > 0.0, along / dist, 1.0)
    wedge = (dist <= s.u_sight_range[:, :, None]) & (cdev >= s.u_sight_cos_half[:, :, None])
    bz = inside_zones(s) & (s.z_type == Z_BUSH)[:, None, :]
    in_bush = bz.any(axis=2)
    shared = (bz[:, :, None, :] & bz[:, None, :, :]).any(axis=3)
    foe = s.u_team[:, :, None] != s.u_team[:, None, :]
    hidden = in_bush[:, None, :] & foe & ~shared & (s.reveal[:, None, :] <= 0.0)
    pair_active = s.u_active[:, :, None] & s.u_active[:, None, :]
    return wedge & ~hidden & pair_active


def strike_box(pos, heading, radius, reach, cos_half):
    """Forward strike rectangle ∩ view wedge, diagonal off (combat.py:16-50)."""
    d = pos[:, None, :, :] - pos[:, :, None, :]
    c, sn = np.cos(heading)[:, :, None], np.sin(heading)[:, :, None]
    lx = d[..., 0] * c + d[..., 1] * sn
    ly = -d[..., 0] * sn + d[..., 1] * c
    cx = np.clip(lx, 0.0, reach[:, :, None])
    hw = radius[:, :, None]
    cy = np.clip(ly, -hw, hw)
    box = (lx - cx) ** 2 + (ly - cy) ** 2 <= radius[:, None, :] ** 2
    dist = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)
    with np.errstate(invalid="ignore", divide="ignore"):
        cdev = np.where(dist > 0.0, lx / dist, 1.0)
    out = box & (cdev >= cos_half[:, :, None])
    n = pos.shape[1]
    out[:, np.arange(n), np.arange(n)] = False
    return out


def can_strike(hurt, vis, damage, team, alive, active):
    """combat.py:53-72."""
    same = team[:, :, None] == team[:, None, :]
    role = np.where(damage[:, :, None] > 0.0, ~same, (damage[:, :, None] < 0.0) & same)
    live = alive & active
    return hurt & vis & role & live[:, :, None] & live[:, None, :]


def fresh_caches(s):
    """refresh_caches (environment.py:147-151)."""
    s.vis = sees(s)
    hurt = strike_box(s.pos, s.heading, s.u_radius, s.u_range, s.u_sight_cos_half)
    s.atk = can_strike(hurt, s.vis, s.u_damage, s.u_team, s.alive, s.u_active)


def first_min(values, allowed):
    filled = np.where(allowed, values, np.inf)
    return np.argmin(filled, axis=2), allowed.any(axis=2)


def _best_step(pos, goal, step, far):
    cand = pos[:, :, None, :] + STEP_DIRS[None, None] * step[:, :, None, None]
    sq = ((cand - goal[:, :, None, :]) ** 2).sum(axis=-1)
    return np.argmax(sq, axis=2) if far else np.argmin(sq, axis=2)


def _rotated_hit(s, tp, tr):
    """heuristics.py:87-100 (heading + rot_step, not wrapped)."""
    hd = s.heading + s.rot_step[:, None]
    d = tp - s.pos
    c, sn = np.cos(hd), np.sin(hd)
    lx = d[..., 0] * c + d[..., 1] * sn
    ly = -d[..., 0] * sn + d[..., 1] * c
    cx = np.clip(lx, 0.0, s.u_range)
    cy = np.clip(ly, -s.u_radius, s.u_radius)
    box = (lx - cx) ** 2 + (ly - cy) ** 2 <= tr ** 2
    dist = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)
    with np.errstate(invalid="ignore", divide="ignore"):
        cdev = np.where(dist > 0.0, lx / dist, 1.0)
    return box & (cdev >= s.u_sight_cos_half)


def _kth_legal(mask, u):
    """Index of the floor(u*n_valid)-th legal action (environment.py:198-201)."""
    n_ok = mask.sum(axis=-1)
    k = np.minimum((u * n_ok).astype(np.int64), n_ok - 1)
    return np.argmax(np.cumsum(mask, axis=-1) > k[..., None], axis=-1)


def scripted_policy(s, vis, atk, dist, mask, u_explore, u_pick):
    """Role targets + 7-level cascade + epsilon (heuristics.py:103-243)."""
    B, N = s.pos.shape[:2]
    ok = s.alive & s.u_active
    eps = np.take_along_axis(s.t_epsilon, s.u_team, axis=1)
    xi = np.take_along_axis(s.t_aggressive, s.u_team, axis=1)
    step = swamp_speed(s) * s.dt[:, None]

    cand = vis & ok[:, None, :] & ~np.eye(N, dtype=bool)[None]
    foe = s.u_team[:, :, None] != s.u_team[:, None, :]
    friends = cand & ~foe
    hurt_f = friends & (s.health < s.u_max_health)[:, None, :]
    heal_pool = np.where(hurt_f.any(axis=2)[..., None], hurt_f, friends)
    t_heal, h_heal = first_min(dist, heal_pool)
    foes = cand & foe
    mh = np.broadcast_to(s.u_max_health[:, None, :], (B, N, N))
    weakest = np.where(foes, mh, np.inf).min(axis=2)
    t_weak, h_weak = first_min(dist, foes & (mh == weakest[..., None]))
    t_near, h_near = first_min(dist, foes)
    tgt = np.where(s.role_healer, t_heal, np.where(s.role_assassin, t_weak, t_near))
    has = np.where(s.role_healer, h_heal, np.where(s.role_assassin, h_weak, h_near)) & ok
    h_near = h_near & ok

    tp = np.take_along_axis(s.pos, tgt[..., None], axis=1)
    tr = np.take_along_axis(s.u_radius, tgt, axis=1)
    th = np.take_along_axis(s.heading, tgt, axis=1)
    atk_t = np.take_along_axis(atk, tgt[:, :, None], axis=2)[..., 0]

    act = np.full((B, N), A_NOOP, np.int64)
    fixed = ~ok

    def take(cond, value):
        nonlocal act, fixed
        cond = ~fixed & cond
        act = np.where(cond, value, act)
        fixed = fixed | cond

    take(has & atk_t & (s.cooldown <= 0.0), A_ATTACK)
    take(has & _rotated_hit(s, tp, tr), A_ROTATE)
    npos = np.take_along_axis(s.pos, t_near[..., None], axis=1)
    ndist = np.take_along_axis(dist, t_near[:, :, None], axis=2)[..., 0]
    take(s.role_ranger & h_near & (ndist < xi * s.u_range), _best_step(s.pos, npos, step, True))
    tvec = np.stack([np.cos(th), np.sin(th)], axis=-1)
    touch = s.u_radius + tr + BUFFER
    standoff = np.maximum(STANDOFF * s.u_range, touch)
    goal = np.where(s.role_healer[..., None], tp,
                    np.where(s.role_assassin[..., None], tp - tvec * touch[..., None],
                             tp + tvec * standoff[..., None]))
    take(has, _best_step(s.pos, goal, step, False))
    gap = np.sqrt(((s.pos - s.mem_pos) ** 2).sum(axis=-1))
    mem_ok = s.mem_valid & (gap > s.u_radius)
    take(mem_ok, _best_step(s.pos, s.mem_pos, step, False))
    if s.n_zones > 0:
        bush = s.z_type == Z_BUSH
        in_bush = (inside_zones(s) & bush[:, None, :]).any(axis=2)
        cd = np.sqrt(((s.z_center[:, None, :, :] - s.pos[:, :, None, :]) ** 2).sum(axis=-1))
        cd = np.where(bush[:, None, :], cd, np.inf)
        nb = np.argmin(cd, axis=2)
        bc = np.take_along_axis(s.z_center, np.maximum(nb, 0)[..., None], axis=1)
        take(s.role_ranger & bush.any(axis=1)[:, None] & ~in_bush,
             _best_step(s.pos, bc, step, False))
    act = np.where(~fixed, A_ROTATE, act)
    act = np.where(ok & (u_explore < eps), _kth_legal(mask, u_pick), act)
    return act, np.where(has[..., None], tp, s.mem_pos), has | mem_ok


def choose_actions(s, external, mask):
    """environment.py:154-204."""
    B, N = s.alive.shape
    live = ~s.done
    ctrl = np.take_along_axis(s.t_controller, s.u_team, axis=1)
    free = s.alive & s.u_active & live[:, None]
    if external is None:
        act = np.full((B, N), A_NOOP, np.int64)
    else:
        act = np.asarray(external, dtype=np.int64).reshape(B, N).copy()
        chk = free & (ctrl == CTRL_EXTERNAL)
        if chk.any():
            oob = (act < 0) | (act >= N_ACTIONS)
            legal = np.take_along_axis(mask, np.clip(act, 0, N_ACTIONS - 1)[..., None], axis=2)[..., 0]
            bad = chk & (oob | ~legal)
            if bad.any():
                b, i = np.argwhere(bad)[0]
                raise OracleActionMaskError(f"invalid action {act[b, i]} for unit {i} in env {b}")
    lanes = np.arange(N)[None, :]
    heur = (ctrl == CTRL_HEURISTIC) & free
    if heur.any():
        ue = unit_uniform(s.seed[:, None], s.t[:, None], TAG_EXPLORE, lanes)
        up = unit_uniform(s.seed[:, None], s.t[:, None], TAG_PICK, lanes)
        h_act, mp, mv = scripted_policy(s, s.vis, s.atk, all_dists(s.pos), mask, ue, up)
        act = np.where(heur, h_act, act)
        s.mem_pos = np.where(heur[..., None], mp, s.mem_pos)
        s.mem_valid = np.where(heur, mv, s.mem_valid)
    rnd = (ctrl == CTRL_RANDOM) & free
    if rnd.any():
        u = unit_uniform(s.seed[:, None], s.t[:, None], TAG_RANDOM, lanes)
        act = np.where(rnd, _kth_legal(mask, u), act)
    return np.where(free, act, A_NOOP)


_PAIRS: dict[int, tuple[np.ndarray, np.ndarray]] = {}


def _pairs(n):
    if n not in _PAIRS:
        _PAIRS[n] = np.triu_indices(n, k=1)
    return _PAIRS[n]


def overlaps(pos, radius, active):
    """physics.py:27-49."""
    iu, ju = _pairs(pos.shape[1])
    d = pos[:, ju, :] - pos[:, iu, :]
    dist = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)
    rs = radius[:, iu] + radius[:, ju]
    same = dist == 0.0
    depth = np.where(same, rs, rs - dist)
    nrm = np.where(same[..., None], np.array([1.0, 0.0]), d / np.where(same, 1.0, dist)[..., None])
    return (depth > 0.0) & active[:, iu] & active[:, ju], nrm, depth


def settle(vel, pos, inv_m, touching, nrm, depth, e, slop, beta):
    """Sequential impulses in ascending pair order (physics.py:52-94)."""
    iu, ju = _pairs(pos.shape[1])
    vel = vel.copy()
    shift = np.zeros_like(pos)
    for p in np.nonzero(touching.any(axis=0))[0]:
        i, j = int(iu[p]), int(ju[p])
        wi, wj = inv_m[:, i], inv_m[:, j]
        w = wi + wj
        on = touching[:, p] & (w > 0.0)
        if not on.any():
            continue
        ws = np.where(w > 0.0, w, 1.0)
        n = nrm[:, p]
        rel = ((vel[:, j] - vel[:, i]) * n).sum(axis=-1)
        jm = np.where(on & (rel <= 0.0), -(1.0 + e) * rel / ws, 0.0)
        vel[:, i] -= (jm * wi)[:, None] * n
        vel[:, j] += (jm * wj)[:, None] * n
        c = np.where(on, beta * np.maximum(depth[:, p] - slop, 0.0) / ws, 0.0)
        shift[:, i] -= (c * wi)[:, None] * n
        shift[:, j] += (c * wj)[:, None] * n
    return vel, pos + shift


def fence(pos, health, alive, active, kinematic, max_h, fw, fh, coeff, dt):
    """physics.py:97-120."""
    w, h = fw[:, None], fh[:, None]
    x, y = pos[..., 0], pos[..., 1]
    outside = (x < 0.0) | (x > w) | (y < 0.0) | (y > h)
    pen = coeff[:, None] * max_h * dt[:, None]
    health = np.where(outside & alive & active, np.maximum(health - pen, 0.0), health)
    clipped = np.stack([np.clip(x, 0.0, w), np.clip(y, 0.0, h)], axis=-1)
    return np.where((active & ~kinematic)[..., None], clipped, pos), health


def strike(atk, dist, act, alive, active, cooldown, damage, health, max_h, cd_spec):
    """combat.py:75-113."""
    swing = (act == A_ATTACK) & alive & active & (cooldown <= 0.0)
    tgt = np.argmin(np.where(atk, dist, np.inf), axis=2)
    tgt = np.where(atk.any(axis=2), tgt, -1)
    landed = swing & (tgt >= 0)
    n = atk.shape[2]
    inter = landed[:, :, None] & (tgt[:, :, None] == np.arange(n))
    delta = (inter * damage[:, :, None]).sum(axis=1)
    health = np.where(active & alive, np.clip(health - delta, 0.0, max_h), health)
    return health, np.where(swing, cd_spec, cooldown), inter


def observe(s, vis, atk):
    """Per-agent observations + global state (perception.py:99-201), float64."""
    B, N, Z = s.batch, s.n_units, s.n_zones
    with np.errstate(divide="ignore", invalid="ignore"):
        cdr = np.where(s.u_cooldown > 0.0, s.cooldown / s.u_cooldown, 0.0)
    own = np.stack([s.health / s.u_max_health, s.u_max_health / HEALTH_NORM,
                    s.pos[..., 0] / s.field_w[:, None], s.pos[..., 1] / s.field_h[:, None],
                    np.cos(s.heading), np.sin(s.heading), s.u_range, s.u_damage, s.cooldown,
                    cdr, s.u_radius, s.u_mass, s.u_sight_angle, s.alive.astype(np.float64),
                    s.u_speed], axis=-1)
    own = np.where(s.u_active[..., None], own, 0.0)
    scale = np.stack([s.field_w, s.field_h], axis=-1)
    rel = (s.pos[:, None, :, :] - s.pos[:, :, None, :]) / scale[:, None, None, :]
    pair = np.empty((B, N, N, 17))
    pair[..., :15] = own[:, None, :, :]
    pair[..., 2:4] = rel
    pair[..., 15] = s.u_team[:, None, :].astype(np.float64)
    pair[..., 16] = atk.astype(np.float64)
    pair = np.where((vis & s.u_active[:, None, :])[..., None], pair, 0.0)
    if N > 1:
        cols = np.array([[j for j in range(N) if j != i] for i in range(N)], dtype=np.int64)
        others = pair[:, np.arange(N)[:, None], cols].reshape(B, N, (N - 1) * 17)
    else:
        others = np.zeros((B, N, 0))
    used = s.z_type != 0
    hot = np.stack([s.z_type == k for k in (1, 2, 3)], axis=-1).astype(np.float64)
    zr = (s.z_center[:, None, :, :] - s.pos[:, :, None, :]) / scale[:, None, None, :]
    zblk = np.concatenate([np.broadcast_to(hot[:, None], (B, N, Z, 3)), zr,
                           np.broadcast_to(s.z_axes[:, None], (B, N, Z, 2)),
                           np.broadcast_to(s.z_effect[:, None, :, None], (B, N, Z, 1))], axis=-1)
    zblk = np.where(used[:, None, :, None], zblk, 0.0).reshape(B, N, Z * 8)
    obs = np.concatenate([own, others, zblk], axis=-1)
    obs = np.where(s.u_active[..., None], obs, 0.0)
    gz = np.concatenate([hot, s.z_center / scale[:, None, :], s.z_axes, s.z_effect[..., None]],
                        axis=-1)
    gz = np.where(used[..., None], gz, 0.0)
    glob = np.concatenate([own.reshape(B, N * 15), gz.reshape(B, Z * 8)], axis=-1)
    return obs, glob


def _result(s, obs, glob, rewards, mask, dense, actions, inter):
    return dict(observations=obs, global_state=glob, rewards=rewards, action_mask=mask,
                terminated=s.terminated.copy(), truncated=s.truncated.copy(),
                done=s.done.copy(), dense_reward=dense, actions=actions, interactions=inter,
                winner=s.winner.copy(), reason=s.reason.copy(),
                first_kill=s.first_kill.copy(), episode_return=s.ep_return.copy(),
                episode_length=s.t.copy(), final_observations=None, final_global_state=None)


def advance(s, external):
    """One batched step in place (environment.py:207-348)."""
    B, N = s.alive.shape
    live = ~s.done
    mask = legal_actions(s.alive, s.u_active, s.cooldown, s.enable_noop)
    act = choose_actions(s, external, mask)

    moving = (act < 4) & s.alive & s.u_active & ~s.u_kinematic
    v_cmd = STEP_DIRS[np.clip(act, 0, 3)] * np.where(moving, swamp_speed(s), 0.0)[..., None]
    v_used = v_cmd + s.imp_dv
    mov = (s.u_active & ~s.u_kinematic & live[:, None])[..., None]
    s.pos = np.where(mov, s.pos + v_used * s.dt[:, None, None], s.pos)
    tick = (s.u_active & live[:, None]).astype(np.float64) * s.dt[:, None]
    s.cooldown = np.maximum(s.cooldown - tick, 0.0)
    s.reveal = np.maximum(s.reveal - tick, 0.0)

    touch, nrm, depth = overlaps(s.pos, s.u_radius, s.u_active)
    touch &= live[:, None]
    v_fin, s.pos = settle(v_used, s.pos, s.u_inv_mass, touch, nrm, depth,
                          s.restitution, s.slop, s.correction)
    s.imp_dv = np.where(live[:, None, None], v_fin - v_used, s.imp_dv)
    s.vel = np.where(live[:, None, None], v_fin, s.vel)

    bpos, bh = fence(s.pos, s.health, s.alive, s.u_active, s.u_kinematic, s.u_max_health,
                     s.field_w, s.field_h, s.boundary_coeff, s.dt)
    s.pos = np.where(live[:, None, None], bpos, s.pos)
    s.health = np.where(live[:, None], bh, s.health)

    turn = (act == A_ROTATE) & s.alive & s.u_active & live[:, None]
    s.heading = np.where(turn, (s.heading + s.rot_step[:, None]) % TWO_PI, s.heading)

    s.vis = sees(s)
    hurt = strike_box(s.pos, s.heading, s.u_radius, s.u_range, s.u_sight_cos_half)
    s.atk = can_strike(hurt, s.vis, s.u_damage, s.u_team, s.alive, s.u_active)
    dist = all_dists(s.pos)
    nh, ncd, inter = strike(s.atk, dist, act, s.alive, s.u_active, s.cooldown, s.u_damage,
                            s.health, s.u_max_health, s.u_cooldown)
    s.health = np.where(live[:, None], nh, s.health)
    s.cooldown = np.where(live[:, None], ncd, s.cooldown)
    inter &= live[:, None, None]
    s.reveal = np.where(inter.any(axis=2) | inter.any(axis=1), s.reveal_duration[:, None], s.reveal)

    lava = inside_zones(s) & (s.z_type == Z_LAVA)[:, None, :]
    burn = np.where(lava, s.z_effect[:, None, :], 0.0).sum(axis=2) * s.dt[:, None]
    burnable = s.alive & s.u_active & live[:, None]
    s.health = np.where(burnable, np.clip(s.health - burn, 0.0, s.u_max_health), s.health)

    still = s.alive & (s.health > 0.0)
    died = s.alive & ~still
    s.alive = still
    first = died.any(axis=1) & (s.first_kill < 0)
    s.first_kill = np.where(first, np.where((died & (s.u_team == ALLY)).any(axis=1), ENEMY, ALLY),
                            s.first_kill)

    gap = ratio_gap(s)
    dense = np.where(live, gap - s.prev_gap, 0.0)
    s.prev_gap = np.where(live, gap, s.prev_gap)
    s.t = s.t + live.astype(np.int64)
    na = (s.alive & s.u_active & (s.u_team == ALLY)).sum(axis=1)
    ne = (s.alive & s.u_active & (s.u_team == ENEMY)).sum(axis=1)
    elim = live & ((na == 0) | (ne == 0))
    trunc = live & ~elim & (s.t >= s.max_steps)
    ra, re = team_ratio(s, ALLY), team_ratio(s, ENEMY)
    win = np.where(elim, np.where((ne == 0) & (na > 0), ALLY, ENEMY),
                   np.where(trunc, np.where(ra > re, ALLY, ENEMY), -1))
    why = np.where(elim, R_ELIM, np.where(trunc, np.where(ra == re, R_TIE, R_TRUNC), R_NONE))
    fin = elim | trunc
    r_ally = dense + np.where(fin, np.where(win == ALLY, 1.0, -1.0), 0.0)
    s.ep_return = s.ep_return + np.where(live, r_ally, 0.0)
    s.terminated |= elim
    s.truncated |= trunc
    s.done |= fin
    s.winner = np.where(fin, win, s.winner)
    s.reason = np.where(fin, why, s.reason)
    rewards = (np.where(s.u_team == ALLY, 1.0, -1.0) * s.u_active) * np.where(live, r_ally, 0.0)[:, None]
    obs, glob = observe(s, s.vis, s.atk)
    out_mask = legal_actions(s.alive, s.u_active, s.cooldown, s.enable_noop)
    return _result(s, obs, glob, rewards, out_mask, dense, act, inter)


def initial_output(s):
    """init_output (environment.py:351-374)."""
    fresh_caches(s)
    s.prev_gap = ratio_gap(s)
    B, N = s.alive.shape
    obs, glob = observe(s, s.vis, s.atk)
    mask = legal_actions(s.alive, s.u_active, s.cooldown, s.enable_noop)
    return _result(s, obs, glob, np.zeros((B, N)), mask, np.zeros(B),
                   np.full((B, N), A_NOOP, np.int64), np.zeros((B, N, N), bool))


class OracleBatchSim:
    """BatchSim restated (environment.py:463-519).

    ``refresh`` in :meth:`step` overrides the batch-wide cache refresh that
    follows an auto-reset (``environment.py:508``): ``None`` keeps the
    reference rule (refresh iff any lane reset), ``True``/``False`` force it.
    Used to replay a GPU shard's refresh decisions on a lane subset.
    """

    def __init__(self, scenarios, seeds, auto_reset=False):
        self.scenarios = list(scenarios)
        self.auto_reset = auto_reset
        self.sim = build_state(self.scenarios, seeds)
        self.last = initial_output(self.sim)

    @property
    def batch(self):
        return self.sim.batch

    def reset_env(self, b, scenario=None, seed=None):
        if scenario is not None:
            self.scenarios[b] = scenario
        if seed is not None:
            self.sim.seed[b] = U64(seed)
        respawn(self.sim, b, self.scenarios[b])
        self.last = initial_output(self.sim)

    def step(self, actions=None, refresh=None):
        out = advance(self.sim, actions)
        s = self.sim
        if self.auto_reset and out["done"].any():
            for b in np.nonzero(out["done"])[0]:
                s.episode[b] += 1
                s.seed[b] = keyed_hash(s.seed[b], int(s.episode[b]), TAG_RESEED)
                respawn(s, b, self.scenarios[b])
            if refresh is None or refresh:
                fresh_caches(s)
            else:
                sel = out["done"]
                tmp = copy_state(s)
                fresh_caches(tmp)
                s.vis = np.where(sel[:, None, None], tmp.vis, s.vis)
                s.atk = np.where(sel[:, None, None], tmp.atk, s.atk)
            s.prev_gap = np.where(out["done"], ratio_gap(s), s.prev_gap)
            obs, glob = observe(s, s.vis, s.atk)
            mask = legal_actions(s.alive, s.u_active, s.cooldown, s.enable_noop)
            sel = out["done"]
            out["final_observations"] = out["observations"]
            out["final_global_state"] = out["global_state"]
            out["observations"] = np.where(sel[:, None, None], obs, out["observations"])
            out["global_state"] = np.where(sel[:, None], glob, out["global_state"])
            out["action_mask"] = np.where(sel[:, None, None], mask, out["action_mask"])
        elif refresh:
            fresh_caches(s)
        self.last = out
        return out


def summarize_lanes(lengths, returns, winners, first_kills):
    """Episode summary fields of ``rollout.summarize`` (rollout.py:122-147)."""
    n = len(lengths)
    if n == 0:
        return dict(episodes=0, win_rate=0.0, mean_return=0.0, mean_length=0.0,
                    first_kill_rate=0.0)
    tot = 0.0
    for r in returns:
        tot += float(r)
    return dict(episodes=n, win_rate=sum(1 for w in winners if w == ALLY) / n,
                mean_return=tot / n, mean_length=sum(int(x) for x in lengths) / n,
                first_kill_rate=sum(1 for f in first_kills if f == ALLY) / n)


def fov_verdict(observer_xy, heading_rad, sight_angle, sight_range, target_xy):
    """Scalar in_fov with hypot (perception.py:246-255), for the FoV fixtures."""
    dx = target_xy[0] - observer_xy[0]
    dy = target_xy[1] - observer_xy[1]
    dist = math.hypot(dx, dy)
    if dist > sight_range:
        return False
    if dist == 0.0:
        return True
    cdev = (dx * math.cos(heading_rad) + dy * math.sin(heading_rad)) / dist
    return cdev >= math.cos(sight_angle / 2.0)
