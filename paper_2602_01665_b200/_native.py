"""ctypes binding of the C ABI in include/tabx.h (the in-tree ``_tabx.so``).

There is no fallback: if the shared object is missing or was built against a
different ABI, importing the package's simulator raises ``ImportError``.
"""
from __future__ import annotations

import ctypes as ct
import os

MAX_UNITS = 256
MAX_ZONES = 32
NUM_ACTIONS = 7
NUM_STATS = 8
ABI_VERSION = 6

OK = 0
E_ARGUMENT, E_CUDA, E_ACTION_MASK, E_SHAPE, E_ALIGNMENT, E_CAPACITY = 1, 2, 3, 4, 5, 6

LIB_NAME = "_tabx.so"
LIB_PATH = os.environ.get("TABX_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                      LIB_NAME)

_d = ct.c_double
_u8 = ct.c_uint8
_i32 = ct.c_int32
_i64 = ct.c_int64


class TabxConfig(ct.Structure):
    _fields_ = [
        ("n_units", _i32), ("n_zones", _i32), ("max_steps", _i32), ("enable_noop", _i32),
        ("controller", _i32 * 2), ("epsilon", _d * 2), ("aggressive", _d * 2),
        ("dt", _d), ("restitution", _d), ("slop", _d), ("correction", _d), ("rot_step", _d),
        ("boundary_coeff", _d), ("reveal_duration", _d), ("field_w", _d), ("field_h", _d),
        ("active", _u8 * MAX_UNITS), ("team", _u8 * MAX_UNITS), ("kinematic", _u8 * MAX_UNITS),
        ("role_assassin", _u8 * MAX_UNITS), ("role_ranger", _u8 * MAX_UNITS),
        ("role_healer", _u8 * MAX_UNITS),
        ("max_health", _d * MAX_UNITS), ("radius", _d * MAX_UNITS), ("mass", _d * MAX_UNITS),
        ("inv_mass", _d * MAX_UNITS), ("speed", _d * MAX_UNITS), ("damage", _d * MAX_UNITS),
        ("attack_range", _d * MAX_UNITS), ("cooldown", _d * MAX_UNITS),
        ("sight_angle", _d * MAX_UNITS), ("sight_cos_half", _d * MAX_UNITS),
        ("sight_range", _d * MAX_UNITS), ("spawn_x", _d * MAX_UNITS), ("spawn_y", _d * MAX_UNITS),
        ("spawn_heading", _d * MAX_UNITS),
        ("zone_type", _i32 * MAX_ZONES), ("zone_cx", _d * MAX_ZONES), ("zone_cy", _d * MAX_ZONES),
        ("zone_ax", _d * MAX_ZONES), ("zone_ay", _d * MAX_ZONES), ("zone_effect", _d * MAX_ZONES),
    ]


OUTPUT_FIELDS = ("observations", "global_state", "rewards", "action_mask", "terminated",
                 "truncated", "done", "dense_reward", "actions", "interactions", "winner",
                 "reason", "first_kill", "episode_return", "episode_length",
                 "final_observations", "final_global_state", "reset_mask")


class TabxOutputs(ct.Structure):
    # + the optional bfloat16 policy feed (tabx.h)
    _fields_ = [(name, ct.c_void_p) for name in OUTPUT_FIELDS] + [
        ("observations_bf16", ct.c_void_p), ("observations_bf16_ld", ct.c_int64)]


STATE_FIELDS = ("seed", "episode", "t", "pos", "heading", "vel", "imp_dv", "health", "cooldown",
                "reveal", "alive", "prev_gap", "ep_return", "done", "terminated", "truncated",
                "winner", "reason", "first_kill", "mem_pos", "mem_valid", "vis", "atk", "config")


class TabxState(ct.Structure):
    _fields_ = [(name, ct.c_void_p) for name in STATE_FIELDS]


class TabxPcg64(ct.Structure):
    """numpy PCG64 bit-generator state (tabx.h)."""
    _fields_ = [("state_hi", ct.c_uint64), ("state_lo", ct.c_uint64), ("inc_hi", ct.c_uint64),
                ("inc_lo", ct.c_uint64), ("has_uint32", ct.c_uint32), ("uinteger", ct.c_uint32)]


class TabxLevelSpec(ct.Structure):
    _fields_ = [
        ("open_units", _i32), ("open_zones", _i32), ("open_heuristic", _i32),
        ("unit_open", _i32 * 3), ("unit_lo", _d * 3), ("unit_hi", _d * 3),
        ("n_zone_types", _i32), ("zone_types", _i32 * 3),
        ("box_x0", _d), ("box_x1", _d), ("box_y0", _d), ("box_y1", _d),
        ("axis_open", _i32), ("axis_lo", _d), ("axis_hi", _d),
        ("effect_open", _i32 * 4), ("effect_lo", _d * 4), ("effect_hi", _d * 4),
        ("eps_open", _i32), ("eps_lo", _d), ("eps_hi", _d),
        ("agg_open", _i32), ("agg_lo", _d), ("agg_hi", _d),
    ]


LEVEL_SAMPLE, LEVEL_PERTURB, LEVEL_SWAP_AXES, LEVEL_RETYPE = 0, 1, 2, 3


class TabxError(ct.Structure):
    _fields_ = [("code", _i32), ("unit", _i32), ("env", _i64), ("action", _i64)]


_LIB = None


def lib() -> ct.CDLL:
    """Load ``_tabx.so`` once; raise ImportError if it is absent or stale."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.isfile(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    L = ct.CDLL(LIB_PATH)
    P = ct.c_void_p
    sig = {
        "tabx_abi_version": (_i32, []),
        "tabx_last_error": (ct.c_char_p, []),
        "tabx_obs_dim": (_i32, [_i32, _i32]),
        "tabx_global_dim": (_i32, [_i32, _i32]),
        "tabx_create": (_i32, [ct.POINTER(TabxConfig), _i32, P, P, _i64, _i32, _i32, P,
                               ct.POINTER(P)]),
        "tabx_destroy": (_i32, [P]),
        "tabx_set_stream": (_i32, [P, P]),
        "tabx_dims": (_i32, [P, P, P, P, P, P]),
        "tabx_init_output": (_i32, [P, ct.POINTER(TabxOutputs)]),
        "tabx_step": (_i32, [P, P, ct.POINTER(TabxOutputs)]),
        "tabx_reset_env": (_i32, [P, _i64, ct.POINTER(TabxConfig), ct.c_uint64, _i32,
                                  ct.POINTER(TabxOutputs), P]),
        "tabx_respawn_all": (_i32, [P, P, P]),
        "tabx_export_state": (_i32, [P, ct.POINTER(TabxState)]),
        "tabx_export_lanes": (_i32, [P, P, ct.c_int64, ct.POINTER(TabxState)]),
        "tabx_import_state": (_i32, [P, ct.POINTER(TabxState)]),
        "tabx_get_error": (_i32, [P, ct.POINTER(TabxError), _i32]),
        "tabx_copy_error_word": (_i32, [P, P]),
        "tabx_episode_stats": (_i32, [P, P, P, _i32]),
        "tabx_struct_sizes": (_i32, [P, P, P, P, P]),
        "tabx_reserve_configs": (_i32, [P, _i32]),
        "tabx_num_configs": (_i32, [P, P, P]),
        "tabx_get_config": (_i32, [P, _i32, ct.POINTER(TabxConfig)]),
        "tabx_config_slot": (_i32, [P, _i32, P, P]),
        "tabx_levels": (_i32, [P, _i32, ct.POINTER(TabxLevelSpec), _d, P, _i32, _i32, P]),
        "tabx_respawn_lanes": (_i32, [P, P, P, P, _i64]),
        "tabx_set_profiling": (_i32, [P, _i32]),
        "tabx_get_profile": (_i32, [P, P, P]),
        "tabx_step_path": (_i32, [P, P]),
        "tabx_pipe_create": (_i32, [P, _i32, P, P, P]),
        "tabx_pipe_submit": (_i32, [P, P, P]),
        "tabx_pipe_result": (_i32, [P, ct.c_int64, P, P, P, P]),
        "tabx_pipe_destroy": (_i32, [P]),
        "tabx_debug_sincos": (_i32, [P, P, P, _i64, P]),
        "tabx_pack_bf16": (_i32, [P, _i64, _i32, _i32, P, P]),
        "tabx_policy_mlp": (_i32, [P, _i64, _i32, _i64, P, P, P, P, P, P]),
        "tabx_policy_mlp_sample": (_i32, [P, _i64, _i32, _i64, P, P, P, P, P, P, ct.c_uint64, P,
                                          ct.c_uint64, P, P, P]),
        "tabx_masked_sample": (_i32, [P, _i32, _i64, P, _i64, ct.c_uint64, P, ct.c_uint64, P, P,
                                      P]),
        "tabx_debug_phase_cycles": (_i32, [P, _i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.tabx_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI {L.tabx_abi_version()} != {ABI_VERSION}")
    sizes = [_i64() for _ in range(5)]
    L.tabx_struct_sizes(*[ct.byref(s) for s in sizes])
    mine = (ct.sizeof(TabxConfig), ct.sizeof(TabxOutputs), ct.sizeof(TabxState),
            ct.sizeof(TabxLevelSpec), ct.sizeof(TabxPcg64))
    if tuple(s.value for s in sizes) != mine:
        raise ImportError(f"{LIB_PATH}: struct layout mismatch {sizes} vs {mine}")
    _LIB = L
    return L


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != OK:
        msg = lib().tabx_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (code {rc}): {msg}")
