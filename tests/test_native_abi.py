"""The C-ABI library loads without a GPU and exports everything tabx.h declares."""
import ctypes as ct
import os
import re

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
HEADER = os.path.join(ROOT, "include", "tabx.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|const char\*)\s+(tabx_\w+)\s*\(", text,
                                 flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_01665_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        from paper_2602_01665_b200.build import build
        build()
    return _native.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("tabx_create", "tabx_step", "tabx_reset_env", "tabx_init_output",
                 "tabx_export_state", "tabx_import_state", "tabx_get_error", "tabx_destroy",
                 "tabx_episode_stats", "tabx_respawn_all"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_struct_layouts_match(lib):
    from paper_2602_01665_b200 import _native as nat
    sizes = [ct.c_int64() for _ in range(5)]
    lib.tabx_struct_sizes(*[ct.byref(s) for s in sizes])
    assert [s.value for s in sizes] == [ct.sizeof(nat.TabxConfig), ct.sizeof(nat.TabxOutputs),
                                        ct.sizeof(nat.TabxState), ct.sizeof(nat.TabxLevelSpec),
                                        ct.sizeof(nat.TabxPcg64)]


def test_dims_and_errors_without_gpu(lib):
    assert lib.tabx_obs_dim(20, 6) == 386 and lib.tabx_global_dim(20, 6) == 348
    assert lib.tabx_obs_dim(100, 0) == 1698 and lib.tabx_global_dim(100, 0) == 1500
    h = ct.c_void_p()
    # bad arguments are rejected before any CUDA call
    assert lib.tabx_create(None, 0, None, None, 0, 0, 0, None, ct.byref(h)) == 1
    assert b"bad argument" in lib.tabx_last_error()


@pytest.mark.parametrize("n,z", [(257, 0), (20, 33), (0, 0)])
def test_capacity_limits_fail_loudly(lib, n, z):
    """The documented capacity (N <= 256 units, Z <= 32 zones)
    is a loud error at both layers, never a silent truncation: the host
    template raises ValueError and tabx_create returns TABX_E_ARGUMENT
    before touching the device."""
    import numpy as np

    from paper_2602_01665_b200 import _native as nat
    from paper_2602_01665_b200.scenario import builtin_scenario
    from paper_2602_01665_b200.template import build_config

    sc = builtin_scenario("c3_10v10_terrain")
    sc.max_units, sc.max_zones = n, z
    with pytest.raises(ValueError, match="outside"):
        build_config(sc, validate=False)
    cfg = build_config(builtin_scenario("c3_10v10_terrain"))
    cfg.n_units, cfg.n_zones = n, z
    seeds = np.zeros(1, dtype=np.uint64)
    h = ct.c_void_p()
    rc = lib.tabx_create(ct.byref(cfg), 1, None, seeds.ctypes.data, 1, 1, 0, None, ct.byref(h))
    assert rc == 1 and not h.value
    assert b"capacity out of range" in lib.tabx_last_error()
    assert nat.MAX_UNITS == 256 and nat.MAX_ZONES == 32


def test_template_matches_oracle_spawn():
    """Host template values equal the oracle's fill_env columns (bit-exact)."""
    import numpy as np

    from harness import orc
    from paper_2602_01665_b200.scenario import builtin_scenario
    from paper_2602_01665_b200.template import build_config

    for name in ("c1_3v3", "c3_10v10_terrain", "c4_50v50", "mixed_kings"):
        sc = builtin_scenario(name).scripted()
        c = build_config(sc)
        s = orc.build_state([sc], np.array([1], np.uint64))
        N = sc.max_units
        for fld, arr in (("max_health", s.u_max_health), ("radius", s.u_radius),
                         ("inv_mass", s.u_inv_mass), ("sight_cos_half", s.u_sight_cos_half),
                         ("spawn_heading", s.heading), ("speed", s.u_speed)):
            assert np.array_equal(np.array(getattr(c, fld)[:N]), arr[0]), (name, fld)
        assert np.array_equal(np.array(c.spawn_x[:N]), s.pos[0, :, 0])
        assert c.rot_step == s.rot_step[0]
        assert list(c.controller) == list(s.t_controller[0])
