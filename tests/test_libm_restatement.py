"""The device scalar math, compiled for the host, equals numpy bit for bit.

csrc/tabx_math.cuh is shared between the CUDA kernels and this host build
(g++ -ffp-contract=off, the same no-contraction rule as nvcc -fmad=false), so
a CPU match here pins the device arithmetic: glibc-2.39 sin/cos restatement
vs np.sin/np.cos, numpy pairwise summation, np.remainder.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "..", "paper_2602_01665_b200", "csrc")


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("libm")
    exe = str(d / "libm_check")
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-I", CSRC,
                           os.path.join(HERE, "native", "libm_check.cpp"), "-o", exe])
    return exe, d


def _run(tool, mode, x, *extra):
    exe, d = tool
    src, dst = str(d / "in.bin"), str(d / "out.bin")
    np.ascontiguousarray(x, dtype=np.float64).tofile(src)
    subprocess.check_call([exe, mode, src, dst, *map(str, extra)])
    return np.fromfile(dst)


def _heading_orbits():
    r = np.radians(30.0)
    out = []
    for h0 in (0.0, np.pi, np.radians(-75.0), np.radians(90.0), np.radians(45.0),
               np.radians(270.0)):
        h = h0
        for _ in range(2000):
            out += [h, h + r]
            h = (h + r) % (2.0 * np.pi)
    return np.array(out)


def test_sin_cos_match_numpy(tool):
    rng = np.random.default_rng(20260822)
    x = np.concatenate([
        rng.uniform(0.0, 2.0 * np.pi, 1_500_000),
        rng.uniform(-60.0, 60.0, 500_000),
        rng.uniform(-0.2, 0.2, 200_000),
        10.0 ** rng.uniform(-12, 0, 100_000),
        np.concatenate([k * np.pi / 2 + rng.uniform(-1e-6, 1e-6, 500) for k in range(-20, 21)]),
        _heading_orbits(),
        np.array([0.0, -0.0, 5e-324, 2.0 ** -27, 2.0 ** -26, 0.126, 0.85546875, 2.426265,
                  np.pi, 2 * np.pi, np.radians(180.0), np.radians(30.0)]),
    ])
    for mode in ("sincos", "sincos2"):  # separate calls / shared reduction
        y = _run(tool, mode, x).reshape(-1, 2)
        bad_s = np.nonzero(y[:, 0] != np.sin(x))[0]
        bad_c = np.nonzero(y[:, 1] != np.cos(x))[0]
        assert len(bad_s) == 0 and len(bad_c) == 0, (mode, x[bad_s[:5]], x[bad_c[:5]])


@pytest.mark.parametrize("n", [1, 3, 6, 7, 8, 9, 15, 16, 20, 31, 100, 127, 128, 129, 200, 256])
def test_pairwise_sum_matches_numpy(tool, n):
    rng = np.random.default_rng(n)
    rows = rng.random((300, n)) * 10.0 ** rng.integers(-4, 5, size=(300, n))
    rows[rng.random((300, n)) < 0.3] = 0.0
    got = _run(tool, "pairwise", rows.ravel(), n)
    assert np.array_equal(got, rows.sum(axis=1))


def test_remainder_matches_numpy(tool):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-20, 20, 100_000), [0.0, -0.0, 2 * np.pi, -2 * np.pi]])
    got = _run(tool, "remainder", x, repr(2.0 * np.pi))
    ref = x % (2.0 * np.pi)
    assert np.array_equal(got, ref) and np.array_equal(np.signbit(got), np.signbit(ref))
