"""Build the in-tree CUDA extension ``_tabx.so`` for sm_100a.

    python -m paper_2602_01665_b200.build

Each translation unit is compiled in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false``
(``-fmad=false``: no product may be fused that the reference's numpy rounds),
then linked into one shared object next to this file.  Objects are cached
by source hash under ``build/`` so unchanged units are not recompiled.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("TABX_BUILD_OUT") or os.path.join(HERE, "_tabx.so")
BUILD = os.path.join(ROOT, "build", "tabx")

UNITS = ["tabx_lane_w1.cu", "tabx_lane_w2.cu", "tabx_lane_w4.cu", "tabx_lane_w8.cu",
         "tabx_fused.cu", "tabx_aux.cu", "tabx_levels.cu", "tabx_policy.cu", "tabx_mlp.cu", "tabx_pipe.cu", "tabx_capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("TABX_NVCC_EXTRA", "").split()
FLAGS = EXTRA + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _digest() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        with open(os.path.join(CSRC, name), "rb") as fh:
            h.update(name.encode())
            h.update(fh.read())
    with open(os.path.join(ROOT, "include", "tabx.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()[:16]


def _drop_stale() -> None:
    """Never leave a library from older sources behind a failed build."""
    for p in (OUT, OUT + ".stamp"):
        if os.path.exists(p):
            os.remove(p)


def build(verbose: bool = False, force: bool = False) -> str:
    tag = _digest()
    stamp = OUT + ".stamp"
    if not force and os.path.exists(OUT) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == tag:
                return OUT
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    procs = []
    objs = []
    for unit in UNITS:
        obj = os.path.join(BUILD, f"{unit}.{tag}.o")
        objs.append(obj)
        if os.path.exists(obj) and not force:
            continue
        cmd = [cc, *ARCH, *FLAGS, "-c", os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((unit, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                             stderr=subprocess.STDOUT, text=True)))
    failed = []
    for unit, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            print(out)
        if p.returncode != 0:
            failed.append((unit, out))
    if failed:
        _drop_stale()
        msg = "\n".join(f"--- {u}\n{o}" for u, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = OUT + ".tmp"
    link = subprocess.run([cc, *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
    if link.returncode != 0:
        _drop_stale()
        raise RuntimeError(f"link failed:\n{link.stdout}{link.stderr}")
    os.replace(tmp, OUT)
    with open(stamp, "w") as fh:
        fh.write(tag + "\n")
    return OUT


CHECKED_OUT = os.path.join(HERE, "_tabx_checked.so")


def build_checked(verbose: bool = False, selftest: bool = False) -> str:
    """The checked variant (-DTABX_CHECKS: device asserts, shared memory
    poisoned per environment, per-lane random delays at phase boundaries),
    a test-only library loaded with TABX_LIB by tests/test_gpu_checked.py."""
    global OUT, FLAGS
    saved = OUT, FLAGS
    OUT = CHECKED_OUT
    FLAGS = ["-DTABX_CHECKS"] + FLAGS
    if selftest:  # negative control: one stage hand-off without its __syncwarp
        OUT = os.path.join(HERE, "_tabx_selftest_race.so")
        FLAGS = ["-DTABX_SELFTEST_RACE"] + FLAGS
    try:
        return build(verbose=verbose)
    finally:
        OUT, FLAGS = saved


if __name__ == "__main__":
    if "--checked" in sys.argv or "--selftest" in sys.argv:
        print(build_checked(verbose="-v" in sys.argv, selftest="--selftest" in sys.argv))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
