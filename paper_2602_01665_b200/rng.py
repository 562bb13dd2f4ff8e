"""Counter-based RNG keys, host side.

The device kernel evaluates the same keyed SplitMix64 hash per (seed, step,
tag, lane) (``pkg/src/skirmish/rng.py:25-48``); the host only needs it to
derive per-lane episode seeds (``bindings/.../__init__.py:51-55``) and to
check the device stream in tests.  Plain Python integers modulo 2**64 — no
numpy overflow semantics to depend on.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MULT_STEP = 0xC2B2AE3D27D4EB4F
MULT_LANE = 0x165667B19E3779F9

TAG_EPISODE = 1
TAG_RESEED = 2
TAG_HEURISTIC_EXPLORE = 3
TAG_HEURISTIC_PICK = 4
TAG_RANDOM_ACTION = 5
TAG_LEVEL = 6


def splitmix_finalize(x: int) -> int:
    x &= MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def key_hash(seed: int, step: int = 0, tag: int = 0, lane: int = 0) -> int:
    """hash_u64 for scalar Python ints (rng.py:31-37)."""
    h = splitmix_finalize(int(seed) + GOLDEN * int(tag))
    h = splitmix_finalize(h + (int(step) & MASK64) * MULT_STEP)
    return splitmix_finalize(h + (int(lane) & MASK64) * MULT_LANE)


def derive_seed(seed: int, index: int, tag: int) -> int:
    """Child seed (rng.py:46-48)."""
    return key_hash(seed, index, tag)


def lane_seeds(run_seed: int, count: int, first: int = 0) -> np.ndarray:
    """derive_seed(run_seed, b, TAG_EPISODE) for b in [first, first+count)."""
    return np.array([derive_seed(run_seed, b, TAG_EPISODE) for b in range(first, first + count)],
                    dtype=np.uint64)


def uniform(seed: int, step: int, tag: int, lane: int) -> float:
    """53-bit uniform in [0, 1) (rng.py:40-43)."""
    return float(key_hash(seed, step, tag, lane) >> 11) * (1.0 / (1 << 53))
