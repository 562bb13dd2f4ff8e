"""Environment sharding across GPUs and the episode-statistics reduction.

Environments are independent, so a run of ``total`` lanes splits into
contiguous per-rank shards with no per-step communication.
Lane ``b`` of the global run always plays episode seed
``derive_seed(run_seed, b, TAG_EPISODE)`` (``bindings/.../__init__.py:51-55``),
whatever rank owns it.  The one collective is a sum all-reduce of a small
statistics vector per reporting window (NCCL over NVLink on GPUs, gloo on
CPU), from which :func:`summarize` derives the reference's
``rollout.summarize`` fields (``rollout.py:122-147``).

Parity contract (documented in DESIGN.md): each shard is one reference
``BatchSim`` over its lanes.  The reference refreshes every lane's
visibility caches whenever any lane of the same ``BatchSim`` resets
(``environment.py:508``); shards make that decision per shard.
"""
from __future__ import annotations

import numpy as np

from .rng import lane_seeds

STAT_KEYS = ("episodes", "ally_wins", "first_kill_ally", "truncation_ties", "sum_length",
             "sum_return", "eliminations", "env_steps")


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first lane, lane count) of ``rank``; the last rank takes the remainder."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    per = total // world
    first = rank * per
    count = total - first if rank == world - 1 else per
    return first, count


def shard_seeds(run_seed: int, total: int, world: int, rank: int) -> np.ndarray:
    first, count = shard_range(total, world, rank)
    return lane_seeds(run_seed, count, first)


def stats_vector(stats: dict):
    import torch
    return torch.tensor([float(stats.get(k, 0.0)) for k in STAT_KEYS], dtype=torch.float64)


def reduce_episode_stats(stats: dict, device=None, group=None) -> dict:
    """Sum the per-shard statistics over all ranks (one all-reduce)."""
    import torch
    import torch.distributed as dist

    vec = stats_vector(stats)
    if device is not None:
        vec = vec.to(device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    return dict(zip(STAT_KEYS, vec.cpu().tolist()))


def summarize(stats: dict) -> dict:
    """rollout.summarize fields from summed statistics."""
    n = int(stats.get("episodes", 0))
    if n == 0:
        return {"episodes": 0, "win_rate": 0.0, "mean_return": 0.0, "mean_length": 0.0,
                "first_kill_rate": 0.0}
    return {"episodes": n, "win_rate": stats["ally_wins"] / n,
            "mean_return": stats["sum_return"] / n, "mean_length": stats["sum_length"] / n,
            "first_kill_rate": stats["first_kill_ally"] / n}


def stats_from_outputs(done, winner, reason, first_kill, episode_length,
                       episode_return, running=None) -> dict:
    """Statistics of one step (host arrays): the lanes that finished, and the
    env-steps taken (``running``: lanes that were running; default all, as
    under auto-reset)."""
    d = np.asarray(done, bool)
    return {
        "env_steps": float(d.size if running is None else np.count_nonzero(running)),
        "episodes": float(d.sum()),
        "ally_wins": float((np.asarray(winner)[d] == 0).sum()),
        "first_kill_ally": float((np.asarray(first_kill)[d] == 0).sum()),
        "truncation_ties": float((np.asarray(reason)[d] == 3).sum()),
        "sum_length": float(np.asarray(episode_length)[d].sum()),
        "sum_return": float(np.asarray(episode_return)[d].sum()),
        "eliminations": float((np.asarray(reason)[d] == 1).sum()),
    }


def add_stats(a: dict, b: dict) -> dict:
    return {k: a.get(k, 0.0) + b.get(k, 0.0) for k in STAT_KEYS}
