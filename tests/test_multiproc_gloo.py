"""Multi-rank path on CPU: env sharding + the episode-statistics all-reduce.

Two gloo ranks each step their own shard (the oracle stands in for the
per-GPU simulator here: the sharding and reduction logic are what is under
test), accumulate statistics, and all-reduce them once.  The reduced vector
must equal the sum of the shards computed independently, and the shards'
seeds must tile the global lane-seed sequence.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_01665_b200 import shard
from paper_2602_01665_b200.rng import lane_seeds

TOTAL = 12
STEPS = 130


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_stats(rank, world):
    from harness import case_scenario, orc

    sc = case_scenario("duel_expert")
    seeds = shard.shard_seeds(7, TOTAL, world, rank)
    sim = orc.OracleBatchSim([sc] * len(seeds), seeds, auto_reset=True)
    acc = {k: 0.0 for k in shard.STAT_KEYS}
    for _ in range(STEPS):
        o = sim.step(None)
        acc = shard.add_stats(acc, shard.stats_from_outputs(
            o["done"], o["winner"], o["reason"], o["first_kill"], o["episode_length"],
            o["episode_return"]))
    return acc


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = _shard_stats(rank, world)
        total = shard.reduce_episode_stats(local)
        out[rank] = (local, total)
    finally:
        dist.destroy_process_group()


def test_shards_tile_the_global_seed_sequence():
    for world in (1, 2, 3, 8):
        parts = [shard.shard_seeds(5, 100, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), lane_seeds(5, 100))
        ranges = [shard.shard_range(100, world, r) for r in range(world)]
        assert sum(c for _, c in ranges) == 100
        assert all(ranges[r][0] + ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))


def test_gloo_two_rank_statistics_reduction():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    expect = {k: 0.0 for k in shard.STAT_KEYS}
    for r in range(world):
        expect = shard.add_stats(expect, _shard_stats(r, world))
    for r in range(world):
        local, total = out[r]
        assert total == pytest.approx(expect, rel=0, abs=1e-9)
    assert expect["episodes"] > 0
    s = shard.summarize(expect)
    assert 0.0 <= s["win_rate"] <= 1.0 and s["mean_length"] > 0
