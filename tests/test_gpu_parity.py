"""Parity of the CUDA step (through the C ABI) with the CPU oracle.

Every golden case is replayed on the GPU and by the oracle side by side from
the same seeds; all outputs and the exported state must be identical at
every step (float32 outputs = float64 oracle rounded to float32; state
bit-exact by value).  The oracle itself is pinned to the reference by
tests/test_oracle_golden.py.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from gpu_compare import compare_outputs, compare_state, oracle_state_dict  # noqa: E402
from harness import CASES, case_scenario, case_seeds, legal_pick, orc  # noqa: E402

from paper_2602_01665_b200.scenario import ActionMaskError, builtin_scenario  # noqa: E402
from paper_2602_01665_b200.sim import BatchSim  # noqa: E402


def _pair(name):
    case = CASES[name]
    sc = case_scenario(name)
    seeds = np.array(case_seeds(case), np.uint64)
    gpu = BatchSim([sc] * case["batch"], seeds, auto_reset=case["auto_reset"], device="cuda:0")
    ora = orc.OracleBatchSim([sc] * case["batch"], seeds, auto_reset=case["auto_reset"])
    return case, gpu, ora


@pytest.mark.parametrize("path", ["k0", "k1"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case_parity(name, path, monkeypatch):
    """path k0: heuristic decisions by the controller pass; k1: inside the
    step kernel (TABX_NO_K0=1, the path below 4,096 lanes)."""
    if path == "k1":
        monkeypatch.setenv("TABX_NO_K0", "1")
    case, gpu, ora = _pair(name)
    gen = np.random.default_rng(case["external"]) if "external" in case else None
    resets = {int(k): v for k, v in case.get("resets", {}).items()}
    bad = compare_outputs(gpu.last, ora.last, f"{name} t=0", check_final=False)
    bad += compare_state(gpu.export_state(), ora.sim, f"{name} t=0")
    assert not bad, "\n".join(bad[:10])
    for t in range(1, case["steps"] + 1):
        acts = legal_pick(ora.last["action_mask"], gen) if gen is not None else None
        o = ora.step(acts)
        g = gpu.step(acts)
        bad = compare_outputs(g, o, f"{name} t={t}")
        bad += compare_state(gpu.export_state(), ora.sim, f"{name} t={t}")
        assert not bad, "\n".join(bad[:10])
        for lane, seed in resets.get(t, []):
            ora.reset_env(lane, seed=seed)
            gpu.reset_env(lane, seed=seed)
            bad = compare_outputs(gpu.last, ora.last, f"{name} t={t} reset", check_final=False)
            bad += compare_state(gpu.export_state(), ora.sim, f"{name} t={t} reset")
            assert not bad, "\n".join(bad[:10])


def _perturbed_states(sc, B, seed):
    """Random mid-episode states: jittered and overlapping bodies, units out of
    the field, random headings / timers / health, dead units, memories."""
    rng = np.random.default_rng(seed)
    sim = orc.OracleBatchSim([sc] * B, np.arange(B, dtype=np.uint64) * 7919 + 1, auto_reset=True)
    s = sim.sim
    N = s.n_units
    act = s.u_active
    s.pos = s.pos + rng.normal(0.0, 4.0, s.pos.shape)
    clump = rng.random(B) < 0.3
    s.pos[clump] = s.pos[clump][:, :1, :] + rng.normal(0.0, 0.6, s.pos[clump].shape)
    out = rng.random((B, N)) < 0.05
    s.pos[out] = rng.uniform(-3.0, 43.0, (int(out.sum()), 2))
    s.heading = rng.uniform(0.0, 2 * np.pi, (B, N))
    s.health = np.where(act, s.u_max_health * rng.uniform(0.05, 1.0, (B, N)), s.health)
    full = rng.random((B, N)) < 0.3
    s.health = np.where(full & act, s.u_max_health, s.health)
    s.cooldown = np.where(rng.random((B, N)) < 0.5, 0.0, rng.uniform(0.0, 3.0, (B, N))) * act
    s.reveal = np.where(rng.random((B, N)) < 0.7, 0.0, rng.uniform(0.0, 1.0, (B, N))) * act
    dead = (rng.random((B, N)) < 0.1) & act
    s.alive = act & ~dead
    s.health = np.where(dead, 0.0, s.health)
    s.imp_dv = rng.normal(0.0, 0.3, s.imp_dv.shape) * act[..., None]
    s.mem_valid = (rng.random((B, N)) < 0.4) & act
    s.mem_pos = rng.uniform(0.0, 40.0, s.mem_pos.shape) * s.mem_valid[..., None]
    s.t = rng.integers(0, sc.max_steps, B).astype(np.int64)
    s.t[:2] = sc.max_steps - 1  # truncation next step
    s.prev_gap = rng.normal(0.0, 0.1, B)
    orc.fresh_caches(s)
    return sim


@pytest.mark.parametrize("scen,B,seed", [("c3_10v10_terrain", 96, 1), ("c2_10v10", 64, 2),
                                         ("mixed_kings", 128, 3), ("duel_terrain", 256, 4),
                                         ("c4_50v50", 6, 5), ("c1_3v3", 256, 6),
                                         ("c6_75v75_terrain", 6, 11)])
def test_injected_state_single_step(scen, B, seed):
    sc = builtin_scenario(scen).with_controllers(ally="random", enemy="heuristic:medium")
    ora = _perturbed_states(sc, B, seed)
    gpu = BatchSim([sc] * B, ora.sim.seed.copy(), auto_reset=True, device="cuda:0")
    gpu.import_state(oracle_state_dict(ora.sim))
    bad = compare_state(gpu.export_state(), ora.sim, f"{scen} injected")
    assert not bad, "\n".join(bad[:10])
    for t in range(3):
        o = ora.step(None)
        g = gpu.step(None)
        bad = compare_outputs(g, o, f"{scen} injected step {t}")
        bad += compare_state(gpu.export_state(), ora.sim, f"{scen} injected step {t}")
        assert not bad, "\n".join(bad[:10])


@pytest.mark.parametrize("path", ["k0", "single"])
def test_action_mask_error_matches_reference_and_mutates_nothing(path, monkeypatch):
    """path k0: controller pass + step kernels; single: the small-batch
    single-launch step (in-kernel controller, TABX_NO_K0=1)."""
    if path == "single":
        monkeypatch.setenv("TABX_NO_K0", "1")
    sc = builtin_scenario("c2_10v10")  # ally external
    B = 4
    seeds = np.arange(B, dtype=np.uint64)
    gpu = BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim([sc] * B, seeds, auto_reset=True)
    acts = np.zeros((B, sc.max_units), np.int64)
    gpu.step(acts)
    ora.step(acts)
    before = {k: v.clone() for k, v in gpu.export_state().items()}
    bad = acts.copy()
    bad[2, 3] = 6  # noop not enabled
    bad[3, 1] = 9  # out of range
    with pytest.raises(orc.OracleActionMaskError) as eo:
        ora.step(bad)
    with pytest.raises(ActionMaskError) as eg:
        gpu.step(bad)
    assert str(eg.value) == str(eo.value) == "invalid action 6 for unit 3 in env 2"
    after = gpu.export_state()
    for k, v in before.items():
        assert torch.equal(v, after[k]), k
    # the simulator keeps working after the error
    o = ora.step(acts)
    g = gpu.step(acts)
    assert gpu.step_path() == ("single" if path == "single" else "split")
    assert not compare_outputs(g, o, "after error")


def test_dead_units_accept_any_action():
    sc = builtin_scenario("c2_10v10")
    gpu = BatchSim([sc], np.array([5], np.uint64), device="cuda:0")
    ora = orc.OracleBatchSim([sc], np.array([5], np.uint64))
    st = oracle_state_dict(ora.sim)
    st["alive"][0, 0] = False
    st["health"][0, 0] = 0.0
    ora.sim.alive[0, 0] = False
    ora.sim.health[0, 0] = 0.0
    gpu.import_state(st)
    acts = np.zeros((1, sc.max_units), np.int64)
    acts[0, 0] = 42
    o = ora.step(acts)
    g = gpu.step(acts)
    assert not compare_outputs(g, o, "dead unit")


def test_device_libm_matches_numpy():
    from paper_2602_01665_b200 import _native as nat
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(0, 2 * np.pi, 2_000_000), rng.uniform(-50, 50, 500_000),
                        rng.uniform(-0.2, 0.2, 200_000), [0.0, -0.0, np.pi, 2 * np.pi]])
    xt = torch.from_numpy(x).cuda()
    s = torch.empty_like(xt)
    c = torch.empty_like(xt)
    nat.check(nat.lib().tabx_debug_sincos(xt.data_ptr(), s.data_ptr(), c.data_ptr(), len(x),
                                          torch.cuda.current_stream().cuda_stream), "sincos")
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), np.sin(x))
    assert np.array_equal(c.cpu().numpy(), np.cos(x))


def test_fov_boundary_fixtures_through_kernel():
    """The reference's 100 FoV boundary verdicts, via the visibility cache."""
    import json
    import os
    from dataclasses import replace

    from golden_cases import GOLDEN_DIR
    from paper_2602_01665_b200.scenario import Field, Scenario, Team, Unit, UnitSpec

    with open(os.path.join(GOLDEN_DIR, "fov_samples.json")) as fh:
        samples = json.load(fh)
    scs, heads = [], []
    for smp in samples:
        spec = UnitSpec(100.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, sight_angle=smp["sight_angle"],
                        sight_range=smp["sight_range"])
        far = UnitSpec(100.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0)
        units = [Unit(0, tuple(smp["position"]), spec=spec),
                 Unit(0, tuple(np.clip(smp["point"], 0.0, 60.0)), spec=far),
                 Unit(1, (59.0, 59.0), spec=far)]
        scs.append(Scenario("fov", units, field=Field(60.0, 60.0, 2.0),
                            teams=(Team(0, "random"), Team(1, "random"))))
        heads.append(smp["heading"])
    gpu = BatchSim(scs, np.arange(len(scs), dtype=np.uint64), device="cuda:0")
    st = {k: v.cpu().numpy() for k, v in gpu.export_state().items()}
    st["heading"][:, 0] = heads
    st["pos"][:, 1] = [s["point"] for s in samples]
    gpu.import_state(st)
    gpu._init_output()  # refresh_caches at the injected state
    vis = gpu.export_state()["vis"].cpu().numpy()
    got = vis[:, 0, 1]
    want = np.array([s["inside"] for s in samples])
    assert np.array_equal(got, want), np.nonzero(got != want)


def test_mixed_configs_and_reset_env_swap():
    a = builtin_scenario("duel_terrain").with_controllers(ally="random", enemy="heuristic:expert")
    b = a.with_controllers(ally="heuristic:novice", enemy="random")
    from dataclasses import replace
    from paper_2602_01665_b200.scenario import Physics
    b = replace(b, physics=Physics(dt=0.05, enable_noop=True), max_steps=50)
    configs = [a, b, a, b, b, a]
    seeds = np.arange(6, dtype=np.uint64) + 100
    gpu = BatchSim(configs, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim(configs, seeds, auto_reset=True)
    for t in range(1, 120):
        o = ora.step(None)
        g = gpu.step(None)
        bad = compare_outputs(g, o, f"mixed t={t}") + compare_state(gpu.export_state(), ora.sim,
                                                                    f"mixed t={t}")
        assert not bad, "\n".join(bad[:10])
        if t == 30:
            ora.reset_env(1, a, seed=77)
            gpu.reset_env(1, a, seed=77)
            assert not compare_outputs(gpu.last, ora.last, "swap", check_final=False)


def test_large_batch_lanes_match_small_batch_oracle():
    """B=4096 on the GPU; lanes 0..47 must equal a 48-lane oracle run given the
    big batch's refresh decisions (the reference's batch-coupled cache refresh,
    environment.py:508)."""
    name = "duel_expert"
    case = CASES[name]
    sc = case_scenario(name)
    big = 4096
    seeds_big = np.array([orc.keyed_hash(np.uint64(7), b, 1) for b in range(big)], np.uint64)
    gpu = BatchSim([sc] * big, seeds_big, auto_reset=True, device="cuda:0")
    sub = 48
    ora = orc.OracleBatchSim([sc] * sub, seeds_big[:sub], auto_reset=True)
    for t in range(1, 200):
        g = gpu.step(None)
        any_reset = bool(g.reset_mask.any().item())
        o = ora.step(None, refresh=any_reset)
        gs = gpu.export_state()
        for k in ("pos", "health", "heading", "alive", "t", "mem_pos"):
            gv = gs[k][:sub].cpu().numpy()
            ov = getattr(ora.sim, k)
            assert np.array_equal(gv, ov), (t, k)
        assert np.array_equal(g.observations[:sub].cpu().numpy(),
                              o["observations"].astype(np.float32)), t


def test_determinism_full_size():
    sc = builtin_scenario("c3_10v10_terrain").scripted()
    B = 65536
    seeds = np.arange(B, dtype=np.uint64)
    runs = []
    for _ in range(2):
        gpu = BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0", interactions=False)
        for _ in range(20):
            out = gpu.step(None)
        st = gpu.export_state()
        runs.append((out.observations.clone(), st["pos"].clone(), st["health"].clone()))
        gpu.close()
    for a, b in zip(*runs):
        assert torch.equal(a, b)


def test_episode_statistics_match_oracle():
    """Device per-lane accumulators == statistics summed from oracle outputs."""
    from paper_2602_01665_b200 import shard
    name = "duel_expert"
    case = CASES[name]
    sc = case_scenario(name)
    seeds = np.array(case_seeds(case), np.uint64)
    gpu = BatchSim([sc] * case["batch"], seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim([sc] * case["batch"], seeds, auto_reset=True)
    acc = {k: 0.0 for k in shard.STAT_KEYS}
    for _ in range(case["steps"]):
        gpu.step(None)
        o = ora.step(None)
        acc = shard.add_stats(acc, shard.stats_from_outputs(
            o["done"], o["winner"], o["reason"], o["first_kill"], o["episode_length"],
            o["episode_return"]))
    got = gpu.episode_stats()
    for k in shard.STAT_KEYS:
        if k == "sum_return":
            assert got[k] == pytest.approx(acc[k], rel=1e-12, abs=1e-12)
        else:
            assert got[k] == acc[k], k


@pytest.mark.parametrize("policy", ["random", "mlp"])
def test_graph_rollout_replays_exactly(policy):
    """C5 loop: the CUDA-graph-captured horizon equals an eager BatchSim fed
    the same recorded actions; every sampled action is legal."""
    from paper_2602_01665_b200.rollout import Rollout
    from paper_2602_01665_b200.rng import lane_seeds
    sc = builtin_scenario("c3_10v10_terrain")
    B, T = 64, 12
    ro = Rollout(sc, B, horizon=T, policy=policy, device=0, seed=3)
    ro.capture()  # runs one eager warm-up horizon, then records the graph
    start = {k: v.clone() for k, v in ro.sim.export_state().items() if k != "config"}
    mask = ro.sim._buf["action_mask"].clone()
    buf = ro.run()
    torch.cuda.synchronize()
    ref = BatchSim([sc.with_controllers(ally="external")] * B, lane_seeds(3, B), auto_reset=True,
                   device="cuda:0", interactions=False)
    ref.import_state(start)
    for t in range(T):
        a = buf.actions[t]
        assert bool(torch.gather(mask, 2, a[..., None]).all()), t
        out = ref.step(a)
        assert torch.equal(out.rewards, buf.rewards[t]), t
        assert torch.equal(out.observations, buf.observations[t + 1]), t
        assert torch.equal(out.terminated, buf.terminated[t]), t
        mask = out.action_mask.clone()
    ro.close()


def _many_zones(n_zones: int):
    """duel_terrain with n_zones overlapping zones (lava stacks at the centre,
    so the burn is a numpy pairwise sum once Z >= 8; bushes and swamps around)."""
    import dataclasses

    from paper_2602_01665_b200.scenario import Zone
    base = builtin_scenario("duel_terrain")
    kinds = ("lava", "bush", "swamp")
    zones = []
    for k in range(n_zones):
        t = kinds[k % 3]
        if t == "lava":
            zones.append(Zone("lava", (20.0 + 0.3 * (k % 5), 20.0), (6.0 + k * 0.7, 4.0 + k * 0.3),
                              1.5 + 0.37 * k))
        elif t == "bush":
            zones.append(Zone("bush", (8.0 + 2.5 * (k % 9), 12.0 + (k % 4)), (3.0, 2.0), 0.0))
        else:
            zones.append(Zone("swamp", (30.0 - (k % 7), 28.0), (4.0, 3.0 + 0.1 * k),
                              0.3 + 0.02 * k))
    return dataclasses.replace(base, zones=zones, max_zones=n_zones, notes=list(base.notes))


@pytest.mark.parametrize("n_zones,B,seed", [(12, 128, 7), (24, 64, 8), (32, 32, 9)])
def test_many_zones_match_oracle(n_zones, B, seed):
    """Zone counts beyond the benchmark maps: the pairwise lava sum (Z >= 8),
    the generic zone-block path of the observation kernel, wide zone masks."""
    sc = _many_zones(n_zones).with_controllers(ally="random", enemy="heuristic:medium")
    ora = _perturbed_states(sc, B, seed)
    ora.sim.pos[:, :, :] = np.clip(ora.sim.pos, 0.0, 40.0) * 0.5 + 10.0  # pull into the zones
    orc.fresh_caches(ora.sim)
    gpu = BatchSim([sc] * B, ora.sim.seed.copy(), auto_reset=True, device="cuda:0")
    gpu.import_state(oracle_state_dict(ora.sim))
    for t in range(4):
        o = ora.step(None)
        g = gpu.step(None)
        bad = compare_outputs(g, o, f"Z={n_zones} step {t}")
        bad += compare_state(gpu.export_state(), ora.sim, f"Z={n_zones} step {t}")
        assert not bad, "\n".join(bad[:10])


def test_two_word_rows_with_zones_match_oracle():
    """W = 2 (40 units) on a map with 10 zones: the multi-word visibility rows,
    the per-CTA env layout and the generic zone / pair paths of the
    observation kernel."""
    import dataclasses
    base = builtin_scenario("c4_50v50")
    allies = [u for u in base.units if u.team == 0][:20]
    enemies = [u for u in base.units if u.team == 1][:20]
    zones = _many_zones(10).zones
    sc = dataclasses.replace(base, units=allies + enemies, zones=zones, max_units=40,
                             max_zones=10, notes=list(base.notes))
    sc = sc.with_controllers(ally="random", enemy="heuristic:medium")
    ora = _perturbed_states(sc, 24, 10)
    gpu = BatchSim([sc] * 24, ora.sim.seed.copy(), auto_reset=True, device="cuda:0")
    gpu.import_state(oracle_state_dict(ora.sim))
    for t in range(3):
        o = ora.step(None)
        g = gpu.step(None)
        bad = compare_outputs(g, o, f"W=2 step {t}")
        bad += compare_state(gpu.export_state(), ora.sim, f"W=2 step {t}")
        assert not bad, "\n".join(bad[:10])


def test_controller_pass_mixed_heuristic_counts():
    """K0 (the packed heuristic-controller pass ahead of K1) over a batch whose
    configs have 10 and 20 heuristic units per env: packing follows the
    largest count, every env matches the oracle."""
    a = builtin_scenario("c3_10v10_terrain").with_controllers(ally="random",
                                                              enemy="heuristic:medium")
    b = builtin_scenario("c3_10v10_terrain").with_controllers(ally="heuristic:expert",
                                                              enemy="heuristic:medium")
    configs = [a, b, b, a, a, b, a, a] * 6
    seeds = np.arange(len(configs), dtype=np.uint64) * 31 + 5
    gpu = BatchSim(configs, seeds, auto_reset=True, device="cuda:0")
    ora = orc.OracleBatchSim(configs, seeds, auto_reset=True)
    for t in range(1, 60):
        o = ora.step(None)
        g = gpu.step(None)
        bad = compare_outputs(g, o, f"k0 mixed t={t}") + compare_state(gpu.export_state(), ora.sim,
                                                                       f"k0 mixed t={t}")
        assert not bad, "\n".join(bad[:10])


@pytest.mark.parametrize("scen,B", [("c3_10v10_terrain", 32768), ("c4_50v50", 2048)])
def test_controller_pass_equals_in_kernel_controller(scen, B, monkeypatch):
    """Large batches (C3: one env per warp; C4: W = 4, four warps per env):
    the K0 decision path and K1's in-kernel controller (TABX_NO_K0=1, read
    when the batch is created) give identical observations and state step
    for step."""
    sc = builtin_scenario(scen)
    seeds = np.arange(B, dtype=np.uint64) + 3
    sims = []
    for flag in ("0", "1"):
        monkeypatch.setenv("TABX_NO_K0", flag)
        sims.append(BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0",
                             interactions=False))
    for t in range(40):
        outs = [s.step(None) for s in sims]
        assert torch.equal(outs[0].observations, outs[1].observations), t
        assert torch.equal(outs[0].rewards, outs[1].rewards), t
    s0, s1 = (s.export_state() for s in sims)
    for k in ("pos", "health", "heading", "alive", "mem_pos", "mem_valid"):
        assert torch.equal(s0[k], s1[k]), k


def test_controller_pass_graph_after_config_growth():
    """A CUDA graph captured while every config had 10 heuristic units keeps
    its K0 packing (3 envs per warp) when reset_env later brings in a config
    with 20: that env's units take a second round on the same lanes, and
    every step still matches the oracle."""
    import ctypes as ct

    from paper_2602_01665_b200 import _native as nat
    a = builtin_scenario("c3_10v10_terrain").with_controllers(ally="random",
                                                              enemy="heuristic:medium")
    b = builtin_scenario("c3_10v10_terrain").with_controllers(ally="heuristic:expert",
                                                              enemy="heuristic:medium")
    B = 48
    seeds = np.arange(B, dtype=np.uint64) + 900
    s = torch.cuda.Stream()
    gpu = BatchSim([a] * B, seeds, auto_reset=True, device="cuda:0", stream=s)
    ora = orc.OracleBatchSim([a] * B, seeds, auto_reset=True)
    L = nat.lib()

    def launch():
        nat.check(L.tabx_step(gpu.handle, None, ct.byref(gpu._outs)), "tabx_step")

    with torch.cuda.stream(s):
        launch()  # eager warm-up step (the handle counts 10 heuristic units)
    s.synchronize()
    ora.step(None)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        launch()
    for lane in (5, 17):
        ora.reset_env(lane, b, seed=lane + 3)
        gpu.reset_env(lane, b, seed=lane + 3)
    for t in range(1, 25):
        graph.replay()
        torch.cuda.synchronize()
        o = ora.step(None)
        bad = compare_state(gpu.export_state(), ora.sim, f"graph t={t}")
        got = gpu._buf["observations"].cpu().numpy()
        if not np.array_equal(got, o["observations"].astype(np.float32)):
            bad.append(f"graph t={t}: observations differ")
        assert not bad, "\n".join(bad[:10])
    gpu.close()


@pytest.mark.parametrize("scen,B", [("c3_10v10_terrain", 8192), ("c2_10v10", 8192),
                                    ("c4_50v50", 1024)])
def test_shape_specialised_kernels_equal_generic(scen, B, monkeypatch):
    """The step and observation kernels compiled for a fixed (N, Z) and the
    generic ones (TABX_GENERIC_SHAPES=1, read when the batch is created) give
    identical observations, rewards and state step for step."""
    sc = builtin_scenario(scen)
    seeds = np.arange(B, dtype=np.uint64) + 11
    sims = []
    for flag in ("0", "1"):
        monkeypatch.setenv("TABX_GENERIC_SHAPES", flag)
        sims.append(BatchSim([sc] * B, seeds, auto_reset=True, device="cuda:0",
                             interactions=False))
    for t in range(30):
        outs = [s.step(None) for s in sims]
        assert torch.equal(outs[0].observations, outs[1].observations), t
        assert torch.equal(outs[0].global_state, outs[1].global_state), t
        assert torch.equal(outs[0].rewards, outs[1].rewards), t
    s0, s1 = (s.export_state() for s in sims)
    for k in ("pos", "health", "heading", "alive", "mem_pos", "vis", "atk"):
        assert torch.equal(s0[k], s1[k]), k


def test_misaligned_global_state_is_rejected_before_launch():
    """global_state leaves through TMA bulk stores: a buffer that is not
    16-byte aligned is refused with TABX_E_ALIGNMENT (no launch, the context
    stays healthy)."""
    import ctypes as ct

    from paper_2602_01665_b200 import _native as nat
    sc = builtin_scenario("c1_3v3").scripted()
    gpu = BatchSim([sc] * 4, np.arange(4, dtype=np.uint64), device="cuda:0")
    raw = torch.empty(4 * gpu.global_dim + 1, dtype=torch.float32, device="cuda:0")
    outs = nat.TabxOutputs.from_buffer_copy(gpu._outs)
    outs.global_state = raw.data_ptr() + 4
    rc = nat.lib().tabx_step(gpu.handle, None, ct.byref(outs))
    assert rc == nat.E_ALIGNMENT
    assert "16-byte" in nat.lib().tabx_last_error().decode()
    gpu.step(None)
    torch.cuda.synchronize()
    gpu.close()
