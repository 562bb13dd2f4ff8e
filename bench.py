"""Throughput of the B200 batched environment step (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--scenario c3] [--envs B]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...     # the reference's CPU step (oracle port)

Workload (BASELINE.json configs[2], the metric's config): C3 = 10v10
heterogeneous roles on the 2L2B2S terrain map, 262,144 environments per GPU
(weak scaling: rank g owns global lanes [g*B, (g+1)*B) with their global lane
seeds; no per-step communication).  Ally team on the in-engine random
controller, enemy heuristic-medium (the reference bench's ``_scripted`` rule,
rollout.py:360-366); auto-reset on; episodes truncate at t=400.

* ``value``: env-steps/s of the whole job, state and outputs resident in
  HBM, CUDA-event timed over K steps (max over ranks).  Each step writes
  ~8.1 GB of observations, so every timed step streams far more than L2.
* ``e2e``: the same metric through the trainer API (``bindings.HostStepper``
  over ``bindings.step``) with host buffers, for the same K steps: int64
  actions copied from pinned host memory every step (ally team external),
  rewards + terminated + truncated copied back every step; the copies run on
  copy streams and overlap the neighbouring steps' kernels.  Observations
  and masks stay on the device; ``host_obs_e2e`` prices copying them out.
* ``c1`` / ``c2`` / ``c4``: the other BASELINE configs (value, roofline, e2e)
  measured the same way in the same run; ``c3_episode``: a whole episode
  (t = 1..410 from the start, across the lockstep t = 400 auto-reset);
  ``reconfig``: the reference's reconfiguration-latency protocol.
* ``roofline``: the step kernel's algorithmic HBM bytes (SURVEY.md §8(d):
  4·N·obs_dim + 4·gdim + 4N + 7N + 3 + 8N + 2·(89N+40) per env-step) per
  launch ÷ its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline``: the oracle port of the reference step (numpy, same
  numerics as the reference) on a bounded sample, 1 host thread.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCENARIOS = {"c1": "c1_3v3", "c2": "c2_10v10", "c3": "c3_10v10_terrain", "c4": "c4_50v50"}
DEFAULT_ENVS = {"c1": 256, "c2": 65536, "c3": 262144, "c4": 131072}
WORKLOAD = {
    "c1": "C1 3v3 farmers, open map, random ally vs heuristic-medium enemy",
    "c2": "C2 10v10 heterogeneous roles (melee/ranged/support), random vs heuristic-medium",
    "c3": "C3 10v10 heterogeneous roles on the 2L2B2S terrain map (lava, bush, swamp), "
          "random vs heuristic-medium",
    "c4": "C4 50v50 large battle, random vs heuristic-medium",
}


def algorithmic_bytes(N: int, Z: int) -> int:
    """SURVEY.md §8(d) compulsory bytes per env-step."""
    D = 15 + 17 * (N - 1) + 8 * Z
    G = 15 * N + 8 * Z
    return 4 * N * D + 4 * G + 4 * N + 7 * N + 3 + 8 * N + 2 * (89 * N + 40)


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML, or
    nvidia-smi when NVML is not importable)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML (nvidia_ml_py) when present: ~2 ms sampling, so even a 60 ms
        # timed region gets tens of samples; nvidia-smi otherwise
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(self.idx), str(sm), str(mx), hex(r)] +
                                 ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.002)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}",
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference(scenario_key: str, envs: int, steps: int, warmup: int, seed: int = 0) -> dict:
    """The reference's CPU step (numpy oracle port) on a bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import tabx_oracle as orc

    from paper_2602_01665_b200.rng import lane_seeds
    from paper_2602_01665_b200.scenario import builtin_scenario

    sc = builtin_scenario(SCENARIOS[scenario_key]).scripted()
    sim = orc.OracleBatchSim([sc] * envs, lane_seeds(seed, envs), auto_reset=True)
    for _ in range(warmup):
        sim.step(None)
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step(None)
    dt = time.perf_counter() - t0
    return {"env_steps_per_s": envs * steps / dt, "seconds": dt, "envs": envs, "steps": steps,
            "n_units": len(sc.units), "numpy": np.__version__}


def _ref_worker(job):
    """One host process: its own oracle BatchSim shard, timed after a barrier."""
    scenario_key, envs, steps, warmup, first, barrier = job
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import tabx_oracle as orc

    from paper_2602_01665_b200.rng import lane_seeds
    from paper_2602_01665_b200.scenario import builtin_scenario

    sc = builtin_scenario(SCENARIOS[scenario_key]).scripted()
    sim = orc.OracleBatchSim([sc] * envs, lane_seeds(0, envs, first), auto_reset=True)
    for _ in range(warmup):
        sim.step(None)
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step(None)
    return t0, time.perf_counter()


def cpu_reference_parallel(scenario_key, envs_per_worker, steps, warmup, workers) -> dict:
    """The reference's CPU step on every host core: one process per core,
    each an independent BatchSim over its own lanes (the reference's own
    parallel bench, rollout.py:384-409, without the GIL)."""
    import multiprocessing as mproc
    import numpy as np

    ctx = mproc.get_context("fork")
    mgr = ctx.Manager()
    barrier = mgr.Barrier(workers)
    jobs = [(scenario_key, envs_per_worker, steps, warmup, k * envs_per_worker, barrier)
            for k in range(workers)]
    with ctx.Pool(workers) as pool:
        spans = pool.map(_ref_worker, jobs)
    t0 = min(s for s, _ in spans)
    t1 = max(e for _, e in spans)
    envs = envs_per_worker * workers
    return {"env_steps_per_s": envs * steps / (t1 - t0), "seconds": t1 - t0, "envs": envs,
            "steps": steps, "workers": workers, "numpy": np.__version__}


def run_reference_arm(args) -> int:
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    workers = args.cpu_workers or (os.cpu_count() or 1)
    r = cpu_reference_parallel(args.scenario, args.cpu_envs, max(args.steps, 1),
                               max(args.warmup, 1), workers)
    from paper_2602_01665_b200.scenario import builtin_scenario
    sc_units = len(builtin_scenario(SCENARIOS[args.scenario]).units)
    v = r["env_steps_per_s"]
    line = {
        "metric": "env_steps_per_s", "value": v, "unit": "env-steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * r["seconds"] / r["steps"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (scenario JSON, seeded lanes)", "impl": "reference",
        "agent_steps_per_s": v * sc_units,
        "config": {"workload": WORKLOAD[args.scenario], "scenario": SCENARIOS[args.scenario],
                   "envs": r["envs"], "host_processes": workers},
        "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": workers, "kind": "port",
                         "sample": f"{workers} processes x {args.cpu_envs} envs x {r['steps']} "
                                   f"steps (+{max(args.warmup, 1)} warm-up), "
                                   f"oracle/tabx_oracle.py numpy {r['numpy']}"},
        "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Ctx:
    """Rank / device plumbing shared by the measurements."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        # TABX_BENCH_SHARED_GPU=1: a control-flow dry run of the N > 1 path on
        # one GPU (every rank on cuda:0, gloo for the collectives); its timings
        # mean nothing -- the real N > 1 run is one rank per GPU over NCCL
        shared = os.environ.get("TABX_BENCH_SHARED_GPU") == "1"
        if shared:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            if shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        self.stream = torch.cuda.current_stream(self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)


def launches_per_step(per: int) -> int:
    # K1, K2, K3 per step, plus the refresh check and K0 (the
    # heuristic-controller pass) from 4,096 lanes on unless disabled
    k0 = per >= int(os.environ.get("TABX_K0_MIN_ENVS", 4096)) and os.environ.get("TABX_NO_K0") != "1"
    return 3 + (2 if k0 else 0)


def measure_device(cx: Ctx, key: str, per: int, steps: int, warmup: int, seed: int,
                   profile: bool = True, stats: bool = False) -> dict:
    """value (+ roofline): K steps of a resident batch, CUDA-event timed."""
    from paper_2602_01665_b200 import shard
    from paper_2602_01665_b200.rng import lane_seeds
    from paper_2602_01665_b200.scenario import builtin_scenario
    from paper_2602_01665_b200.sim import BatchSim

    torch = cx.torch
    total = per * cx.world
    first, _ = shard.shard_range(total, cx.world, cx.rank)
    sc = builtin_scenario(SCENARIOS[key]).scripted()
    N, Z = sc.max_units, sc.max_zones
    sim = BatchSim([sc] * per, lane_seeds(seed, per, first), auto_reset=True, device=cx.dev,
                   interactions=False, final_observations=(key != "c4"))
    for _ in range(warmup):
        sim.step(None)
    cx.barrier()
    t0, t1 = cx.event(), cx.event()
    with ClockSampler(cx.local) as clk:
        t0.record(cx.stream)
        for _ in range(steps):
            sim.step(None)
        t1.record(cx.stream)
        cx.barrier()
    elapsed_ms = cx.max_over_ranks(t0.elapsed_time(t1))
    out = {"value": total * steps / (elapsed_ms / 1000.0), "unit": "env-steps/s",
           "ms_per_step": elapsed_ms / steps, "steps": steps, "warmup": warmup,
           "agent_steps_per_s": total * steps / (elapsed_ms / 1000.0) * len(sc.units),
           "envs": total, "envs_per_gpu": per, "n_units": N, "n_zones": Z,
           "clocks": clk.summary(), "step_path": sim.step_path(),
           "gpu_launches": {"split": launches_per_step(per), "fused": launches_per_step(per) - 1,
                            "single": 1}[sim.step_path()] * steps}
    if profile:
        # per-kernel times (roofline) from a second pass of the same length with
        # CUDA events around every kernel, so their host cost stays out of `value`
        starts = [cx.event() for _ in range(steps)]
        ends = [cx.event() for _ in range(steps)]
        sim.set_profiling(True)
        for k in range(steps):
            starts[k].record(cx.stream)
            sim.step(None)
            ends[k].record(cx.stream)
        cx.barrier()
        kprof = sim.kernel_profile()
        sim.set_profiling(False)
        kern_ms = statistics.mean(s.elapsed_time(e) for s, e in zip(starts, ends))
        out["roofline"] = roofline(key, N, Z, per, kern_ms, kprof)
    if stats:
        # the one collective: per-window episode statistics, NCCL all-reduce over NVLink
        st = shard.reduce_episode_stats(sim.episode_stats(), device=cx.dev)
        st["summary"] = shard.summarize(st)
        out["episode_stats"] = st
    sim.close()
    del sim
    torch.cuda.empty_cache()
    return out


def roofline(key: str, N: int, Z: int, per: int, kern_ms: float, kprof: dict) -> dict:
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs", 6547.5)
    bytes_per = algorithmic_bytes(N, Z)
    achieved = bytes_per * per / (kern_ms / 1000.0) / 1e9
    D, G = sim_dims(N, Z)
    obs_bytes = 4 * N * D + 4 * G + 57 * N + 5  # writes + the per-unit view it reads
    step_bytes = bytes_per - (4 * N * D + 4 * G)
    kernels = []
    if kprof.get("fused") == "single":
        rows = (("single_kernel (K1 + K2 + K3 of a small batch in one launch: step, observation "
                 "rows, auto-resets)", kprof["single_kernel_ms"], step_bytes + obs_bytes),)
    elif kprof.get("fused"):
        # refresh check + K0 (re-reads of the unit view only), then one fused
        # kernel: the step's state traffic + the observation stream
        rows = (("ctrl_kernels (refresh check + K0 heuristic-controller pass)",
                 kprof["ctrl_kernel_ms"], None),
                ("fused_kernel (K1 actions..rewards, caches, state + K2 observation and "
                 "global-state stream, TMA; warp-specialised)", kprof["fused_kernel_ms"],
                 step_bytes + obs_bytes),
                ("reset_kernel (K3: deferred auto-resets)", kprof["reset_kernel_ms"], None))
    else:
        rows = (("step_kernels (K0 heuristic-controller pass + K1 actions..rewards, "
                 "caches, state)", kprof["step_kernel_ms"], step_bytes),
                ("obs_kernel (K2: observation + global-state stream, TMA)",
                 kprof["obs_kernel_ms"], obs_bytes),
                ("reset_kernel (K3: deferred auto-resets)", kprof["reset_kernel_ms"], None))
    for name, ms, nbytes in rows:
        ent = {"kernel": name, "ms_avg": ms}
        if nbytes and ms > 0:
            gbs = nbytes * per / (ms / 1000.0) / 1e9
            ent.update({"bytes_per_env_step": nbytes, "achieved_gbs": gbs, "frac": gbs / peak})
        if ("obs_kernel" in name or "fused_kernel" in name or "single_kernel" in name) and ms > 0:
            strict = (4 * N * D + 4 * G) * per / (ms / 1000.0) / 1e9
            ent["frac_obs_bytes_only"] = strict / peak
        kernels.append(ent)
    # issue roofline of the latency-bound step kernels: ncu warp-instruction
    # counts per env-step (profiles/instructions_<key>.json) over the measured
    # time, against 4 warp-instructions per SM-cycle at the max SM clock
    ins = os.path.join(ROOT, "profiles", f"instructions_{key}.json")
    if os.path.exists(ins):
        with open(ins) as fh:
            doc = json.load(fh)
        wi = doc["warp_instructions"]
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak_ips = doc["peak_warp_instructions_per_sm_cycle"] * doc["sm_count"] * mhz * 1e6
        for ent in kernels:
            parts = (("K0", "K1") if ent["kernel"].startswith("step_kernels") else
                     ("K2",) if ent["kernel"].startswith("obs_kernel") else ())
            if parts and ent.get("ms_avg"):
                n = sum(wi[p] for p in parts) / doc["envs"] * per
                ent["warp_instructions_per_env_step"] = round(n / per, 1)
                ent["issue_frac"] = n / (ent["ms_avg"] / 1000.0) / peak_ips
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{key}.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("bytes_per_env_step", 0) * per or None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "bytes_per_env_step": bytes_per,
            "kernel_ms_avg": kern_ms,
            "scope": "one step = controller pass + step kernel + observation kernel + reset "
                     "kernel (SURVEY.md 8(d) bytes per env-step x envs / step time)",
            "kernels": kernels,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks
            else "fallback (B200_PROFILING.md)"}


def measure_e2e(cx: Ctx, key: str, per: int, steps: int, warmup: int, seed: int) -> dict:
    """The metric through the trainer API with host buffers (bindings.HostStepper)."""
    import numpy as np

    from paper_2602_01665_b200 import bindings, shard
    from paper_2602_01665_b200.scenario import builtin_scenario, save_scenario

    torch = cx.torch
    total = per * cx.world
    first, _ = shard.shard_range(total, cx.world, cx.rank)
    base = builtin_scenario(SCENARIOS[key])
    N = base.max_units
    doc = save_scenario(base).encode()  # ally external, enemy heuristic-medium
    h = bindings.make_batch(doc, per, seed, device=cx.dev, first_lane=first,
                            interactions=False, final_observations=(key != "c4"))
    gen = np.random.default_rng(1234 + cx.rank)
    pinned = [torch.from_numpy(gen.integers(0, 5, size=(per, N), dtype=np.int64)).pin_memory()
              for _ in range(4)]  # moves/rotate: always legal, no host mask round trip
    # bindings.HostStepper: every step uploads its host actions and downloads
    # its rewards / terminated / truncated through pinned double buffers on
    # copy streams, overlapping the neighbouring steps' kernels; the host
    # consumes step k-1's results while step k runs
    stepper = bindings.HostStepper(h)
    host_sum = 0.0

    def run(n):
        nonlocal host_sum
        prev = None
        for k in range(n):
            t = stepper.submit(pinned[k % len(pinned)])
            if prev is not None:
                rew_h, term_h, trunc_h = stepper.result(prev)
                host_sum += float(rew_h[0, 0]) + int(term_h[0]) + int(trunc_h[0])
            prev = t
        if prev is not None:
            rew_h, term_h, trunc_h = stepper.result(prev)
            host_sum += float(rew_h[0, 0])

    run(warmup)
    cx.barrier()
    e0, e1 = cx.event(), cx.event()
    w0 = time.perf_counter()
    e0.record(cx.stream)
    run(steps)
    e1.record(cx.stream)
    cx.barrier()
    wall = time.perf_counter() - w0
    ms = cx.max_over_ranks(max(e0.elapsed_time(e1), 1000.0 * wall))
    h.sim.close()
    del h, stepper
    torch.cuda.empty_cache()
    return {"value": total * steps / (ms / 1000.0), "unit": "env-steps/s",
            "h2d_bytes_per_step": per * N * 8, "d2h_bytes_per_step": per * N * 4 + 2 * per,
            "steps": steps}


def measure_host_obs(cx: Ctx, key: str, per: int, steps: int, seed: int) -> dict:
    """What a host-side consumer of the reference's numpy outputs pays: each
    step's host actions uploaded, then the float32 observations and the
    action mask copied back to pinned host memory (PCIe bound), with the
    strict (synchronous) action check of bindings.step."""
    import numpy as np

    from paper_2602_01665_b200 import bindings, shard
    from paper_2602_01665_b200.scenario import builtin_scenario, save_scenario

    torch = cx.torch
    total = per * cx.world
    first, _ = shard.shard_range(total, cx.world, cx.rank)
    base = builtin_scenario(SCENARIOS[key])  # ally external, enemy heuristic-medium
    N = base.max_units
    h = bindings.make_batch(save_scenario(base).encode(), per, seed, device=cx.dev,
                            first_lane=first, interactions=False, final_observations=False)
    obs = h.sim.last.observations
    host = torch.empty(obs.shape, dtype=obs.dtype).pin_memory()
    mask_host = torch.empty(h.sim.last.action_mask.shape, dtype=torch.bool).pin_memory()
    gen = np.random.default_rng(99 + cx.rank)
    act_host = torch.from_numpy(gen.integers(0, 5, size=(per, N), dtype=np.int64)).pin_memory()
    act_dev = torch.empty_like(act_host, device=cx.dev)

    def one():
        act_dev.copy_(act_host, non_blocking=True)
        out = bindings.step(h, act_dev)
        host.copy_(out[0], non_blocking=True)
        mask_host.copy_(out[5], non_blocking=True)

    one()
    cx.barrier()
    e0, e1 = cx.event(), cx.event()
    e0.record(cx.stream)
    for _ in range(steps):
        one()
    e1.record(cx.stream)
    cx.barrier()
    ms = cx.max_over_ranks(e0.elapsed_time(e1))
    h.sim.close()
    del h, host, mask_host
    torch.cuda.empty_cache()
    D = obs.shape[2]
    return {"value": total * steps / (ms / 1000.0), "unit": "env-steps/s", "steps": steps,
            "h2d_bytes_per_step": per * N * 8,
            "d2h_bytes_per_step": per * N * (4 * D + 7),
            "note": "host int64 actions in, float32 observations + action mask out to pinned "
                    "host memory every step (the reference's bindings.step returns numpy "
                    "arrays); bound by the PCIe device-to-host link"}


def measure_reconfig(cx: Ctx, batches=(8, 262144)) -> dict:
    from paper_2602_01665_b200.reconfig import reconfiguration_latency
    from paper_2602_01665_b200.scenario import builtin_scenario

    out = {"protocol": "rollout.py:422-448 (100 distinct scenarios through reset_env(i % "
                       "lanes, config_i, seed=i), a step after each); gate: worst < 10 ms "
                       "(pkg/tests/test_acceptance.py:425-433); times to completion (host call "
                       "+ stream synchronise)"}
    for b in batches:
        r = reconfiguration_latency(builtin_scenario(SCENARIOS["c3"]), count=100, batch=b,
                                    device=cx.local)
        out[f"batch_{b}"] = {"worst_ms": 1000 * max(r["times"]),
                             "mean_ms": 1000 * statistics.mean(r["times"]),
                             "host_call_mean_ms": 1000 * statistics.mean(r["host_times"]),
                             "config_rows": r["config_rows"]}
        cx.torch.cuda.empty_cache()
    return out


def run_gpu_arm(args) -> int:
    cx = Ctx()
    key = args.scenario
    per = args.envs or DEFAULT_ENVS[key]
    total = per * cx.world
    from paper_2602_01665_b200.scenario import builtin_scenario
    sc = builtin_scenario(SCENARIOS[key]).scripted()
    N, Z = sc.max_units, sc.max_zones

    # ---------------- headline: device-resident throughput (value + roofline)
    head = measure_device(cx, key, per, args.steps, args.warmup, args.seed, stats=True)
    # ---------------- end-to-end through the trainer API with host buffers
    e2e = None if args.no_e2e else measure_e2e(cx, key, per, args.steps, args.warmup, args.seed)

    # ---------------- the other BASELINE configs, each timed the same way
    extras = {}
    for k in [c for c in args.configs.split(",") if c and c != key]:
        p = DEFAULT_ENVS[k]
        m = measure_device(cx, k, p, args.steps, args.warmup, args.seed)
        if not args.no_e2e:
            m["e2e"] = measure_e2e(cx, k, p, args.steps, args.warmup, args.seed)
        m["workload"] = WORKLOAD[k]
        extras[k] = m
    # ---------------- a whole episode of the headline config: t = 1..K,
    # across the lockstep truncation at t = 400 (every lane auto-resets, the
    # next step refreshes every cache)
    episode = None
    if args.episode_steps > 0:
        episode = measure_device(cx, key, per, args.episode_steps, 0, args.seed, profile=False)
        episode["window"] = (f"t = 1..{args.episode_steps} from the episode start (no warm-up), "
                             "including the lockstep t = 400 truncation + auto-reset")
    host_obs = None
    if args.host_obs_steps > 0:
        host_obs = measure_host_obs(cx, key, per, args.host_obs_steps, args.seed)
    reconfig = measure_reconfig(cx) if args.reconfig and cx.world == 1 else None

    # ---------------- C5: full rollout loop (policy + step + auto-reset), CUDA graph
    c5 = None
    if args.rollout_envs > 0:
        from paper_2602_01665_b200 import shard
        from paper_2602_01665_b200.rollout import Rollout
        base = builtin_scenario(SCENARIOS[key])
        r_total = args.rollout_envs * cx.world
        r_first, r_per = shard.shard_range(r_total, cx.world, cx.rank)
        ro = Rollout(base, r_per, horizon=args.horizon, policy=args.policy, device=cx.local,
                     seed=args.seed, first_lane=r_first)
        ro.run()  # capture + first horizon
        cx.barrier()
        r0, r1 = cx.event(), cx.event()
        r0.record(cx.stream)
        for _ in range(args.rollout_iters):
            ro.run()
        r1.record(cx.stream)
        cx.barrier()
        r_ms = cx.max_over_ranks(r0.elapsed_time(r1))
        c5 = {"value": r_total * args.horizon * args.rollout_iters / (r_ms / 1000.0),
              "unit": "env-steps/s", "envs": r_total, "horizon": args.horizon,
              "policy": args.policy, "iterations": args.rollout_iters,
              "ms_per_horizon": r_ms / args.rollout_iters,
              "note": "policy forward + masked sampling + batched step + auto-reset, whole "
                      "horizon in one CUDA graph; observations written in place into the "
                      "[T+1,B,N,D] horizon buffer"}
        if ro.policy is not None:
            # the rollout's policy kernel alone (tcgen05 MLP + fused masked
            # sampler, tabx_policy_mlp_sample) on the rollout's own input and
            # mask: HBM-bound, x read once, mask in, action + log-prob out
            import ctypes as _ct
            from paper_2602_01665_b200 import _native as _nat
            pol, xin = ro.policy, ro._xin
            rows = xin.shape[0] * xin.shape[1]
            mask = ro.sim._buf["action_mask"]
            act, lp = ro.buf.actions[0], ro.buf.logp[0]
            ptr = lambda t: _ct.c_void_p(t.data_ptr())  # noqa: E731
            lib = _nat.lib()

            def _pol():
                lib.tabx_policy_mlp_sample(
                    ptr(xin), rows, pol.in_dim, pol.in_dim, ptr(pol.l1.weight),
                    ptr(pol.l1.bias), ptr(pol.l2.weight), ptr(pol.l2.bias), None, ptr(mask),
                    _ct.c_uint64(0), None, 0, ptr(act), ptr(lp),
                    _ct.c_void_p(cx.stream.cuda_stream))
            for _ in range(3):
                _pol()
            m0, m1 = cx.event(), cx.event()
            m0.record(cx.stream)
            for _ in range(20):
                _pol()
            m1.record(cx.stream)
            cx.stream.synchronize()
            mlp_ms = m0.elapsed_time(m1) / 20
            mlp_bytes = rows * (pol.in_dim * 2 + 7 + 8 + 4)
            peak = load_peaks().get("hbm_gbs", 6547.5)
            c5["policy_mlp"] = {
                "kernel": "mlp_policy_tma_kernel (tcgen05.mma M128 N128 K16, TMA 128B-swizzled "
                          "boxes, TMEM accumulators) with the masked sampler in its epilogue",
                "us_avg": round(mlp_ms * 1000.0, 2), "rows": rows, "k": pol.in_dim,
                "bound": "hbm", "achieved_gbps": round(mlp_bytes / (mlp_ms / 1000.0) / 1e9, 1),
                "peak_gbps": peak, "frac": round(mlp_bytes / (mlp_ms / 1000.0) / 1e9 / peak, 3),
                "algorithmic_bytes": mlp_bytes}
        ro.close()
        del ro
        cx.torch.cuda.empty_cache()

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if cx.rank == 0 and cx.world == 1 and not args.no_cpu:
        r = cpu_reference(key, args.cpu_envs, args.cpu_steps, 1)
        cpu = {"value": r["env_steps_per_s"], "unit": "env-steps/s", "cores": 1, "kind": "port",
               "sample": f"{r['envs']} envs x {r['steps']} steps (+1 warm-up), "
                         f"oracle/tabx_oracle.py numpy {r['numpy']}, {r['seconds']:.1f} s"}

    if cx.rank == 0:
        D, G = sim_dims(N, Z)
        line = {
            "metric": "env_steps_per_s", "value": head["value"], "unit": "env-steps/s",
            "n_gpus": cx.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (scenario JSON, seeded lanes)",
            "agent_steps_per_s": head["agent_steps_per_s"],
            "config": {"workload": WORKLOAD[key], "scenario": SCENARIOS[key],
                       "envs": total, "envs_per_gpu": per, "n_units": N, "n_zones": Z,
                       "obs_dim": D, "global_dim": G,
                       "parallelism": f"env-shard x{cx.world}",
                       "l2": "inputs larger than L2: every step writes "
                             f"{4 * N * D * per / 1e9:.1f} GB of observations",
                       "e2e_workload": "bindings.HostStepper (one step per call, K steps), "
                                       "ally external: int64 actions H2D from pinned host "
                                       "and rewards/terminated/truncated D2H every step, "
                                       "copies overlapped with the neighbouring steps; "
                                       "observations and action masks stay on the device "
                                       "(a GPU policy reads them in place; host_obs_e2e "
                                       "prices copying them out)"},
            "roofline": head["roofline"],
            "e2e": e2e,
            "gpu_launches": head["gpu_launches"], "step_path": head.get("step_path"),
            "clocks": head["clocks"],
            "episode_stats": head["episode_stats"],
        }
        for k, m in extras.items():
            line[k] = m
        if episode is not None:
            line["c3_episode" if key == "c3" else f"{key}_episode"] = episode
        if host_obs is not None:
            line["host_obs_e2e"] = host_obs
        if reconfig is not None:
            line["reconfig"] = reconfig
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if c5 is not None:
            line["rollout_c5"] = c5
        print(json.dumps(line), flush=True)
    if cx.world > 1:
        cx.dist.destroy_process_group()
    return 0


def sim_dims(N, Z):
    return 15 + 17 * (N - 1) + 8 * Z, 15 * N + 8 * Z


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("tabx", "reference"), default="tabx")
    ap.add_argument("--scenario", choices=sorted(SCENARIOS), default="c3")
    ap.add_argument("--envs", type=int, default=0,
                    help="environments per GPU (weak scaling: the job runs n_gpus x envs)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--configs", default="c1,c2,c4",
                    help="other BASELINE configs timed in the same run (comma list)")
    ap.add_argument("--episode-steps", type=int, default=410,
                    help="whole-episode window of the headline config (0 = skip)")
    ap.add_argument("--host-obs-steps", type=int, default=3,
                    help="steps of the host-observation e2e variant (0 = skip)")
    ap.add_argument("--no-reconfig", dest="reconfig", action="store_false")
    ap.add_argument("--cpu-envs", type=int, default=1024)
    ap.add_argument("--cpu-steps", type=int, default=100)
    ap.add_argument("--cpu-workers", type=int, default=0, help="reference arm processes (0 = all cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rollout-envs", type=int, default=16384,
                    help="C5 rollout loop envs per GPU (0 = skip)")
    ap.add_argument("--horizon", type=int, default=128)
    ap.add_argument("--policy", choices=("random", "mlp"), default="mlp")
    ap.add_argument("--rollout-iters", type=int, default=2)
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
