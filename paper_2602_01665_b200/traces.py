"""Episode traces, replay and trace-driven summaries on the GPU engine.

SURVEY.md §8(f) rank 3.  Mirrors ``pkg/src/skirmish/rollout.py``:

* ``parse_policy`` / ``apply_policies`` (``rollout.py:37-69``): ``random``,
  ``heuristic:<tier>``, ``replay:<trace>`` (replayed teams become external);
* ``ReplayBook`` (``:72-109``): recorded actions indexed by (episode, step);
* ``EpisodeStats`` / ``summarize`` (``:112-147``) and ``summary_from_trace``
  (``:322-345``), the same float accumulation order;
* ``record_line`` and the record layout of ``_build_record`` (``:150-188``);
* ``run_rollouts`` (``:271-319``) with ``_run_chunk``'s lane scheduling
  (``:200-268``): ``batch`` lanes pull episodes from a queue, a finished
  lane is restarted with ``reset_env(b, seed=derive_seed(seed, e,
  TAG_EPISODE))``, and records are emitted grouped by episode in index order,
  so trace bytes depend only on (scenario, policies, episodes, seed, batch,
  threads) exactly as the reference's do.

The simulation runs on the device (``sim.BatchSim``); per step, the traced
lanes' post-step state is gathered on the device by ``tabx_export_lanes`` and
copied to the host together with the step outputs the record needs (executed
actions, dense reward, flags, outcome codes).  ``TraceStream`` is the same
gather for a sampled subset of a large training batch, double-buffered into
pinned host memory so the copy overlaps the next step.
"""
from __future__ import annotations

import json
import math
from collections import deque
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .rng import TAG_EPISODE, derive_seed
from .scenario import HEURISTIC_TIERS, Scenario
from .template import build_config

POLICY_KINDS = ("random", "heuristic", "replay")
TEAM_ALLY, TEAM_ENEMY = 0, 1
REASON_NAMES = {1: "elimination", 2: "truncation", 3: "truncation_tie"}
TRACE_FIELDS = ("pos", "heading", "health", "alive", "cooldown", "reveal", "t", "done",
                "winner", "reason", "first_kill")
OUT_FIELDS = ("actions", "dense_reward", "episode_length", "terminated", "truncated", "done",
              "winner", "episode_return")


def parse_policy(text: str):
    """random | heuristic:<tier> | replay:<trace path> (rollout.py:37-51)."""
    if text == "random":
        return "random", None
    kind, sep, arg = text.partition(":")
    if kind == "heuristic" and sep:
        if arg not in HEURISTIC_TIERS:
            known = ", ".join(sorted(HEURISTIC_TIERS))
            raise ValueError(f"unknown heuristic tier {arg!r} (expected one of {known})")
        return "heuristic", HEURISTIC_TIERS[arg]
    if kind == "replay" and sep and arg:
        return "replay", arg
    raise ValueError(f"unknown policy {text!r}")


def apply_policies(config: Scenario, ally: str, enemy: str):
    """Controllers overridden by policy specs; replay teams come back as
    external plus team id -> trace path (rollout.py:54-69)."""
    replays: dict[int, str] = {}
    specs = {}
    for team_id, spec in ((TEAM_ALLY, ally), (TEAM_ENEMY, enemy)):
        kind, arg = parse_policy(spec)
        if kind == "replay":
            replays[team_id] = str(arg)
            specs[team_id] = "external"
        elif kind == "heuristic":
            tier = spec.split(":", 1)[1]
            specs[team_id] = f"heuristic:{tier}"
        else:
            specs[team_id] = "random"
    return config.with_controllers(ally=specs[TEAM_ALLY], enemy=specs[TEAM_ENEMY]), replays


class ReplayBook:
    """Recorded actions from a trace file, indexed by (episode, step)."""

    def __init__(self, path: str, episodes: list[np.ndarray]) -> None:
        self.path = path
        self.episodes = episodes

    @classmethod
    def load(cls, path: str) -> "ReplayBook":
        episodes: list = []
        current = None
        with open(path, encoding="utf-8") as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                rec = json.loads(line)
                if rec["t"] == 1:
                    current = []
                    episodes.append(current)
                if current is None:
                    raise ValueError(f"{path}: trace does not start at t=1")
                current.append([u["action"] for u in rec["units"]])
        return cls(path, [np.asarray(e, dtype=np.int64) for e in episodes])

    def actions(self, episode: int, t: int) -> np.ndarray:
        if episode >= len(self.episodes):
            raise ValueError(f"{self.path}: replay holds {len(self.episodes)} episodes,"
                             f" episode {episode} requested")
        steps = self.episodes[episode]
        if not 1 <= t <= len(steps):
            raise ValueError(f"{self.path}: episode {episode} ends at step {len(steps)},"
                             f" step {t} requested")
        return steps[t - 1]


@dataclass(frozen=True)
class EpisodeStats:
    episode: int
    winner: int
    reason: str
    length: int
    episode_return: float
    first_kill_team: int | None


def summarize(stats: list[EpisodeStats]) -> dict:
    """rollout.py:122-147 (same summation order, so bit-identical)."""
    n = len(stats)
    if n == 0:
        return {"episodes": 0, "win_rate": 0.0, "mean_return": 0.0, "mean_length": 0.0,
                "first_kill_rate": 0.0}
    wins = sum(1 for s in stats if s.winner == TEAM_ALLY)
    first = sum(1 for s in stats if s.first_kill_team == TEAM_ALLY)
    total_return = 0.0
    total_length = 0
    for s in stats:
        total_return += s.episode_return
        total_length += s.length
    return {"episodes": n, "win_rate": wins / n, "mean_return": total_return / n,
            "mean_length": total_length / n, "first_kill_rate": first / n}


def record_line(rec: dict) -> str:
    return json.dumps(rec, sort_keys=True, separators=(",", ":")) + "\n"


def summary_from_trace(path) -> dict:
    """Rebuild the rollout summary from a trace file alone (rollout.py:322-345)."""
    stats: list[EpisodeStats] = []
    acc = 0.0
    with open(path, encoding="utf-8") as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            rec = json.loads(line)
            if rec["t"] == 1:
                acc = 0.0
            acc += rec["reward"]
            if "outcome" in rec:
                o = rec["outcome"]
                stats.append(EpisodeStats(episode=len(stats), winner=o["winner"],
                                          reason=o["reason"], length=o["episode_length"],
                                          episode_return=acc,
                                          first_kill_team=o["first_kill_team"]))
    return summarize(stats)


class RecordBuilder:
    """Trace records of one scenario from gathered lane rows (rollout.py:150-188)."""

    def __init__(self, config: Scenario):
        cfg = build_config(config, validate=False)
        N = config.max_units
        self.n_units = len(config.units)
        self.team = np.array([cfg.team[i] for i in range(N)], np.int64)
        self.active = np.array([bool(cfg.active[i]) for i in range(N)])
        self.max_h = np.array([cfg.max_health[i] for i in range(N)], np.float64)

    def _ratio(self, health: np.ndarray, team: int) -> float:
        # arrays.py:390-394 on a one-lane batch (numpy pairwise row sum)
        members = (self.active & (self.team == team))[None, :]
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = np.where(members, health[None, :] / self.max_h[None, :], 0.0)
        count = members.sum(axis=1)
        return float((ratio.sum(axis=1) / np.maximum(count, 1))[0])

    def record(self, st: dict, out: dict, k: int, b: int) -> dict:
        """Row k of the gathered state ``st``, lane b of the step outputs ``out``."""
        final = bool(out["done"][b])
        units = []
        for i in range(self.n_units):
            units.append({
                "id": i,
                "team": int(self.team[i]),
                "position": [float(st["pos"][k, i, 0]), float(st["pos"][k, i, 1])],
                "heading": math.degrees(float(st["heading"][k, i])),
                "health": float(st["health"][k, i]),
                "alive": bool(st["alive"][k, i]),
                "action": int(out["actions"][b, i]),
                "cooldown_timer": float(st["cooldown"][k, i]),
                "reveal_timer": float(st["reveal"][k, i]),
            })
        reward = float(out["dense_reward"][b])
        if final:
            reward += 1.0 if int(out["winner"][b]) == TEAM_ALLY else -1.0
        rec = {"t": int(out["episode_length"][b]), "units": units, "reward": reward,
               "terminated": bool(out["terminated"][b]), "truncated": bool(out["truncated"][b])}
        if final:
            fk = int(st["first_kill"][k])
            rec["outcome"] = {
                "winner": int(st["winner"][k]),
                "reason": REASON_NAMES[int(st["reason"][k])],
                "ally_health_ratio": self._ratio(st["health"][k], TEAM_ALLY),
                "enemy_health_ratio": self._ratio(st["health"][k], TEAM_ENEMY),
                "episode_length": int(st["t"][k]),
                "first_kill_team": None if fk < 0 else fk,
            }
        return rec

    def stats(self, st: dict, out: dict, k: int, b: int, episode: int) -> EpisodeStats:
        fk = int(st["first_kill"][k])
        return EpisodeStats(episode=episode, winner=int(st["winner"][k]),
                            reason=REASON_NAMES[int(st["reason"][k])], length=int(st["t"][k]),
                            episode_return=float(out["episode_return"][b]),
                            first_kill_team=None if fk < 0 else fk)


class GpuEngine:
    """The run loop's view of a device BatchSim: step, gather, reset."""

    def __init__(self, configs, seeds, device=None):
        import torch

        from .sim import BatchSim
        self._torch = torch
        self.sim = BatchSim(configs, seeds, auto_reset=False, device=device,
                            interactions=False, final_observations=False)
        self.lanes = torch.arange(self.sim.batch, dtype=torch.int64, device=self.sim.device)

    def step(self, actions):
        out = self.sim.step(actions)
        st = self.sim.export_lanes(self.lanes, TRACE_FIELDS)
        host = {k: v.cpu().numpy() for k, v in st.items()}
        outs = {k: getattr(out, k).cpu().numpy() for k in OUT_FIELDS}
        return outs, host

    def reset_env(self, b: int, seed: int) -> None:
        self.sim.reset_env(b, seed=seed)

    def close(self) -> None:
        self.sim.close()


def _run_chunk(config, ep_ids, run_seed, batch, keep_records, replays, engine_factory):
    results: dict = {}
    if not ep_ids:
        return results
    books = {team: ReplayBook.load(path) for team, path in replays.items()}
    for book in books.values():
        if len(book.episodes) <= max(ep_ids):
            raise ValueError(f"{book.path}: replay holds {len(book.episodes)} episodes,"
                             f" {max(ep_ids) + 1} needed")
    team_slots = {team: [i for i, u in enumerate(config.units) if u.team == team]
                  for team in books}
    queue = deque(ep_ids)
    lanes = min(max(1, batch), len(ep_ids))
    lane_ep: list = []
    seeds = []
    for _ in range(lanes):
        e = queue.popleft()
        lane_ep.append(e)
        seeds.append(derive_seed(run_seed, e, TAG_EPISODE))
    eng = engine_factory([config] * lanes, np.array(seeds, dtype=np.uint64))
    builder = RecordBuilder(config)
    N = config.max_units
    t_lane = [0] * lanes  # s.t of each lane (0 after a spawn)
    buffers: dict = {e: [] for e in ep_ids}
    try:
        while any(e is not None for e in lane_ep):
            actions = None
            if books:
                actions = np.zeros((lanes, N), dtype=np.int64)
                for b, e in enumerate(lane_ep):
                    if e is None:
                        continue
                    for team, book in books.items():
                        row = book.actions(e, t_lane[b] + 1)
                        for i in team_slots[team]:
                            actions[b, i] = row[i]
            out, st = eng.step(actions)
            for b in range(lanes):
                t_lane[b] = int(st["t"][b])
                e = lane_ep[b]
                if e is None:
                    continue
                final = bool(out["done"][b])
                if keep_records:
                    buffers[e].append(record_line(builder.record(st, out, b, b)))
                if not final:
                    continue
                results[e] = (builder.stats(st, out, b, b, e), buffers.pop(e))
                if queue:
                    nxt = queue.popleft()
                    lane_ep[b] = nxt
                    eng.reset_env(b, derive_seed(run_seed, nxt, TAG_EPISODE))
                    t_lane[b] = 0
                else:
                    lane_ep[b] = None
    finally:
        eng.close()
    return results


def run_rollouts(config: Scenario, ally: str = "heuristic:medium",
                 enemy: str = "heuristic:medium", episodes: int = 1, seed: int = 0, trace=None,
                 threads: int = 1, batch: int = 1, device=None, engine_factory=None) -> dict:
    """Play episodes and return the summary; optionally write the JSONL trace
    (rollout.py:271-319).  ``threads`` splits the episodes into the same
    chunks as the reference (episode k goes to chunk k mod threads, one
    BatchSim each); the chunks run one after another on the device.
    ``engine_factory(configs, seeds)`` overrides the device engine (tests
    drive the CPU oracle through it)."""
    config, replays = apply_policies(config, ally, enemy)
    keep = trace is not None
    if episodes <= 0:
        if keep:
            Path(trace).write_text("", encoding="utf-8")
        return summarize([])
    factory = engine_factory or (lambda cfgs, seeds: GpuEngine(cfgs, seeds, device=device))
    ep_ids = list(range(episodes))
    threads = max(1, min(threads, episodes))
    merged: dict = {}
    for k in range(threads):
        merged.update(_run_chunk(config, ep_ids[k::threads], seed, batch, keep, replays, factory))
    stats = [merged[e][0] for e in range(episodes)]
    if keep:
        with open(trace, "w", encoding="utf-8", newline="\n") as f:
            for e in range(episodes):
                f.writelines(merged[e][1])
    return summarize(stats)


class TraceStream:
    """Device -> host trace of sampled lanes of a running batch.

    Each :meth:`capture` (after a step) gathers the sampled lanes' state and
    the step outputs the record needs into device buffers, then copies them
    on a side stream into one of two pinned host slots; :meth:`records`
    turns a completed slot into JSONL records.  The copy overlaps the next
    step; the gather is one small kernel on the simulator's stream.
    """

    def __init__(self, sim, lanes, config: Scenario):
        import torch
        self._torch = torch
        self.sim = sim
        self.lanes = torch.as_tensor(np.asarray(lanes, dtype=np.int64), device=sim.device)
        self.builder = RecordBuilder(config)
        self.copy_stream = torch.cuda.Stream(sim.device)
        self._slots = [None, None]
        self._events = [None, None]
        self._next = 0

    def capture(self) -> int:
        """Queue the gather + D2H copy of the current step; returns the slot."""
        torch = self._torch
        st = self.sim.export_lanes(self.lanes, TRACE_FIELDS)
        out = self.sim.last
        dev = {f"s_{k}": v for k, v in st.items()}
        for k in OUT_FIELDS:
            dev[f"o_{k}"] = getattr(out, k).index_select(0, self.lanes)
        slot = self._next
        self._next ^= 1
        if self._events[slot] is not None:
            self._events[slot].synchronize()
        host = self._slots[slot]
        if host is None:
            host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
                    for k, v in dev.items()}
            self._slots[slot] = host
        self.copy_stream.wait_stream(torch.cuda.current_stream(self.sim.device))
        with torch.cuda.stream(self.copy_stream):
            for k, v in dev.items():
                v.record_stream(self.copy_stream)
                host[k].copy_(v, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self._events[slot] = ev
        return slot

    def records(self, slot: int) -> list[dict]:
        """Records of the sampled lanes for a captured slot (waits for its copy)."""
        self._events[slot].synchronize()
        host = self._slots[slot]
        st = {k[2:]: v.numpy() for k, v in host.items() if k.startswith("s_")}
        out = {k[2:]: v.numpy() for k, v in host.items() if k.startswith("o_")}
        return [self.builder.record(st, out, k, k) for k in range(len(self.lanes))]
