"""Helpers comparing the CUDA BatchSim with the numpy oracle, step by step."""
from __future__ import annotations

import numpy as np

STATE_F64 = ("pos", "heading", "vel", "imp_dv", "health", "cooldown", "reveal", "prev_gap",
             "ep_return", "mem_pos")
STATE_EXACT = ("episode", "t", "alive", "done", "terminated", "truncated", "winner", "reason",
               "first_kill", "mem_valid", "vis", "atk")


def to_np(t):
    return None if t is None else t.detach().cpu().numpy()


def compare_outputs(gpu_out, ora: dict, where: str, check_final: bool = True) -> list[str]:
    """Return a list of mismatch descriptions (empty when identical).

    Floats are compared by value (signed zeros are equal); float32 outputs
    against the float64 oracle rounded to float32.
    """
    bad = []

    def cmp(name, g, o):
        if g is None:
            return
        if g.shape != o.shape:
            bad.append(f"{where}: {name} shape {g.shape} vs {o.shape}")
            return
        if g.dtype.kind == "f":
            eq = (g == o) | (np.isnan(g) & np.isnan(o))
        else:
            eq = g == o
        if not np.all(eq):
            idx = np.argwhere(~eq)[0]
            bad.append(f"{where}: {name} differs at {tuple(idx)}: gpu {g[tuple(idx)]!r} "
                       f"oracle {o[tuple(idx)]!r} ({int((~eq).sum())} elements)")

    cmp("observations", to_np(gpu_out.observations), ora["observations"].astype(np.float32))
    cmp("global_state", to_np(gpu_out.global_state), ora["global_state"].astype(np.float32))
    cmp("rewards", to_np(gpu_out.rewards), ora["rewards"].astype(np.float32))
    cmp("action_mask", to_np(gpu_out.action_mask), ora["action_mask"])
    for k in ("terminated", "truncated", "done", "dense_reward", "actions", "winner", "reason",
              "first_kill", "episode_return", "episode_length"):
        cmp(k, to_np(getattr(gpu_out, k)), np.asarray(ora[k]))
    if gpu_out.interactions is not None:
        cmp("interactions", to_np(gpu_out.interactions), ora["interactions"])
    if check_final:
        fo = gpu_out.final_observations
        if (fo is None) != (ora["final_observations"] is None):
            bad.append(f"{where}: final_observations presence differs")
        elif fo is not None:
            cmp("final_observations", to_np(fo), ora["final_observations"].astype(np.float32))
            cmp("final_global_state", to_np(gpu_out.final_global_state),
                ora["final_global_state"].astype(np.float32))
    return bad


def compare_state(gpu_state: dict, sim, where: str) -> list[str]:
    bad = []
    for k in STATE_F64 + STATE_EXACT:
        g = to_np(gpu_state[k])
        o = np.asarray(getattr(sim, k))
        if g.shape != o.shape:
            bad.append(f"{where}: state {k} shape {g.shape} vs {o.shape}")
            continue
        eq = g == o
        if not np.all(eq):
            idx = np.argwhere(~eq)[0]
            bad.append(f"{where}: state {k} differs at {tuple(idx)}: gpu {g[tuple(idx)]!r} "
                       f"oracle {o[tuple(idx)]!r}")
    g = to_np(gpu_state["seed"]).view(np.uint64)
    if not np.array_equal(g, sim.seed):
        bad.append(f"{where}: state seed differs")
    return bad


def oracle_state_dict(sim) -> dict:
    """Oracle state in the import_state layout."""
    keys = ("seed", "episode", "t") + STATE_F64 + ("alive", "done", "terminated", "truncated",
                                                   "winner", "reason", "first_kill", "mem_valid",
                                                   "vis", "atk")
    return {k: np.ascontiguousarray(getattr(sim, k)) for k in keys}
