"""``BatchSim`` on the GPU: the reference's batched simulator API over the C ABI.

Mirrors ``pkg/src/skirmish/environment.py:463-519``:

* ``BatchSim(configs, seeds, auto_reset=False)`` builds one lane per config,
* ``.step(actions=None) -> BatchOutput`` advances every lane,
* ``.reset_env(b, config=None, seed=None)`` restarts lane ``b``,
* ``.last`` is the latest ``BatchOutput``, ``.configs``, ``.batch``.

Outputs are torch tensors on the simulator's CUDA device, written in place
into persistent buffers (the next ``step`` overwrites them; clone to keep).
Observations, global state and rewards are float32 — the float64 values of
the reference rounded to nearest — the rest keeps the reference's dtypes.
``ActionMaskError`` is raised synchronously before any lane is mutated
(``strict=True``, the default); with ``strict=False`` the step is fully
asynchronous (CUDA-Graph capturable) and :meth:`check_errors` raises later.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .scenario import ActionMaskError, Scenario, ensure_valid
from .template import build_config

STATE_DTYPES = {
    "seed": (torch.int64, ()),  # uint64 bits
    "episode": (torch.int64, ()),
    "t": (torch.int64, ()),
    "pos": (torch.float64, (2,)),
    "heading": (torch.float64, ()),
    "vel": (torch.float64, (2,)),
    "imp_dv": (torch.float64, (2,)),
    "health": (torch.float64, ()),
    "cooldown": (torch.float64, ()),
    "reveal": (torch.float64, ()),
    "alive": (torch.bool, ()),
    "prev_gap": (torch.float64, ()),
    "ep_return": (torch.float64, ()),
    "done": (torch.bool, ()),
    "terminated": (torch.bool, ()),
    "truncated": (torch.bool, ()),
    "winner": (torch.int64, ()),
    "reason": (torch.int64, ()),
    "first_kill": (torch.int64, ()),
    "mem_pos": (torch.float64, (2,)),
    "mem_valid": (torch.bool, ()),
    "vis": (torch.bool, ("N",)),
    "atk": (torch.bool, ("N",)),
    "config": (torch.int32, ()),
}
PER_LANE = {"seed", "episode", "t", "prev_gap", "ep_return", "done", "terminated", "truncated",
            "winner", "reason", "first_kill", "config"}


@dataclass
class BatchOutput:
    """environment.py:113-136, as device tensors."""

    observations: torch.Tensor
    global_state: torch.Tensor
    rewards: torch.Tensor
    action_mask: torch.Tensor
    terminated: torch.Tensor
    truncated: torch.Tensor
    done: torch.Tensor
    dense_reward: torch.Tensor
    actions: torch.Tensor
    interactions: torch.Tensor | None
    winner: torch.Tensor
    reason: torch.Tensor
    first_kill: torch.Tensor
    episode_return: torch.Tensor
    episode_length: torch.Tensor
    reset_mask: torch.Tensor
    _final_obs: torch.Tensor | None = None
    _final_glob: torch.Tensor | None = None
    _auto_reset: bool = False

    @property
    def any_reset(self) -> bool:
        return bool(self._auto_reset and self.reset_mask.any().item())

    @property
    def final_observations(self) -> torch.Tensor | None:
        """Terminal observations of auto-reset lanes, others = observations."""
        if not self.any_reset:
            return None
        return torch.where(self.reset_mask[:, None, None], self._final_obs, self.observations)

    @property
    def final_global_state(self) -> torch.Tensor | None:
        if not self.any_reset:
            return None
        return torch.where(self.reset_mask[:, None], self._final_glob, self.global_state)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ct.c_void_p(t.data_ptr())


class BatchSim:
    def __init__(self, configs: list[Scenario], seeds, auto_reset: bool = False,
                 device: int | str | torch.device | None = None, strict: bool = True,
                 interactions: bool = True, final_observations: bool = True,
                 stream: torch.cuda.Stream | None = None):
        if not configs:
            raise ValueError("need at least one environment")
        L = nat.lib()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("BatchSim runs on a CUDA device only")
        self.dev_index = self.device.index if self.device.index is not None else 0
        seen = {id(c): c for c in configs}
        for c in seen.values():
            ensure_valid(c)
        self.configs = list(configs)
        self.auto_reset = bool(auto_reset)
        self.strict = strict
        self.batch = len(configs)
        self.n_units = configs[0].max_units
        self.n_zones = configs[0].max_zones
        for c in configs[1:]:
            if (c.max_units, c.max_zones) != (self.n_units, self.n_zones):
                raise ValueError(
                    "batched environments must share max_units and max_zones; "
                    f"got ({c.max_units}, {c.max_zones}) vs ({self.n_units}, {self.n_zones})")
        self.obs_dim = int(L.tabx_obs_dim(self.n_units, self.n_zones))
        self.global_dim = int(L.tabx_global_dim(self.n_units, self.n_zones))
        # distinct configs (by content: equal templates share a slot) -> table
        built: dict[int, int] = {}
        by_bytes: dict[bytes, int] = {}
        table = []
        lane_cfg = np.zeros(self.batch, np.int32)
        for b, c in enumerate(configs):
            k = built.get(id(c))
            if k is None:
                row = build_config(c, validate=False)
                k = by_bytes.setdefault(bytes(row), len(table))
                if k == len(table):
                    table.append(row)
                built[id(c)] = k
            lane_cfg[b] = k
        # the config-table slot every lane runs on (the C side's mirror)
        self.lane_slots = lane_cfg.copy()
        arr = (nat.TabxConfig * len(table))(*table)
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(self.batch))
        self._stream = stream or torch.cuda.current_stream(self.device)
        # a caller-given stream other than the current one needs cross-stream
        # ordering on every call (see _consume / _publish)
        self._side_stream = stream is not None
        h = ct.c_void_p()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_create(arr, len(table), lane_cfg.ctypes.data_as(ct.c_void_p),
                                    seeds.ctypes.data_as(ct.c_void_p), self.batch,
                                    int(self.auto_reset), self.dev_index,
                                    ct.c_void_p(self._stream.cuda_stream), ct.byref(h)),
                      "tabx_create")
        self._h = h
        self._alloc_outputs(interactions, final_observations)
        self._init_output()

    # ------------------------------------------------------------ buffers --
    def _alloc_outputs(self, interactions: bool, final_obs: bool) -> None:
        B, N, D, G = self.batch, self.n_units, self.obs_dim, self.global_dim
        dev = self.device
        e = lambda *s, dt: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
        self._buf = {
            "observations": e(B, N, D, dt=torch.float32),
            "global_state": e(B, G, dt=torch.float32),
            "rewards": e(B, N, dt=torch.float32),
            "action_mask": e(B, N, nat.NUM_ACTIONS, dt=torch.bool),
            "terminated": e(B, dt=torch.bool),
            "truncated": e(B, dt=torch.bool),
            "done": e(B, dt=torch.bool),
            "dense_reward": e(B, dt=torch.float64),
            "actions": e(B, N, dt=torch.int64),
            "interactions": e(B, N, N, dt=torch.bool) if interactions else None,
            "winner": e(B, dt=torch.int64),
            "reason": e(B, dt=torch.int64),
            "first_kill": e(B, dt=torch.int64),
            "episode_return": e(B, dt=torch.float64),
            "episode_length": e(B, dt=torch.int64),
            "final_observations": e(B, N, D, dt=torch.float32) if final_obs else None,
            "final_global_state": e(B, G, dt=torch.float32) if final_obs else None,
            "reset_mask": e(B, dt=torch.bool),
        }
        self._outs = nat.TabxOutputs(*[_ptr(self._buf[k]) for k in nat.OUTPUT_FIELDS])
        self._outs_ref = ct.byref(self._outs)
        self._step_fn = nat.lib().tabx_step

    def _output(self) -> BatchOutput:
        # the buffers are persistent and BatchOutput derives final_* on
        # access, so one view object serves every step
        cached = getattr(self, "_out_view", None)
        if cached is not None:
            return cached
        b = self._buf
        self._out_view = BatchOutput(
            observations=b["observations"], global_state=b["global_state"], rewards=b["rewards"],
            action_mask=b["action_mask"], terminated=b["terminated"], truncated=b["truncated"],
            done=b["done"], dense_reward=b["dense_reward"], actions=b["actions"],
            interactions=b["interactions"], winner=b["winner"], reason=b["reason"],
            first_kill=b["first_kill"], episode_return=b["episode_return"],
            episode_length=b["episode_length"], reset_mask=b["reset_mask"],
            _final_obs=b["final_observations"], _final_glob=b["final_global_state"],
            _auto_reset=self.auto_reset)
        return self._out_view

    def _init_output(self) -> None:
        L = nat.lib()
        if self._side_stream:
            self._consume()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_init_output(self._h, ct.byref(self._outs)), "tabx_init_output")
        if self._side_stream:
            self._publish()
        self.last = self._output()

    # ------------------------------------------------------------ streams --
    # Inputs are produced on torch's current stream and the kernels run on
    # the simulator's stream: order the two before each launch, and tell the
    # caching allocator the simulator's stream reads the input.
    def _consume(self, *tensors) -> None:
        if not self._side_stream:
            return
        cur = torch.cuda.current_stream(self.device)
        if cur != self._stream:
            self._stream.wait_stream(cur)
            for t in tensors:
                if t is not None and t.is_cuda:
                    t.record_stream(self._stream)

    def _publish(self) -> None:
        """Make torch's current stream see the simulator stream's writes."""
        if not self._side_stream:
            return
        cur = torch.cuda.current_stream(self.device)
        if cur != self._stream:
            cur.wait_stream(self._stream)

    # ---------------------------------------------------------------- api --
    def step(self, actions=None, strict: bool | None = None, outs=None) -> BatchOutput:
        """One step of every lane; ``strict`` (default: the simulator's)
        raises a latched ActionMaskError synchronously.  ``outs`` (a
        ``TabxOutputs`` by reference) redirects outputs away from the
        simulator's own buffers (``HostStepper`` writes each step's rewards /
        flags straight into its per-slot buffers; the returned view then holds
        stale values for those fields)."""
        act_t = None
        if actions is not None:
            act_t = self._actions_tensor(actions)
        if self._side_stream:
            self._consume(act_t)
        # (the C side selects the handle's device for its launches)
        rc = self._step_fn(self._h, _ptr(act_t), self._outs_ref if outs is None else outs)
        if rc:
            nat.check(rc, "tabx_step")
        self._keep_actions = act_t  # keep alive until the stream consumed it
        if self._side_stream:
            self._publish()
        if act_t is not None and (self.strict if strict is None else strict):
            self.check_errors()
        self.last = self._output()
        return self.last

    def _actions_tensor(self, actions) -> torch.Tensor:
        if isinstance(actions, torch.Tensor):
            t = actions
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(actions, dtype=np.int64)))
        if t.numel() != self.batch * self.n_units:
            raise ValueError(f"actions of shape {tuple(t.shape)} do not match "
                             f"[batch, agents] = ({self.batch}, {self.n_units})")
        t = t.reshape(self.batch, self.n_units)
        if t.dtype != torch.int64:
            t = t.to(torch.int64)
        if t.device != self.device:
            t = t.to(self.device, non_blocking=True)
        return t.contiguous()

    def check_errors(self) -> None:
        """Raise ActionMaskError for a latched invalid action (synchronises)."""
        L = nat.lib()
        err = nat.TabxError()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_get_error(self._h, ct.byref(err), 1), "tabx_get_error")
        if err.code == nat.E_ACTION_MASK:
            raise ActionMaskError(f"invalid action {err.action} for unit {err.unit} in env {err.env}")

    def reset_env(self, b: int, config: Scenario | None = None, seed: int | None = None) -> None:
        """Restart lane ``b`` (environment.py:490-498).  Asynchronous: a new
        config's row is staged and uploaded on the stream; the lane's slot
        (shared with equal configs, recycled once no lane uses it) is kept in
        ``lane_slots``."""
        L = nat.lib()
        if not 0 <= b < self.batch:
            raise IndexError(f"env {b} out of range")
        cfg_ptr = None
        if config is not None:
            ensure_valid(config)
            cfg = build_config(config, validate=False)
            cfg_ptr = ct.byref(cfg)
        slot = ct.c_int32(-1)
        if self._side_stream:
            self._consume()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_reset_env(self._h, int(b), cfg_ptr,
                                       ct.c_uint64(0 if seed is None else int(seed) & (2**64 - 1)),
                                       0 if seed is None else 1, ct.byref(self._outs),
                                       ct.byref(slot)),
                      "tabx_reset_env")
        if config is not None:
            self.configs[b] = config
        self.lane_slots[b] = slot.value
        if self._side_stream:
            self._publish()
        self.last = self._output()

    def config_slot_info(self, slot: int) -> tuple[int, bool]:
        """(lanes on ``slot``, pinned) as tracked by the C side."""
        lanes, pinned = ct.c_int64(), ct.c_int32()
        nat.check(nat.lib().tabx_config_slot(self._h, int(slot), ct.byref(lanes),
                                             ct.byref(pinned)), "tabx_config_slot")
        return lanes.value, bool(pinned.value)

    def num_configs(self) -> tuple[int, int]:
        """(rows, capacity) of the handle's config table."""
        n, cap = ct.c_int32(), ct.c_int32()
        nat.check(nat.lib().tabx_num_configs(self._h, ct.byref(n), ct.byref(cap)),
                  "tabx_num_configs")
        return n.value, cap.value

    def respawn_all(self, seeds) -> None:
        """Fresh episodes for every lane with new seeds (bindings reset)."""
        L = nat.lib()
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(self.batch))
        lane_cfg = np.ascontiguousarray(self.lane_slots, dtype=np.int32)
        with torch.cuda.device(self.device):
            nat.check(L.tabx_respawn_all(self._h, seeds.ctypes.data_as(ct.c_void_p),
                                         lane_cfg.ctypes.data_as(ct.c_void_p)),
                      "tabx_respawn_all")
        self._init_output()

    def export_state(self) -> dict[str, torch.Tensor]:
        """Dynamic state with the reference SimArrays names and dtypes."""
        L = nat.lib()
        B, N = self.batch, self.n_units
        out = {}
        for k, (dt, tail) in STATE_DTYPES.items():
            shape = (B,) if k in PER_LANE else (B, N) + tuple(N if x == "N" else x for x in tail)
            out[k] = torch.empty(shape, dtype=dt, device=self.device)
        st = nat.TabxState(*[_ptr(out[k]) for k in nat.STATE_FIELDS])
        if self._side_stream:
            self._consume()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_export_state(self._h, ct.byref(st)), "tabx_export_state")
        self._stream.synchronize()
        return out

    def export_lanes(self, lanes: torch.Tensor, fields=None) -> dict[str, torch.Tensor]:
        """State rows of ``lanes`` (device int64) for ``fields`` (default all),
        gathered on the simulator's stream without synchronising and without
        materialising a pending cache refresh (the trace gather)."""
        L = nat.lib()
        N = self.n_units
        lanes = lanes.to(device=self.device, dtype=torch.int64).contiguous()
        n = lanes.numel()
        out = {}
        for k in (fields or STATE_DTYPES):
            dt, tail = STATE_DTYPES[k]
            shape = (n,) if k in PER_LANE else (n, N) + tuple(N if x == "N" else x for x in tail)
            out[k] = torch.empty(shape, dtype=dt, device=self.device)
        st = nat.TabxState(*[_ptr(out.get(k)) for k in nat.STATE_FIELDS])
        if self._side_stream:
            self._consume(lanes)
        with torch.cuda.device(self.device):
            nat.check(L.tabx_export_lanes(self._h, _ptr(lanes), n, ct.byref(st)),
                      "tabx_export_lanes")
        if self._side_stream:
            for v in out.values():
                v.record_stream(self._stream)
        self._keep_lanes = lanes
        return out

    def import_state(self, state: dict) -> None:
        """Overwrite dynamic state (parity injection); missing keys are kept."""
        L = nat.lib()
        keep = {}
        for k, (dt, _tail) in STATE_DTYPES.items():
            if k not in state or state[k] is None:
                continue
            v = state[k]
            if isinstance(v, np.ndarray):
                if v.dtype == np.uint64:
                    v = v.view(np.int64)
                v = torch.from_numpy(np.ascontiguousarray(v))
            keep[k] = v.to(device=self.device, dtype=dt).contiguous()
        st = nat.TabxState(*[_ptr(keep.get(k)) for k in nat.STATE_FIELDS])
        if self._side_stream:
            self._consume(*keep.values())
        with torch.cuda.device(self.device):
            nat.check(L.tabx_import_state(self._h, ct.byref(st)), "tabx_import_state")
        self._stream.synchronize()
        if "config" in keep:
            self.lane_slots = keep["config"].cpu().numpy().astype(np.int32)

    def episode_stats(self, reset: bool = False, device_out: torch.Tensor | None = None) -> dict:
        """Per-shard episode statistics (rollout.summarize inputs)."""
        L = nat.lib()
        host = (ct.c_double * nat.NUM_STATS)()
        with torch.cuda.device(self.device):
            nat.check(L.tabx_episode_stats(self._h, host, _ptr(device_out), int(reset)),
                      "tabx_episode_stats")
        keys = ("episodes", "ally_wins", "first_kill_ally", "truncation_ties", "sum_length",
                "sum_return", "eliminations", "env_steps")
        return dict(zip(keys, list(host)))

    def set_profiling(self, enable: bool = True) -> None:
        """Time the step's three kernels with CUDA events (restarts the sums)."""
        nat.check(nat.lib().tabx_set_profiling(self._h, int(enable)), "tabx_set_profiling")

    def kernel_profile(self) -> dict:
        """Average milliseconds per step of each kernel since set_profiling (syncs)."""
        ms = (ct.c_double * 3)()
        n = ct.c_int64()
        with torch.cuda.device(self.device):
            nat.check(nat.lib().tabx_get_profile(self._h, ms, ct.byref(n)), "tabx_get_profile")
        k = max(n.value, 1)
        fused = ct.c_int32()
        nat.check(nat.lib().tabx_step_path(self._h, ct.byref(fused)), "tabx_step_path")
        if fused.value == 2:  # the single-launch step (small batches)
            return {"steps": n.value, "fused": "single", "single_kernel_ms": ms[1] / k}
        if fused.value:  # [refresh check + K0 | fused step + observation kernel | K3]
            return {"steps": n.value, "fused": True, "ctrl_kernel_ms": ms[0] / k,
                    "fused_kernel_ms": ms[1] / k, "reset_kernel_ms": ms[2] / k}
        return {"steps": n.value, "fused": False, "step_kernel_ms": ms[0] / k,
                "obs_kernel_ms": ms[1] / k, "reset_kernel_ms": ms[2] / k}

    def step_path(self) -> str:
        """Kernels of the last step: 'split' (K1, K2, K3 and, from 4,096 lanes,
        the controller pass), 'fused' (fused step + observation kernel, opt-in)
        or 'single' (the whole step in one launch, small batches)."""
        fused = ct.c_int32()
        nat.check(nat.lib().tabx_step_path(self._h, ct.byref(fused)), "tabx_step_path")
        return {0: "split", 1: "fused", 2: "single"}[fused.value]

    def close(self) -> None:
        if getattr(self, "_h", None):
            nat.lib().tabx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h
