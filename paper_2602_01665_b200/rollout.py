"""Full on-device rollout loop (BASELINE config C5).

A trainer's collection loop with nothing on the host: each step the policy
reads the previous observation in place, samples legal actions from the
current action mask, and the batched step writes the next observation
straight into the horizon buffer slot (no copies).  The whole horizon —
policy forward, masked sampling and the environment kernels — is captured
once into a CUDA graph and replayed per iteration.

Policies: ``random`` (uniform over legal actions, the reference's random
controller semantics) or ``mlp`` (a bf16 two-layer MLP over the per-agent
observation).  Either way the actions come from the library's fused masked
Gumbel-max sampler (``tabx_masked_sample``, fused into the policy-MLP kernel
for ``mlp``: one pass per agent producing the action and its log-probability, noise keyed on a device step counter so the
replayed graph draws fresh noise).  The MLP reads a bf16 copy of the
observation padded to a multiple of 8 features (aligned GEMM rows) and emits
8 logits of which the first 7 are the actions.  The ally team is driven by
the policy (external controller); the enemy keeps its scenario controller.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import torch

from . import _native as nat
from .rng import lane_seeds
from .scenario import Scenario
from .sim import BatchSim


class MLPPolicy(torch.nn.Module):
    """Two-layer MLP over padded per-agent observations -> 8 logits (7 used).

    On CUDA (bf16, hidden 128) the forward is one launch of the library's
    tcgen05 kernel (``tabx_policy_mlp``: x read once, the hidden tile kept in
    TMEM / registers, fp32 accumulation, hidden rounded to bf16);
    ``reference`` is the same function in torch ops (tests and CPU)."""

    def __init__(self, obs_dim: int, hidden: int = 128, n_actions: int = 7):
        super().__init__()
        self.in_dim = (obs_dim + 7) // 8 * 8
        self.l1 = torch.nn.Linear(self.in_dim, hidden)
        self.l2 = torch.nn.Linear(hidden, (n_actions + 7) // 8 * 8)

    def reference(self, obs: torch.Tensor) -> torch.Tensor:
        x = obs.reshape(-1, self.in_dim)
        # bias + ReLU in the first GEMM's epilogue (cuBLASLt on CUDA)
        h = torch._addmm_activation(self.l1.bias, x, self.l1.weight.t())
        out = torch.addmm(self.l2.bias, h, self.l2.weight.t())
        return out.reshape(*obs.shape[:-1], out.shape[-1])

    def forward(self, obs: torch.Tensor) -> torch.Tensor:
        if not obs.is_cuda:
            return self.reference(obs)
        if (self.l1.out_features != 128 or self.l2.out_features != 8
                or obs.dtype != torch.bfloat16 or self.l1.weight.dtype != torch.bfloat16):
            raise ValueError("tabx_policy_mlp needs bf16, hidden 128, 8 logits")
        x = obs.reshape(-1, self.in_dim)
        if x.stride(-1) != 1:
            x = x.contiguous()
        out = torch.empty(x.shape[0], 8, device=x.device, dtype=torch.bfloat16)
        ptr = lambda t: ct.c_void_p(t.data_ptr())  # noqa: E731
        nat.check(nat.lib().tabx_policy_mlp(
            ptr(x), x.shape[0], self.in_dim, x.stride(0), ptr(self.l1.weight), ptr(self.l1.bias),
            ptr(self.l2.weight), ptr(self.l2.bias), ptr(out),
            ct.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)), "tabx_policy_mlp")
        return out.reshape(*obs.shape[:-1], 8)


def masked_sample(logits: torch.Tensor, mask: torch.Tensor):
    """Gumbel-max sample over legal actions with torch ops (reference
    semantics of the fused sampler); returns (actions int64, logp f32)."""
    u = torch.rand_like(logits, dtype=torch.float32).clamp_(1e-12, 1.0)
    g = -torch.log(-torch.log(u))
    neg = torch.finfo(torch.float32).min
    masked = torch.where(mask, logits.float(), neg)
    act = torch.argmax(masked + g, dim=-1)
    logp = torch.log_softmax(masked, dim=-1).gather(-1, act[..., None])[..., 0]
    return act, logp


@dataclass
class RolloutBuffers:
    observations: torch.Tensor | None  # [T+1, B, N, D] float32 (slot 0 = start)
    actions: torch.Tensor  # [T, B, N] int64
    logp: torch.Tensor  # [T, B, N] float32
    rewards: torch.Tensor  # [T, B, N] float32
    terminated: torch.Tensor  # [T, B] bool
    truncated: torch.Tensor  # [T, B] bool


class Rollout:
    def __init__(self, scenario: Scenario, envs: int, horizon: int = 128, policy: str = "random",
                 device=0, seed: int = 0, first_lane: int = 0, store_obs: bool = True,
                 hidden: int = 128, use_graph: bool = True):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        sc = scenario.with_controllers(ally="external")
        self.sim = BatchSim([sc] * envs, lane_seeds(seed, envs, first_lane), auto_reset=True,
                            device=self.device, strict=False, interactions=False,
                            final_observations=False)
        self.B, self.N, self.D = envs, self.sim.n_units, self.sim.obs_dim
        self.T = horizon
        self.kind = policy
        dev = self.device
        T, B, N, D = self.T, self.B, self.N, self.D
        self.buf = RolloutBuffers(
            observations=torch.empty(T + 1, B, N, D, device=dev) if store_obs else None,
            actions=torch.empty(T, B, N, dtype=torch.int64, device=dev),
            logp=torch.empty(T, B, N, device=dev),
            rewards=torch.empty(T, B, N, device=dev),
            terminated=torch.empty(T, B, dtype=torch.bool, device=dev),
            truncated=torch.empty(T, B, dtype=torch.bool, device=dev))
        self.policy = None
        if policy == "mlp":
            self.policy = MLPPolicy(D, hidden).to(dev).to(torch.bfloat16)
            self._xin = torch.zeros(B, N, self.policy.in_dim, dtype=torch.bfloat16, device=dev)
        elif policy == "random":
            self._zero_logits = torch.zeros(B * N, 8, device=dev)
        else:
            raise ValueError(f"unknown policy {policy!r}")
        self.seed = int(seed)
        self._ctr = torch.zeros(1, dtype=torch.int64, device=dev)  # sampler noise counter
        self._outs = []
        for t in range(T):
            o = nat.TabxOutputs()
            for k in nat.OUTPUT_FIELDS:
                setattr(o, k, None)
            obs = self.buf.observations[t + 1] if store_obs else self.sim._buf["observations"]
            o.observations = obs.data_ptr()
            o.global_state = self.sim._buf["global_state"].data_ptr()
            o.rewards = self.buf.rewards[t].data_ptr()
            o.action_mask = self.sim._buf["action_mask"].data_ptr()
            o.terminated = self.buf.terminated[t].data_ptr()
            o.truncated = self.buf.truncated[t].data_ptr()
            o.done = self.sim._buf["done"].data_ptr()
            o.reset_mask = self.sim._buf["reset_mask"].data_ptr()
            if self.policy is not None:
                # the step's emitter also writes the policy's bf16 input rows
                o.observations_bf16 = self._xin.data_ptr()
                o.observations_bf16_ld = self.policy.in_dim
            self._outs.append(o)
        if store_obs:
            self.buf.observations[0].copy_(self.sim._buf["observations"])
        if self.policy is not None:  # the start observation, once
            nat.check(nat.lib().tabx_pack_bf16(
                ct.c_void_p(self.sim._buf["observations"].data_ptr()), B * N, D,
                self.policy.in_dim, ct.c_void_p(self._xin.data_ptr()),
                ct.c_void_p(torch.cuda.current_stream(dev).cuda_stream)), "tabx_pack_bf16")
        self.graph = None
        self.use_graph = use_graph

    def _current_obs(self, t):
        if self.buf.observations is not None:
            return self.buf.observations[t]
        return self.sim._buf["observations"]

    def _step(self, t):
        mask = self.sim._buf["action_mask"]
        L = nat.lib()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ptr = lambda x: ct.c_void_p(x.data_ptr())  # noqa: E731
        if self.policy is None:
            logits = self._zero_logits
            nat.check(L.tabx_masked_sample(
                ptr(logits), 0, logits.shape[-1], ptr(mask), self.B * self.N,
                ct.c_uint64(self.seed), ptr(self._ctr), t, ptr(self.buf.actions[t]),
                ptr(self.buf.logp[t]), ct.c_void_p(stream)), "tabx_masked_sample")
        else:
            # _xin: the current observation in bf16, written by the last step;
            # policy MLP + masked sampler in one tcgen05 kernel (no logits in HBM)
            p = self.policy
            nat.check(L.tabx_policy_mlp_sample(
                ptr(self._xin), self.B * self.N, p.in_dim, p.in_dim, ptr(p.l1.weight),
                ptr(p.l1.bias), ptr(p.l2.weight), ptr(p.l2.bias), None, ptr(mask),
                ct.c_uint64(self.seed), ptr(self._ctr), t, ptr(self.buf.actions[t]),
                ptr(self.buf.logp[t]), ct.c_void_p(stream)), "tabx_policy_mlp_sample")
        nat.check(L.tabx_step(self.sim.handle, ct.c_void_p(self.buf.actions[t].data_ptr()),
                              ct.byref(self._outs[t])), "tabx_step")

    def _horizon(self):
        for t in range(self.T):
            self._step(t)
        self._ctr.add_(self.T)  # next horizon's noise

    def _set_stream(self, stream):
        nat.check(nat.lib().tabx_set_stream(self.sim.handle, ct.c_void_p(stream.cuda_stream)),
                  "tabx_set_stream")

    def capture(self) -> None:
        """Record the whole horizon into one CUDA graph (after a warm-up run)."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self._set_stream(s)
            self._horizon()  # warm-up: cuBLAS handles, allocator pools
            if self.buf.observations is not None:
                self.buf.observations[0].copy_(self.buf.observations[self.T])
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._set_stream(torch.cuda.current_stream(self.device))
            self._horizon()
        self._set_stream(torch.cuda.current_stream(self.device))

    def run(self) -> RolloutBuffers:
        """Collect one horizon (graph replay when captured)."""
        if self.use_graph:
            if self.graph is None:
                self.capture()
            self.graph.replay()
        else:
            self._horizon()
        if self.buf.observations is not None:
            # next horizon starts from the last observation
            self.buf.observations[0].copy_(self.buf.observations[self.T])
        return self.buf

    def close(self):
        self.sim.close()
