"""Pipelined host stepping (``bindings.HostStepper``) against plain ``step``.

The stepper overlaps each step's host->device action upload and
device->host result download with the neighbouring steps; its results must
equal the synchronous trainer API's step for step, and an invalid action
must surface as the reference's ``ActionMaskError`` (environment.py:166-178)
with no lane mutated.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2602_01665_b200 import bindings
from paper_2602_01665_b200.scenario import ActionMaskError, builtin_scenario, save_scenario

pytestmark = pytest.mark.gpu


def _doc():
    return save_scenario(builtin_scenario("c3_10v10_terrain")).encode()


def test_stepper_matches_synchronous_steps():
    B, T = 512, 24
    a = bindings.make_batch(_doc(), B, 11, device=0)
    b = bindings.make_batch(_doc(), B, 11, device=0)
    gen = np.random.default_rng(5)
    acts = [torch.from_numpy(gen.integers(0, 5, size=(B, a.agents), dtype=np.int64)).pin_memory()
            for _ in range(T)]
    st = bindings.HostStepper(b)
    tickets = []
    for k in range(T):
        _, _, rew, term, trunc, _ = bindings.step(a, acts[k].to(0))
        want = (rew.cpu(), term.cpu(), trunc.cpu())
        tickets.append((st.submit(acts[k]), want))
        if len(tickets) == 2:
            t, w = tickets.pop(0)
            got = st.result(t)
            for x, y in zip(got, w):
                assert torch.equal(x, y)
    t, w = tickets.pop(0)
    for x, y in zip(st.result(t), w):
        assert torch.equal(x, y)
    torch.cuda.synchronize()
    assert torch.equal(a.sim.last.observations, b.sim.last.observations)


def test_stepper_raises_action_mask_error_without_mutation():
    B = 64
    h = bindings.make_batch(_doc(), B, 3, device=0)
    st = bindings.HostStepper(h)
    ok = np.zeros((B, h.agents), np.int64)
    st.result(st.submit(ok))
    before = h.sim.export_state()
    bad = ok.copy()
    bad[7, 2] = 9  # out of range for a controllable external unit
    k = st.submit(bad)
    with pytest.raises(ActionMaskError, match="invalid action 9 for unit 2 in env 7"):
        st.result(k)
    after = h.sim.export_state()
    for key in ("pos", "health", "t"):
        assert torch.equal(before[key], after[key])
    st.result(st.submit(ok))  # the latch was cleared: stepping resumes
    assert int(h.sim.export_state()["t"][0]) == int(before["t"][0]) + 1
