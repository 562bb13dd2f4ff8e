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


def test_c_caller_matches_python_bindings(tmp_path):
    """The C ABI driven from a plain C program (tests/native/abi_driver.c,
    linked against the in-tree _tabx.so and libcudart) gives the same
    rewards and observations as the Python BatchSim over the same ABI."""
    import os
    import shutil
    import subprocess

    from paper_2602_01665_b200 import _native as nat
    from paper_2602_01665_b200.sim import BatchSim
    from paper_2602_01665_b200.template import build_config
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    lib = os.path.dirname(nat.LIB_PATH)
    cuda = "/usr/local/cuda"
    exe = str(tmp_path / "abi_driver")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(root, "include"), "-I",
                           f"{cuda}/include", os.path.join(here, "native", "abi_driver.c"),
                           "-o", exe, f"-L{lib}", "-l:_tabx.so", f"-L{cuda}/lib64", "-lcudart",
                           f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{cuda}/lib64"])
    sc = builtin_scenario("c3_10v10_terrain")
    cfg = build_config(sc)
    (tmp_path / "cfg.bin").write_bytes(bytes(memoryview(cfg)))
    B, T, seed0 = 96, 6, 1000
    res = subprocess.run([exe, str(tmp_path / "cfg.bin"), str(B), str(T), str(seed0)],
                         capture_output=True, text=True, check=True)
    got = [tuple(float(x) for x in ln.split()[1:]) for ln in res.stdout.strip().splitlines()]
    sim = BatchSim([sc] * B, np.arange(seed0, seed0 + B, dtype=np.uint64), auto_reset=True,
                   device=0, interactions=False)
    N, D = sim.n_units, sim.obs_dim
    wr = torch.tensor([(k % 7) + 1 for k in range(B * N)], dtype=torch.float64)
    wo = (torch.arange(B * N * D, dtype=torch.int64) % 13 + 1).double()
    for t in range(T):
        acts = (torch.arange(B)[:, None] + torch.arange(N)[None, :] + t) % 5
        out = sim.step(acts.to(torch.int64))
        rs = float((out.rewards.cpu().double().reshape(-1) * wr).sum())
        os_ = float((out.observations.cpu().double().reshape(-1) * wo).sum())
        assert got[t][0] == pytest.approx(rs, rel=1e-12, abs=1e-9), t
        assert got[t][1] == pytest.approx(os_, rel=1e-12), t
    sim.close()
