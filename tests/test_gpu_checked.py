"""The parity cases through the CHECKED build of the kernels.

compute-sanitizer is not available on the GPU pool this project runs on (it
is closed there: runs under it left GPUs needing a reset), so the race /
initialisation / bounds evidence comes from a checked variant of the same
sources, ``_tabx_checked.so`` (``-DTABX_CHECKS``, built by ``build()``):

* every environment's shared memory (K1's env state, K0's controller view,
  K2's view and visible-pair list) is filled with 0xFF bytes before use, so
  a read of a value that environment never wrote is a NaN / -1 and breaks
  bit-exact parity (initcheck);
* each lane sleeps a pseudo-random 0-1 us at every phase boundary of the
  step (and before K2's stage flushes and K0's decision write), so lanes of
  a warp reach later shared-memory reads in shuffled order: a hand-off
  missing its ``__syncwarp`` / ``__syncthreads`` / proxy fence reads a stale
  or half-written value (racecheck / synccheck);
* device asserts on unit / pair / target indices and on every TMA bulk
  store's range and 16-byte alignment trap the context (memcheck-lite).

The selected parity tests (golden trajectories through both controller
paths, injected states for W = 1/2/4/8, many zones, mixed configs, slot
recycling, device levels) run in a subprocess with ``TABX_LIB`` pointing at
the checked library and must pass bit-exactly.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CHECKED = os.path.join(ROOT, "paper_2602_01665_b200", "_tabx_checked.so")
SELFTEST = os.path.join(ROOT, "paper_2602_01665_b200", "_tabx_selftest_race.so")

SELECT = ("test_golden_case_parity or test_injected_state_single_step or "
          "test_many_zones_match_oracle or test_two_word_rows_with_zones_match_oracle or "
          "test_mixed_configs_and_reset_env_swap or test_controller_pass_mixed_heuristic_counts "
          "or test_action_mask_error or test_dead_units or test_fov_boundary or "
          "test_slot_recycling or test_batch_of_levels_and_respawn or "
          "test_fused_small_and_ragged_batches_match_oracle or test_single_launch_step_matches_oracle")


def test_parity_cases_through_checked_kernels():
    if not os.path.exists(CHECKED):
        pytest.fail(f"{CHECKED} missing: run build() (it builds the checked variant too)")
    env = dict(os.environ, TABX_LIB=CHECKED)
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_reconfig.py"),
           os.path.join(HERE, "test_gpu_levels.py"), os.path.join(HERE, "test_gpu_fused.py"),
           "-k", SELECT]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    tail = (r.stdout + r.stderr)[-4000:]
    print(r.stdout[-600:])
    assert r.returncode == 0, tail
    assert "TABX_CHECK failed" not in r.stdout + r.stderr, tail
    import re
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 30, tail  # the selection really ran


def test_checked_build_catches_a_dropped_barrier():
    """Negative control: the checked build with ONE barrier removed (the
    W > 1 step kernel's hand-off between ranking the units along y and the
    contact sweep that reads that order, -DTABX_SELFTEST_RACE, with half the
    threads publishing their ranks late) must fail the W > 1 parity cases --
    evidence that the method sees a missing barrier."""
    if not os.path.exists(SELFTEST):
        pytest.fail(f"{SELFTEST} missing: run build() (it builds the negative control too)")
    env = dict(os.environ, TABX_LIB=SELFTEST)
    sel = ("test_golden_case_parity and (c4 or w8) or test_injected_state_single_step or "
           "test_two_word_rows_with_zones_match_oracle")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(HERE, "test_gpu_parity.py"), "-k", sel]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    print(r.stdout[-800:])
    assert r.returncode != 0 and " failed" in r.stdout, (r.stdout + r.stderr)[-3000:]
