"""B200-native batched environment step for TABX (arxiv 2602.01665).

A drop-in for the reference engine's batch path (``skirmish.BatchSim`` and
``skirmish_bindings``): same scenario documents, reset/step semantics and
observation / global-state / reward / action-mask layouts, executed by
hand-written sm_100a CUDA kernels behind a C ABI (``include/tabx.h``).

Host-only modules (scenario parsing, RNG keys, templates) import without a
GPU; :class:`BatchSim` and the bindings load the CUDA extension and fail
loudly if it is missing.
"""
from .rng import TAG_EPISODE, TAG_RESEED, derive_seed, key_hash, lane_seeds  # noqa: F401
from .scenario import (ActionMaskError, Scenario, ScenarioFormatError,  # noqa: F401
                       builtin_scenario, load_scenario, load_scenario_file, save_scenario,
                       validate_scenario)

__version__ = "0.1.0"


def __getattr__(name):
    import importlib

    if name in ("BatchSim", "BatchOutput"):
        return getattr(importlib.import_module(".sim", __name__), name)
    if name in ("bindings", "sim"):
        return importlib.import_module("." + name, __name__)
    raise AttributeError(name)
