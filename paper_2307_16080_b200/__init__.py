"""B200-native execution backend for staircase (arXiv 2307.16080 kernels).

A drop-in engine for the reference's CPU tape evaluators
(staircase/interp/machine.py:26-34,105-112): loop nests captured with the
unchanged DSL run as hand-written sm_100a CUDA kernels behind the C ABI in
include/b200k.h.

    import paper_2307_16080_b200 as b2
    b2.install()                     # every staircase run() now uses the GPU
    staircase.interp.machine.run(module, "matmul", [A, B, C])
"""
from .host import ensure_staircase

ensure_staircase()

from . import engine  # noqa: E402
from .engine import (ENGINE_NAME, ExecContext, Session, configure, install,  # noqa: E402
                     run_tape, settings, uninstall, using)
from .races import check_races  # noqa: E402

__all__ = ["engine", "install", "uninstall", "configure", "using", "settings", "run_tape",
           "ExecContext", "Session", "ENGINE_NAME", "check_races"]
