"""Locate the host framework (the reference's staircase package) and make it
importable on CPython 3.12.

The B200 backend plugs into staircase's engine protocol
(staircase/interp/machine.py:26-34,105-112); staircase itself is the host
framework the user already runs.  In this repository it is installed,
unmodified, into ``baseline/_ref`` by ``baseline/install_ref.sh``.

staircase/frontend/bytecode.py:28 reads ``dis.opmap["JUMP_ABSOLUTE"]``,
which CPython 3.12 removed; the bytecode patch it feeds is gated to 3.10
(bytecode.py:37-38,50-53), so registering a dummy opcode number is harmless
and lets capture fall back to source flattening (capture.py:142-147).
"""
from __future__ import annotations

import dis
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(_REPO, "baseline", "_ref")


def ensure_staircase():
    """Import and return the staircase package (shimmed for py3.12)."""
    dis.opmap.setdefault("JUMP_ABSOLUTE", -1)
    try:
        import staircase  # noqa: F401
    except ImportError:
        if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import staircase  # noqa: F401
    return sys.modules["staircase"]


def errors():
    """staircase.errors — the exception types run() callers expect."""
    ensure_staircase()
    import staircase.errors as e

    return e
