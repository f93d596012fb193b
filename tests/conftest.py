"""Shared test setup.

- registers the ``gpu`` marker (tests that need a B200);
- makes the repo root and the host framework (staircase, installed
  unmodified in baseline/_ref) importable, with the py3.12 capture shim.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ref_engine():
    """The reference's own compiled executor (_evalcy), the ground truth."""
    from staircase.interp import _evalcy

    return _evalcy


@pytest.fixture(scope="session")
def oracle_engine():
    import oracle

    oracle.build()
    return oracle


# max normalised errors of the tensor-core parity tests (tcbound.check):
# printed in the session summary so every run reports them
TC_ERRORS = []


def pytest_terminal_summary(terminalreporter):
    if TC_ERRORS:
        terminalreporter.write_sep("-", "tensor-core parity: max normalised errors")
        for label, K, e, *rest in TC_ERRORS:
            how = rest[0] if rest else "|got-want| / (2^-24 sqrt(K) sum|ab|), bound 8"
            terminalreporter.write_line(f"{label}: K={K} max_norm_err={e:.3g} ({how})")


@pytest.fixture(autouse=True)
def _fresh_plan_cache():
    """Each test starts with an empty region plan cache (plancache.py), so a
    test that inspects matching (monkeypatched templates) sees it happen;
    repeated runs inside one test still hit the cache."""
    from paper_2307_16080_b200 import plancache

    plancache.clear()
    yield
