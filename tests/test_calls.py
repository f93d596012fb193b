"""func.call (and memref.alloc) inside loop regions, CPU side: the reference
executor, the oracle and the engine's host pipeline on the kernel simulator
agree (results, stats, errors).  tests/test_gpu_calls.py runs them on the
B200 against the oracle."""
import pytest

import call_cases
from vm_sim import SimEngine


@pytest.mark.parametrize("name", sorted(call_cases.CASES))
def test_calls_in_loops(name, ref_engine, oracle_engine):
    want = call_cases.outcome(ref_engine, name)
    assert call_cases.outcome(oracle_engine, name) == want
    assert call_cases.outcome(SimEngine(), name) == want


def test_call_in_parallel_keeps_the_band():
    """The inlined call does not serialise the parallel nest."""
    from paper_2307_16080_b200 import engine

    call_cases.outcome(SimEngine(), "call_in_parallel")
    assert engine.last_plan == [("vm", 2, "unchecked", "static")]
