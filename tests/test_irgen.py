"""The reference's random modules (pkg/tests/irgen.py) against the reference
executor's recorded outcome (tests/golden/irgen.json, make_irgen_golden.py).

Nested loops, conditionals, parallel nests, memref.alloc inside loop bodies,
unchecked indices (about a third raise OutOfBounds): the oracle must match
every fixture, and so must the B200 engine's host pipeline driven by the
CPU simulator of its kernels (tests/vm_sim.py) — buffers, the 25-slot tally,
error type and message.  The same fixtures run on the B200 in
tests/test_gpu_irgen.py.
"""
import pytest

import irgen_cases
from vm_sim import SimEngine

IDS = [f"seed{c['seed']}" for c in irgen_cases.CASES]


@pytest.mark.parametrize("case", irgen_cases.CASES, ids=IDS)
def test_oracle_matches_reference(case, oracle_engine):
    irgen_cases.check(oracle_engine, case, exact_fault_tally=True)


@pytest.mark.parametrize("case", irgen_cases.CASES, ids=IDS)
def test_engine_sim_matches_reference(case):
    irgen_cases.check(SimEngine(), case)


def test_fixtures_exercise_allocs_in_loops():
    loops = ("scf.for", "affine.for", "scf.parallel")
    n = 0
    for c in irgen_cases.CASES:
        lines = c["sir"].splitlines()
        depth_alloc = [ln for ln in lines if "memref.alloc" in ln and ln.startswith("      ")]
        if depth_alloc and any(k in c["sir"] for k in loops):
            n += 1
    assert n >= 10
