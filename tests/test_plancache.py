"""The region plan cache (paper_2307_16080_b200/plancache.py), CPU side.

A cached plan is reused only for the same region code, the same scalar
values (bit for bit), the same buffer geometry and the same aliasing; every
golden fixture must come out identical when served from the cache, and a
change of any key component must miss.
"""
import pytest

import corpus
import harness
from test_oracle import GOLDEN, check_against_golden
from vm_sim import SimEngine


@pytest.mark.parametrize("case", GOLDEN,
                         ids=[f"{c['kernel']}-{c['variant']}-s{c['seed']}" for c in GOLDEN])
def test_golden_fixtures_from_the_cache(case):
    from paper_2307_16080_b200 import plancache

    check_against_golden(SimEngine(), case)        # fills the cache
    hits = plancache.STATS["hits"]
    check_against_golden(SimEngine(), case)        # served from it
    if "error" not in case:
        assert plancache.STATS["hits"] > hits


def test_scalar_values_are_part_of_the_key(oracle_engine):
    from staircase.interp import Buffer, machine

    fn = corpus.scalar_args
    for n in (20, 7, 20, 32):
        for s in (0.5, -0.0, 0.0):
            a = Buffer((32,), "f32", [float(i) - 3.5 for i in range(32)])
            b = Buffer((32,), "f32", [float(i) - 3.5 for i in range(32)])
            _, st = machine.run(fn.module, "scalar_args", [a, s, n], engine=SimEngine())
            _, sw = machine.run(fn.module, "scalar_args", [b, s, n], engine=oracle_engine)
            assert a.data.tobytes() == b.data.tobytes() and st.total == sw.total


def test_aliasing_is_part_of_the_key(oracle_engine):
    """y = y + 2x with x and y distinct, then with x and y the same Buffer:
    the aliased call must not reuse the distinct call's plan (its JIT kernel
    declares the operands non-aliasing)."""
    from staircase.interp import Buffer, machine

    fn = corpus.saxpy_f32      # y = y + x * 2 over (64, 128)
    for alias in (False, True, False):
        args = harness.make_args(fn, 1)
        want = harness.make_args(fn, 1)
        if alias:
            args = [args[0], args[0]]
            want = [want[0], want[0]]
        machine.run(fn.module, fn.__name__, args, engine=SimEngine())
        machine.run(fn.module, fn.__name__, want, engine=oracle_engine)
        assert [a.data.tobytes() for a in args] == [w.data.tobytes() for w in want]


def test_linear32_repeated_runs_hit():
    from paper_2307_16080_b200 import engine, plancache
    from staircase.interp import machine

    fn = corpus.linear32
    machine.run(fn.module, fn.__name__, harness.make_args(fn, 0), engine=SimEngine())
    first = list(engine.last_plan)
    misses = plancache.STATS["misses"]
    for seed in (1, 2):
        machine.run(fn.module, fn.__name__, harness.make_args(fn, seed), engine=SimEngine())
        assert engine.last_plan == first          # same fused plan
    assert plancache.STATS["misses"] == misses    # every region served from the cache
