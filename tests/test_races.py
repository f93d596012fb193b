"""races.check_races (static-affine race proof) against the reference's
check_races (staircase/interp/races.py:20-97), on CPU through the engine
simulator.

Race-free affine parallels must be proven without running the reference
simulation; racy or data-dependent ones must return the reference's exact
conflict list.
"""
import pytest

import bench_kernels as bk
import corpus
import harness
from vm_sim import SimEngine

RACY = '''
@staged
def racy(x: MemRef[(16, 8), F32], acc: MemRef[(4,), F32]):
    for i, j in parallel((0, 0), (16, 8)):
        acc[1] = acc[1] + x[i, j]
'''

GATHER = '''
@staged
def gather(x: MemRef[(32,), F32], y: MemRef[(1024,), F32]):
    for i in parallel((0,), (32,)):
        y[i * i] = x[i]
'''

STENCIL = '''
@staged
def stencil(x: MemRef[(34, 34), F32], y: MemRef[(34, 34), F32]):
    for i, j in parallel((1, 1), (33, 33)):
        y[i, j] = x[i - 1, j] + x[i + 1, j] + x[i, j - 1] + x[i, j + 1]
'''

SHIFT = '''
@staged
def shift(x: MemRef[(64,), F32]):
    for i in parallel((0,), (63,)):
        x[i] = x[i + 1]
'''


def _kernels():
    return {name: bk._capture_from_source(src, name, {}, "races")
            for name, src in (("racy", RACY), ("gather", GATHER), ("stencil", STENCIL),
                              ("shift", SHIFT))}


def _reference(fn, args):
    from staircase.interp.races import check_races

    return check_races(fn.module, fn.__name__, args)


@pytest.mark.parametrize("name,proven", [("racy", False), ("gather", False),
                                         ("stencil", True), ("shift", False)])
def test_small_kernels_match_reference(name, proven, monkeypatch):
    from paper_2307_16080_b200 import races
    import staircase.interp.races as ref_races

    fn = _kernels()[name]
    args = harness.make_args(fn, 3)
    want = _reference(fn, args)
    calls = []
    orig = ref_races.check_races
    monkeypatch.setattr(ref_races, "check_races",
                        lambda *a, **k: calls.append(1) or orig(*a, **k))
    got = races.check_races(fn.module, fn.__name__, args, engine=SimEngine())
    assert got == want
    assert (not calls) == proven
    if name == "racy":
        assert want, "the racy kernel must have conflicts"


@pytest.mark.parametrize("fn", [corpus.matmul_par, corpus.conv_f32, corpus.saxpy_f32,
                                corpus.ewise_gpu])
def test_corpus_parallel_kernels_are_proven(fn, monkeypatch):
    from paper_2307_16080_b200 import races
    import staircase.interp.races as ref_races

    args = harness.make_args(fn, 1)
    assert _reference(fn, args) == []
    monkeypatch.setattr(ref_races, "check_races",
                        lambda *a, **k: pytest.fail("fell back to the simulation"))
    assert races.check_races(fn.module, fn.__name__, args, engine=SimEngine()) == []
