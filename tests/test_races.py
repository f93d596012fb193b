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


SCATTER_SIR = """
module {
  func.func @scatter(%arg0: memref<32xi64>, %arg1: memref<32xf32>, %arg2: memref<16xf32>) {
    %0 = arith.constant 0 : index
    %1 = arith.constant 32 : index
    %2 = arith.constant 1 : index
    scf.parallel (%arg3) = (%0) to (%1) step (%2) {
      %3 = memref.load %arg0[%arg3] : memref<32xi64>
      %4 = arith.index_cast %3 : i64 to index
      %5 = memref.load %arg1[%arg3] : memref<32xf32>
      memref.store %5, %arg2[%4] : memref<16xf32>
      scf.yield
    }
    return
  }
}
"""


def scatter_module():
    from staircase.ir.core import create_context
    from staircase.textio import parse_module

    return parse_module(SCATTER_SIR, create_context())


def scatter_args():
    from staircase.interp import Buffer

    return [Buffer((32,), "i64", [(7 * i) % 16 for i in range(32)]),
            Buffer((32,), "f32", [float(i) for i in range(32)]), Buffer((16,), "f32", [0.0] * 16)]


@pytest.mark.parametrize("name,ok", [("racy", True), ("gather", True), ("shift", True),
                                     ("stencil", True)])
def test_recordable_regions(name, ok):
    """Which unproven regions the device recorder takes (races.recordable):
    data-independent address streams over argument buffers."""
    from paper_2307_16080_b200 import analysis, engine, races

    fn = _kernels()[name]
    args = harness.make_args(fn, 3)
    labels = {id(a): f"arg{i}" for i, a in enumerate(args)}
    seen = []
    with engine.region_hook(lambda r, acc: seen.append(races.recordable(r, acc, labels))):
        harness.run_engine(SimEngine(), fn, None, "gpu_emulated", 3, args=args)
    assert seen == [ok]
    del analysis


def test_data_dependent_scatter_is_not_recordable():
    """y[idx[i]] = x[i]: the address comes from loaded data, so the replay
    without data is not the program — the reference simulation decides."""
    from staircase.interp import machine

    from paper_2307_16080_b200 import engine, races

    module, args = scatter_module(), scatter_args()
    labels = {id(a): f"arg{i}" for i, a in enumerate(args)}
    seen = []
    with engine.region_hook(lambda r, acc: seen.append(races.recordable(r, acc, labels))):
        machine.run(module, "scatter", args, mode="gpu_emulated", engine=SimEngine())
    assert seen == [False]
    got = races.check_races(module, "scatter", scatter_args(), engine=SimEngine())
    from staircase.interp.races import check_races

    assert got == check_races(module, "scatter", scatter_args()) and got


@pytest.mark.parametrize("name", ["racy", "gather", "shift", "stencil"])
def test_record_kernel_compiles(name):
    """The recorder's replay kernel (native.vm_source(record=True)) compiles
    for sm_100a with NVRTC (no GPU needed)."""
    from paper_2307_16080_b200 import analysis, engine, jit, native, vmcode

    fn = _kernels()[name]
    args = harness.make_args(fn, 3)
    got = []
    with engine.region_hook(lambda r, acc: got.append((r, acc))):
        harness.run_engine(SimEngine(), fn, None, "gpu_emulated", 3, args=args)
    (r, acc), = got
    links, remainder = analysis.chain_of(r)
    band = [v.id for v in r.tree[0].vars]
    prog = vmcode.encode(r, links, remainder, band, False,
                         checked=not analysis.statically_in_bounds(r, acc))
    env_regs = [v for v in r.env if r.kind[v] != "buf"]
    src, kname, _ = native.vm_source(prog, r.buffers, env_regs, record=True)
    assert "rec(PASS" in src and kname == "b200_vm_record"
    assert jit.cubin(src, kname)[:4] == b"\x7fELF"
