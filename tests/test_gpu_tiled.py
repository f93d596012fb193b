"""Reference-tiled matmul / Linear nests on the B200 at full size (-m gpu).

BASELINE configs[1]: linalg.matmul 4096^3 "with reference tile sizes".  The
parallel-form matmul nest goes through the reference's own
scf-parallel-loop-tiling pass with the reference tile sizes (8, 8) and
(4, 16) (reference SPEC.md:778; passes/tiling.py:56-80) and then through
staircase's run() with the B200 engine.  The tiled nest must

* be recognised as one strided GEMM and run on the tensor cores at bf16 /
  tf32 (plan gemm_tc_*), bit-exact on the FP32 pipes at exact precision;
* run with the CTA tile its tile sizes select (runtime.cta_tile) — recorded
  in the plan as tile<tm>x<tn>->cta<BM>x<BN>;
* match: exact — the reference's f32 chain bit for bit on sampled outputs;
  bf16 / tf32 — the tight sqrt(K) bound (tests/tcbound.py).
"""
import numpy as np
import pytest

import harness
import tcbound

pytestmark = pytest.mark.gpu

SAMPLES = 96
TILES = {"8x8": (harness.TILE88, (8, 8)), "4x16": (harness.TILE416, (4, 16)),
         "16x4": (harness._spec("scf-parallel-loop-tiling{sizes=[16, 4]}"), (16, 4)),
         "2x2": (harness._spec("scf-parallel-loop-tiling{sizes=[2, 2]}"), (2, 2))}


def _inputs(fn, seed=0):
    import torch
    from staircase.interp import Buffer

    out = []
    for i, a in enumerate(fn.func_op.body().args):
        shape = tuple(a.type.shape)
        g = torch.Generator().manual_seed(seed + i)
        t = torch.rand(shape, generator=g, dtype=torch.float32) * 2 - 1
        out.append(Buffer(shape, "f32", t.numpy().tobytes()))
    return out


def _np(buf):
    return np.frombuffer(buf.data, dtype=np.float32).reshape(buf.shape)


def _run(module, name, args, precision):
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    b2.configure(precision=precision, strict=True)
    try:
        machine.run(module, name, args, engine=b2.engine)
    finally:
        b2.configure(precision="exact", strict=False)
    return list(b2.engine.last_plan)


def _f32_chain(c0, a, b):
    c = c0.astype(np.float32).copy()
    for k in range(a.shape[1]):
        c = (c + (a[:, k] * b[:, k]).astype(np.float32)).astype(np.float32)
    return c


def _plan_cta(plan):
    notes = [n for p in plan for n in (p[4] if len(p) > 4 else ()) if n.startswith("tile")]
    return notes


@pytest.mark.parametrize("precision,tile", [(p, t) for p in ("exact", "bf16", "tf32")
                                            for t in ("8x8", "4x16")] +
                         [("exact", "16x4"), ("exact", "2x2")])
def test_tiled_matmul_4096(tile, precision):
    import bench_kernels as bk
    from paper_2307_16080_b200.runtime import cta_tile

    pipe, sizes = TILES[tile]
    fn = bk.mm_par4096
    module = harness.transformed(fn, pipe)
    args = _inputs(fn)
    A, B, C0 = (_np(a).copy() for a in args)
    plan = _run(module, fn.__name__, args, precision)
    want_kernel = {"exact": "gemm_f32_exact", "bf16": "gemm_tc_bf16", "tf32": "gemm_tc_tf32"}
    assert plan[-1][0] == want_kernel[precision], plan
    bm, bn = cta_tile(precision, sizes)
    assert _plan_cta(plan) == [f"tile{sizes[0]}x{sizes[1]}->cta{bm}x{bn}"], plan
    C = _np(args[2])
    rng = np.random.default_rng(11)
    i, k = rng.integers(0, 4096, SAMPLES), rng.integers(0, 4096, SAMPLES)
    if precision == "exact":
        want = _f32_chain(C0[i, k], A[i, :], B[:, k].T)
        assert np.array_equal(C[i, k].view(np.int32), want.view(np.int32))
        return
    r = tcbound.rounder(precision)
    a, b = r(A[i, :]).astype(np.float64), r(B[:, k].T).astype(np.float64)
    prod = a * b
    want = C0[i, k].astype(np.float64) + prod.sum(axis=1)
    tcbound.check(C[i, k], want, np.abs(prod).sum(axis=1), 4096,
                  f"mm4096 tiled {tile} {precision}")


@pytest.mark.parametrize("tile", ["8x8", "4x16"])
def test_tiled_linear_stack_bf16(tile):
    """The Linear stack (fill / contraction / bias nests, 8192 rows) tiled by
    the reference pass: both layers on the tensor cores with the fused fill
    and bias, the bf16 shadow of H still feeding the second layer."""
    import bench_kernels as bk

    pipe, sizes = TILES[tile]
    fn = bk.make_linear_stack(8192)
    module = harness.transformed(fn, pipe)
    args = _inputs(fn)
    X, W1, b1, _, W2, b2v, _ = (_np(a).copy() for a in args)
    plan = _run(module, fn.__name__, args, "bf16")
    assert [p[0] for p in plan] == ["gemm_tc_bf16", "gemm_tc_bf16"], plan
    assert all(any(n.startswith(f"tile{sizes[0]}x{sizes[1]}") for n in p[4]) for p in plan)
    H, Y = _np(args[3]), _np(args[6])
    rows = np.random.default_rng(5).integers(0, 8192, 8)
    x16, w1 = tcbound.bf16(X[rows]).astype(np.float64), tcbound.bf16(W1).astype(np.float64)
    want_h = x16 @ w1 + b1.astype(np.float64)
    tcbound.check(H[rows], want_h, np.abs(x16) @ np.abs(w1) + np.abs(b1), 1024,
                  f"linear stack layer 1 tiled {tile}")
    h16, w2 = tcbound.bf16(H[rows]).astype(np.float64), tcbound.bf16(W2).astype(np.float64)
    want_y = h16 @ w2 + b2v.astype(np.float64)
    tcbound.check(Y[rows], want_y, np.abs(h16) @ np.abs(w2) + np.abs(b2v), 4096,
                  f"linear stack layer 2 tiled {tile}")


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_untiled_matmul_4096_tight(precision):
    """The untiled affine matmul 4096^3 (the default bench nest) through run():
    bf16 takes b200_gemm_tc_kn (B read MN-major), tf32 the K-major kernel."""
    import bench_kernels as bk

    fn = bk.mm4096
    args = _inputs(fn)
    A, B, C0 = (_np(a).copy() for a in args)
    plan = _run(fn.module, fn.__name__, args, precision)
    assert plan[-1][0] == f"gemm_tc_{precision}"
    C = _np(args[2])
    rng = np.random.default_rng(12)
    i, k = rng.integers(0, 4096, SAMPLES), rng.integers(0, 4096, SAMPLES)
    r = tcbound.rounder(precision)
    a, b = r(A[i, :]).astype(np.float64), r(B[:, k].T).astype(np.float64)
    prod = a * b
    want = C0[i, k].astype(np.float64) + prod.sum(axis=1)
    tcbound.check(C[i, k], want, np.abs(prod).sum(axis=1), 4096, f"mm4096 {precision}")


def test_precision_fallback_is_reported():
    """A bf16 request a contraction cannot honour (K not 16-byte aligned)
    warns, is noted in the plan and raises under strict."""
    import warnings

    import corpus
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200.runtime import PrecisionFallback, PrecisionUnavailable
    from staircase.interp import machine

    fn = corpus.matmul_odd          # K = 150: bf16 rows of 300 bytes
    args = harness.make_args(fn, 0)
    b2.configure(precision="bf16")
    try:
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            machine.run(fn.module, fn.__name__, args, engine=b2.engine)
        assert any(issubclass(x.category, PrecisionFallback) for x in w)
        plan = b2.engine.last_plan
        assert plan[-1][0] == "gemm_f32_exact"
        assert any("bf16 requested" in n for n in plan[-1][4])
        b2.configure(strict=True)
        with pytest.raises(PrecisionUnavailable):
            machine.run(fn.module, fn.__name__, harness.make_args(fn, 0), engine=b2.engine)
    finally:
        b2.configure(precision="exact", strict=False)
