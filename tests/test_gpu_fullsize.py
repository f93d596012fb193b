"""Parity at BASELINE.json's full sizes (run with -m gpu on a B200).

The oracle cannot run 4096^3 or the N=256 ResNet conv in test time, so the
full-size runs through staircase's run() with the B200 engine are checked
on sampled outputs, each recomputed independently in numpy:

* exact paths — the reference's own arithmetic: a sequential f32 chain,
  every product and sum rounded to f32 (no FMA), in nest order
  (interp/_evalpy.py:115-127); must match bit for bit;
* bf16 tensor-core paths — float64 sums of the bf16-rounded operands, within
  |got - want| <= 2 K 2^-24 sum|a b| + 4 2^-24 |want|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SAMPLES = 64


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


def _f32_chain(c0, a, b):
    """c = f32(c + f32(a_k * b_k)) for k in order; a, b: (samples, K)."""
    c = c0.astype(np.float32).copy()
    for k in range(a.shape[1]):
        c = (c + (a[:, k] * b[:, k]).astype(np.float32)).astype(np.float32)
    return c


def _bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).float().numpy()


def _run(fn, args, precision):
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    b2.configure(precision=precision)
    try:
        machine.run(fn.module, fn.__name__, args, engine=b2.engine)
    finally:
        b2.configure(precision="exact")
    return list(b2.engine.last_plan)


def test_matmul_4096_exact_bit_identical():
    import bench_kernels as bk

    args = _inputs(bk.mm4096)
    A, B, C0 = (_np(a).copy() for a in args)
    plan = _run(bk.mm4096, args, "exact")
    assert plan[-1][0] == "gemm_f32_exact"
    C = _np(args[2])
    rng = np.random.default_rng(1)
    i, k = rng.integers(0, 4096, SAMPLES), rng.integers(0, 4096, SAMPLES)
    want = _f32_chain(C0[i, k], A[i, :], B[:, k].T)
    assert np.array_equal(C[i, k].view(np.int32), want.view(np.int32))


def test_conv_resnet_exact_bit_identical():
    import bench_kernels as bk

    fn = bk.make_conv(256)
    args = _inputs(fn)
    X, W, O0 = (_np(a).copy() for a in args)
    plan = _run(fn, args, "exact")
    assert plan[-1][0] == "conv2d_exact"
    O = _np(args[2])
    rng = np.random.default_rng(2)
    n, f = rng.integers(0, 256, SAMPLES), rng.integers(0, 64, SAMPLES)
    h, w = rng.integers(0, 56, SAMPLES), rng.integers(0, 56, SAMPLES)
    # terms in nest order ci -> ki -> kj
    xs = np.stack([X[n, c, h + ki, w + kj] for c in range(64) for ki in range(3)
                   for kj in range(3)], axis=1)
    ws = np.stack([W[f, c, ki, kj] for c in range(64) for ki in range(3)
                   for kj in range(3)], axis=1)
    want = _f32_chain(O0[n, f, h, w], xs, ws)
    assert np.array_equal(O[n, f, h, w].view(np.int32), want.view(np.int32))


def _check_bound(got, want, mag, K):
    bound = 2 * K * 2.0 ** -24 * mag + 4 * 2.0 ** -24 * np.abs(want) + 1e-30
    bad = np.abs(got.astype(np.float64) - want) > bound
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside the bound"


def test_conv_resnet_bf16_within_bound():
    import bench_kernels as bk

    fn = bk.make_conv(256)
    args = _inputs(fn)
    X, W, O0 = (_np(a).copy() for a in args)
    plan = _run(fn, args, "bf16")
    assert plan[-1][0] == "conv2d_tc_bf16"
    O = _np(args[2])
    rng = np.random.default_rng(3)
    n, f = rng.integers(0, 256, SAMPLES), rng.integers(0, 64, SAMPLES)
    h, w = rng.integers(0, 56, SAMPLES), rng.integers(0, 56, SAMPLES)
    xs = _bf16(np.stack([X[n, :, h + ki, w + kj] for ki in range(3) for kj in range(3)],
                        axis=2)).astype(np.float64)
    ws = _bf16(np.stack([W[f, :, ki, kj] for ki in range(3) for kj in range(3)],
                        axis=2)).astype(np.float64)
    prod = xs * ws
    want = O0[n, f, h, w].astype(np.float64) + prod.sum(axis=(1, 2))
    _check_bound(O[n, f, h, w], want, np.abs(prod).sum(axis=(1, 2)), 64 * 9)


def test_linear_stack_bf16_within_bound():
    """65536 x 1024 -> 4096 -> 1024 with fused fill / bias and the bf16 shadow
    of H feeding the second layer: H and Y checked on sampled rows."""
    import bench_kernels as bk

    fn = bk.make_linear_stack(65536)
    args = _inputs(fn)
    X, W1, b1, _, W2, b2v, _ = (_np(a).copy() for a in args)
    plan = _run(fn, args, "bf16")
    assert [p[0] for p in plan] == ["gemm_tc_bf16", "gemm_tc_bf16"]
    H, Y = _np(args[3]), _np(args[6])
    rows = np.random.default_rng(4).integers(0, 65536, 8)
    x16, w1 = _bf16(X[rows]).astype(np.float64), _bf16(W1).astype(np.float64)
    want_h = x16 @ w1 + b1.astype(np.float64)
    _check_bound(H[rows], want_h, np.abs(x16) @ np.abs(w1) + np.abs(b1), 1024)
    # the second layer consumes bf16(H) — exactly what the shadow / pack hold
    h16, w2 = _bf16(H[rows]).astype(np.float64), _bf16(W2).astype(np.float64)
    want_y = h16 @ w2 + b2v.astype(np.float64)
    _check_bound(Y[rows], want_y, np.abs(h16) @ np.abs(w2) + np.abs(b2v), 4096)


def test_race_check_of_the_resnet_conv_is_proven():
    """check_races at the paper's conv size: the reference simulates 59 GFLOP
    of the nest in Python (hours); the static proof answers after one device
    run, with the same (empty) result."""
    import time

    import bench_kernels as bk
    import paper_2307_16080_b200 as b2
    import staircase.interp.races as ref_races

    fn = bk.make_conv(256)
    args = _inputs(fn)
    saved = ref_races.check_races
    ref_races.check_races = lambda *a, **k: pytest.fail("fell back to the simulation")
    try:
        t0 = time.perf_counter()
        assert b2.check_races(fn.module, fn.__name__, args) == []
        assert time.perf_counter() - t0 < 60
    finally:
        ref_races.check_races = saved
