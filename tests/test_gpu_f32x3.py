"""The fp32-accurate tensor-core contraction, precision "f32x3" (-m gpu).

Each f32 operand is split x = hi + lo + d with hi = tf32(x), lo = tf32(x -
hi), |d| <= 2^-22 |x| (b200_pack_operand kinds 2 / 3); one tf32 tcgen05 GEMM
over K' = 3K sums hiA.hiB + hiA.loB + loA.hiB (the dropped loA.loB is
<= 2^-22 |ab|).  Inputs are NOT pre-rounded: this is the reference's f32
problem.  Tolerance (north_star "fp32 rel 1e-5", relative to the magnitude
of the dot product):

    |got - want| <= 1e-5 * sum_k |a_k b_k|

per output, ``want`` the reference's own result — the sequential f32 chain,
every product and sum rounded (interp/_evalpy.py:115-127) — so the bound
covers both the split error and the two summation orders.  The observed
maximum is recorded (conftest.TC_ERRORS, printed in the summary).
"""
import ctypes

import numpy as np
import pytest

import conftest

pytestmark = pytest.mark.gpu

TOL = 1e-5


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
    c = c0.astype(np.float32).copy()
    for k in range(a.shape[1]):
        c = (c + (a[:, k] * b[:, k]).astype(np.float32)).astype(np.float32)
    return c


def _check(got, want, mag, label, K):
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    norm = float((err / mag).max())
    conftest.TC_ERRORS.append((label, K, norm,
                               "f32x3: |got-want| / sum|ab| vs the reference chain, bound 1e-5"))
    assert (err <= TOL * mag).all(), f"{label}: max normalised error {norm:.3g}"
    return norm


def _run(module, name, args, precision):
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    b2.configure(precision=precision, strict=True)
    try:
        machine.run(module, name, args, engine=b2.engine)
    finally:
        b2.configure(precision="exact", strict=False)
    return list(b2.engine.last_plan)


@pytest.mark.parametrize("tiles", [None, "8x8"])
def test_mm4096_f32x3_within_fp32_tolerance(tiles):
    import bench_kernels as bk
    import harness

    fn = bk.mm_par4096 if tiles else bk.mm4096
    module = harness.transformed(fn, harness.TILE88 if tiles else None)
    args = _inputs(fn)
    A, B, C0 = (_np(a).copy() for a in args)
    plan = _run(module, fn.__name__, args, "f32x3")
    assert plan[-1][0] == "gemm_tc_f32x3", plan
    C = _np(args[2])
    rng = np.random.default_rng(21)
    i, k = rng.integers(0, 4096, 64), rng.integers(0, 4096, 64)
    want = _f32_chain(C0[i, k], A[i, :], B[:, k].T)
    mag = np.abs(A[i, :].astype(np.float64) * B[:, k].T.astype(np.float64)).sum(axis=1) + \
        np.abs(C0[i, k])
    _check(C[i, k], want, mag, f"mm4096 f32x3 tiles={tiles}", 4096)


@pytest.mark.parametrize("shape", [(96, 200, 160), (130, 72, 148), (256, 256, 1024)])
def test_random_f32x3_vs_oracle(shape, oracle_engine):
    """Parallel-form matmuls (odd M / N) against the oracle's exact result."""
    from staircase import F32, MemRef, parallel, staged  # noqa: F401
    import harness

    M, N, K = shape
    src = f'''
@staged
def mmx(A: MemRef[({M}, {K}), F32], B: MemRef[({K}, {N}), F32], C: MemRef[({M}, {N}), F32]):
    for i, k in parallel((0, 0), ({M}, {N})):
        for j in range({K}):
            C[i, k] += A[i, j] * B[j, k]
'''
    import bench_kernels as bk

    fn = bk._capture_from_source(src, "mmx", {"F32": F32, "MemRef": MemRef,
                                                "parallel": parallel, "staged": staged},
                                 f"f32x3_{M}_{N}_{K}")
    args = harness.make_args(fn, 3)
    want = harness.make_args(fn, 3)
    from staircase.interp import machine

    machine.run(fn.module, "mmx", want, engine=oracle_engine)
    plan = _run(fn.module, "mmx", args, "f32x3")
    assert plan[-1][0] == "gemm_tc_f32x3", plan
    A = np.array(want[0].data, dtype=np.float64).reshape(M, K)
    B = np.array(want[1].data, dtype=np.float64).reshape(K, N)
    C0 = np.array(harness.make_args(fn, 3)[2].data, dtype=np.float64).reshape(M, N)
    mag = np.abs(A) @ np.abs(B) + np.abs(C0)
    _check(_np(args[2]), _np(want[2]), mag, f"mm {M}x{N}x{K} f32x3", K)


def test_split_pack_layout():
    """kind 2 -> [hi | hi | lo], kind 3 -> [hi | lo | hi]; hi = tf32_rn(x),
    lo = tf32_rn(x - hi), for row-contiguous and transposed sources."""
    import torch

    import tcbound
    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.rand(64, 96, device="cuda", generator=g) * 2 - 1
    x = X.cpu().numpy()
    hi = tcbound.tf32(x)
    lo = tcbound.tf32((x - hi).astype(np.float32))
    for kind, segs in ((2, (hi, hi, lo)), (3, (hi, lo, hi))):
        out = torch.empty(64, 3 * 96, device="cuda")
        assert lib.b200_pack_operand(kind, P(X.data_ptr()), 96, 1, P(out.data_ptr()), 64, 96,
                                     s) == 0
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), np.concatenate(segs, axis=1))
        XT = X.t().contiguous()   # the same matrix read column-contiguous
        out2 = torch.empty(64, 3 * 96, device="cuda")
        assert lib.b200_pack_operand(kind, P(XT.data_ptr()), 1, 64, P(out2.data_ptr()), 64, 96,
                                     s) == 0
        torch.cuda.synchronize()
        assert torch.equal(out, out2)
