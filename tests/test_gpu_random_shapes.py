"""Seeded random shapes through the whole engine on the B200, against the C
oracle: matmul nests (plain and row-major-transposed B) and convolutions of
random sizes — odd extents, one-element dimensions, non-square filters —
must be bit-identical (buffers and the 25-slot tally) at exact precision,
and within the stated bf16 bound at bf16 precision.
"""
import os
import random

import numpy as np
import pytest

import bench_kernels as bk
import harness
import oracle

pytestmark = pytest.mark.gpu

# B200_RANDOM_SCALE=k runs k times as many seeds (extended stress runs)
SCALE = max(1, int(os.environ.get("B200_RANDOM_SCALE", "1")))
OFFSET = int(os.environ.get("B200_RANDOM_OFFSET", "0"))   # a fresh range of seeds

MM = '''
@staged
def mm_r(A: MemRef[({M}, {K}), F32], B: MemRef[({K}, {N}), F32], C: MemRef[({M}, {N}), F32]):
    for i, j in parallel((0, 0), ({M}, {N})):
        for k in range(0, {K}):
            C[i, j] += A[i, k] * B[k, j]
'''

CONV = '''
@staged
def conv_r(inp: MemRef[({nb}, {c}, {hp}, {wp}), F32], ker: MemRef[({f}, {c}, {kh}, {kw}), F32],
           out: MemRef[({nb}, {f}, {ho}, {wo}), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), ({nb}, {f}, {ho}, {wo})):
        for ci in range(0, {c}):
            for ki in range(0, {kh}):
                for kj in range(0, {kw}):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]
'''


def _mm_shape(seed):
    r = random.Random(seed)
    return dict(M=r.choice([1, 3, 17, 64, 96, 130, 257]), N=r.choice([1, 8, 31, 64, 72, 200]),
                K=r.choice([1, 5, 16, 33, 64, 100, 136]))


def _conv_shape(seed):
    r = random.Random(1000 + seed)
    kh, kw = r.choice([(1, 1), (3, 3), (5, 5), (1, 3), (3, 1), (2, 4)])
    ho, wo = r.randint(1, 20), r.randint(1, 40)
    return dict(nb=r.randint(1, 3), c=r.choice([1, 3, 8, 16, 20]), f=r.choice([1, 4, 8, 32, 48]),
                ho=ho, wo=wo, hp=ho + kh - 1, wp=wo + kw - 1, kh=kh, kw=kw)


def _both(fn, seed):
    import paper_2307_16080_b200 as b2

    _, got, t_got, _ = harness.run_engine(b2.engine, fn, None, "sequential", seed)
    plan = list(b2.engine.last_plan)
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", seed)
    return got, t_got, want, t_want, plan


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 30 * SCALE))
def test_random_matmul_exact(seed):
    shp = _mm_shape(seed)
    fn = bk._capture_from_source(MM.format(**shp), "mm_r", {}, "_".join(map(str, shp.values())))
    got, t_got, want, t_want, plan = _both(fn, seed)
    assert t_got == t_want, plan
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes(), (shp, plan)


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 30 * SCALE))
def test_random_conv_exact(seed):
    shp = _conv_shape(seed)
    fn = bk._capture_from_source(CONV.format(**shp), "conv_r", {},
                                 "_".join(map(str, shp.values())))
    got, t_got, want, t_want, plan = _both(fn, seed)
    assert t_got == t_want, plan
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes(), (shp, plan)


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 16 * SCALE))
def test_random_matmul_bf16_within_bound(seed):
    """bf16 precision on bf16-representable inputs: every output within
    2 K 2^-24 sum|a b| + 4 2^-24 |want| of the float64 result."""
    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    shp = _mm_shape(100 + seed)
    M, N, K = shp["M"], shp["N"], shp["K"]
    fn = bk._capture_from_source(MM.format(**shp), "mm_r", {}, "_".join(map(str, shp.values())))
    rng = np.random.default_rng(seed)

    def bf16(x):
        import torch

        return torch.from_numpy(x).bfloat16().float().numpy()

    A = bf16(rng.uniform(-1, 1, (M, K)).astype(np.float32))
    B = bf16(rng.uniform(-1, 1, (K, N)).astype(np.float32))
    C = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    args = [Buffer(x.shape, "f32", x.tobytes()) for x in (A, B, C)]
    b2.configure(precision="bf16")
    try:
        machine.run(fn.module, "mm_r", args, engine=b2.engine)
    finally:
        b2.configure(precision="exact")
    got = np.frombuffer(args[2].data, dtype=np.float32).reshape(M, N).astype(np.float64)
    want = C.astype(np.float64) + A.astype(np.float64) @ B.astype(np.float64)
    mag = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    bound = 2 * K * 2.0 ** -24 * mag + 4 * 2.0 ** -24 * np.abs(want) + 1e-30
    assert (np.abs(got - want) <= bound).all(), (shp, b2.engine.last_plan)


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 20 * SCALE))
def test_random_tile_unroll_pipelines_exact(seed):
    """The sweep's knobs on random nests: random tile sizes (tiling applies
    only where they divide the trip counts) and unroll factors on random
    matmul / conv shapes; engine == oracle, bit for bit, tally included."""
    import paper_2307_16080_b200 as b2
    from staircase.tuner.search import default_pipeline

    r = random.Random(5000 + seed)
    if seed % 2 == 0:
        shp = _mm_shape(200 + seed)
        fn = bk._capture_from_source(MM.format(**shp), "mm_r", {},
                                     "_".join(map(str, shp.values())))
        tiles = [r.choice([1, 2, 4, 8, 16]) for _ in range(2)]
    else:
        shp = _conv_shape(200 + seed)
        fn = bk._capture_from_source(CONV.format(**shp), "conv_r", {},
                                     "_".join(map(str, shp.values())))
        tiles = [r.choice([1, 2, 4, 8]) for _ in range(4)]
    pipe = default_pipeline(tiles, r.choice([1, 2, 3, 4]))
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, pipe, "sequential", seed)
    plan = list(b2.engine.last_plan)
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, pipe, "sequential", seed)
    assert t_got == t_want, (shp, pipe, plan)
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes(), (shp, pipe, plan)


def _ewise_src(seed):
    r = random.Random(7000 + seed)
    rows, cols = r.choice([1, 3, 16, 33, 64]), r.choice([1, 4, 7, 64, 100, 256])

    def expr(d):
        if d == 0 or r.random() < 0.3:
            return r.choice(["a[i, j]", "b[i, j]", f"constant({r.uniform(-3, 3):.6f}, F32)"])
        return f"({expr(d - 1)} {r.choice(['+', '-', '*', '/'])} {expr(d - 1)})"

    body = expr(3)
    src = f'''
@staged
def ew_r(a: MemRef[({rows}, {cols}), F32], b: MemRef[({rows}, {cols}), F32],
         c: MemRef[({rows}, {cols}), F32]):
    for i, j in parallel((0, 0), ({rows}, {cols})):
        c[i, j] = {body}
'''
    return src, f"{rows}_{cols}_{seed}"


@pytest.mark.parametrize("jit_on", [True, False], ids=["nvrtc", "map_f32"])
@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 20 * SCALE))
def test_random_elementwise_exact(seed, jit_on, monkeypatch):
    """Random f32 expression trees (+ - * / and constants, depth <= 3) over
    random shapes, as pointwise NVRTC kernels: bit-identical to the oracle
    (per-op rounding, no contraction).  Quotients of random values can be
    inf or NaN; those compare by class, finite values bit for bit."""
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import jit

    monkeypatch.setattr(jit, "ENABLED", jit_on)   # off: the b200_map_f32 kernel
    src, key = _ewise_src(seed)
    fn = bk._capture_from_source(src, "ew_r", {}, key)
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, None, "sequential", seed)
    plan = list(b2.engine.last_plan)
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", seed)
    assert t_got == t_want, plan
    g = np.frombuffer(got[2].data, dtype=np.float32)
    w = np.frombuffer(want[2].data, dtype=np.float32)
    assert np.array_equal(np.isnan(g), np.isnan(w)), (src, plan)
    fin = ~np.isnan(w)
    assert np.array_equal(g[fin].view(np.int32), w[fin].view(np.int32)), (src, plan)


def _irregular_src(seed):
    r = random.Random(9000 + seed)
    n = r.choice([5, 16, 33, 64])
    thr = f"{r.uniform(-0.5, 0.5):.4f}"
    k1, k2 = f"{r.uniform(-2, 2):.4f}", f"{r.uniform(-2, 2):.4f}"
    kind = seed % 3
    if kind == 0:    # triangular, reads what earlier iterations wrote
        body = f'''
    for i in range(1, {n}):
        for j in range(i):
            v = a[i, j] + a[j, i] * constant({k1}, F32)
            if v > constant({thr}, F32):
                a[i, j] = v
            else:
                a[i, j] = a[i - 1, j] - v'''
    elif kind == 1:  # running sums along rows (loop-carried)
        body = f'''
    for i in range(0, {n}):
        for j in range(1, {n}):
            a[i, j] = a[i, j - 1] * constant({k1}, F32) + a[i, j]'''
    else:            # data-dependent branch inside a parallel nest
        body = f'''
    for i, j in parallel((0, 0), ({n}, {n})):
        v = a[i, j]
        if v > constant({thr}, F32):
            b[i, j] = v * constant({k1}, F32)
        else:
            b[i, j] = v + constant({k2}, F32)'''
    src = f'''
@staged
def irr_r(a: MemRef[({n}, {n}), F32], b: MemRef[({n}, {n}), F32]):{body}
'''
    return src, f"{n}_{seed}"


@pytest.mark.parametrize("native", [True, False], ids=["native", "interpreter"])
@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 15 * SCALE))
def test_random_irregular_nests_exact(seed, native, monkeypatch):
    """Nests no template matches (triangular bounds, loop-carried updates,
    data-dependent branches) run as NVRTC-specialised VM programs — or, with
    the native tier off, on the device VM interpreter: buffers and tally
    bit-identical to the oracle either way."""
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import native as nat

    monkeypatch.setattr(nat, "ENABLED", native)

    src, key = _irregular_src(seed)
    fn = bk._capture_from_source(src, "irr_r", {}, key)
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, None, "sequential", seed)
    plan = list(b2.engine.last_plan)
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", seed)
    assert t_got == t_want, (src, plan)
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes(), (src, plan)


@pytest.mark.parametrize("shape", [(4096, 4096, 8), (3900, 4096, 12), (4096, 4000, 5)])
def test_exact_gemm_balanced_last_round(shape, monkeypatch):
    """Shapes whose 128 x 128 tile count leaves a short last round run that
    round as half-width tiles (gemm_exact.cu launch_128): C must still be
    the reference's per-op-rounded f32 chain, bit for bit (numpy float32
    emulation of the chain in k order)."""
    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    monkeypatch.setenv("B200_GEMM_EXACT_TAIL", "1")   # the split is opt-in
    M, N, K = shape
    fn = bk._capture_from_source(MM.format(M=M, N=N, K=K), "mm_r", {}, f"{M}_{N}_{K}")
    rng = np.random.default_rng(M + N + K)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    args = [Buffer(x.shape, "f32", x.tobytes()) for x in (A, B, C)]
    machine.run(fn.module, "mm_r", args, engine=b2.engine)
    assert b2.engine.last_plan[-1][0] == "gemm_f32_exact"
    want = C.copy()
    for k in range(K):
        want = (want + (A[:, k, None] * B[None, k, :]).astype(np.float32)).astype(np.float32)
    got = np.frombuffer(args[2].data, dtype=np.float32).reshape(M, N)
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + 12 * SCALE))
def test_random_conv_bf16_within_bound(seed):
    """The tensor-core conv (F in {32, 64, 128}; 1x1, 3x3, 5x5; random
    batch, channels and sizes) on bf16-representable inputs: every output
    within 2 K 2^-24 sum|x w| + 4 2^-24 |want| of the float64 conv."""
    import torch
    import torch.nn.functional as Fn

    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    r = random.Random(11000 + seed)
    f, (kh, kw) = r.choice([(32, (3, 3)), (64, (3, 3)), (32, (5, 5)), (64, (1, 1)),
                            (128, (1, 1)), (128, (3, 3))])
    nb, c = r.randint(1, 3), r.choice([8, 16, 64, 70, 128])
    ho, wo = r.randint(1, 24), r.randint(1, 40)
    hp, wp = ho + kh - 1, wo + kw - 1
    shp = dict(nb=nb, c=c, f=f, ho=ho, wo=wo, hp=hp, wp=wp, kh=kh, kw=kw)
    fn = bk._capture_from_source(CONV.format(**shp), "conv_r", {},
                                 "_".join(map(str, shp.values())))
    g = torch.Generator().manual_seed(seed)
    x = (torch.rand(nb, c, hp, wp, generator=g) * 2 - 1).bfloat16().float()
    w = (torch.rand(f, c, kh, kw, generator=g) * 2 - 1).bfloat16().float()
    o = torch.rand(nb, f, ho, wo, generator=g) * 2 - 1
    args = [Buffer(tuple(t.shape), "f32", t.numpy().tobytes()) for t in (x, w, o)]
    b2.configure(precision="bf16")
    try:
        machine.run(fn.module, "conv_r", args, engine=b2.engine)
    finally:
        b2.configure(precision="exact")
    got = torch.frombuffer(args[2].data, dtype=torch.float32).reshape(nb, f, ho, wo).double()
    want = o.double() + Fn.conv2d(x.double(), w.double())
    mag = Fn.conv2d(x.double().abs(), w.double().abs())
    bound = 2 * c * kh * kw * 2.0 ** -24 * mag + 4 * 2.0 ** -24 * want.abs() + 1e-30
    # the tensor-core kernel keeps the whole filter resident in shared memory
    # (runtime.conv_tc_supported); e.g. 5x5 over two 64-channel blocks does
    # not fit and takes the exact kernel
    from types import SimpleNamespace

    from paper_2307_16080_b200.runtime import conv_tc_supported

    fits = conv_tc_supported(SimpleNamespace(c=c, f=f, kh=kh, kw=kw, wo=wo))
    kernels = {"conv2d_tc_bf16" if fits else "conv2d_exact"}
    if kh == kw == 1:
        kernels.add("gemm_tc_bf16")   # a 1x1 conv with a single row/column is a strided GEMM
    assert b2.engine.last_plan[-1][0] in kernels, (shp, b2.engine.last_plan)
    assert ((got - want).abs() <= bound).all(), (shp, b2.engine.last_plan)


def test_constant_operands_are_rounded_at_run_time():
    """(c1 - c2) with both operands constants, found by the extended random
    run (seed 362): ptxas folds an f32 sub of two immediates without ties-
    to-even (0x3f065226 - 0x4027a8c1 -> 0xc0061437; the reference and the
    hardware FADD give 0xc0061438).  The NVRTC tiers read such constants
    from a __constant__ table, so the subtraction runs on the device."""
    import paper_2307_16080_b200 as b2

    src = '''
@staged
def ew_c(a: MemRef[(3, 1), F32], b: MemRef[(3, 1), F32], c: MemRef[(3, 1), F32]):
    for i, j in parallel((0, 0), (3, 1)):
        c[i, j] = (((constant(0.524691, F32) - constant(2.619675, F32)) *
                    (a[i, j] + constant(-1.845358, F32))) * a[i, j])
'''
    fn = bk._capture_from_source(src, "ew_c", {}, "fold")
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, None, "sequential", 362)
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", 362)
    assert t_got == t_want
    assert got[2].data.tobytes() == want[2].data.tobytes()
