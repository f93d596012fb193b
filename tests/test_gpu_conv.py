"""Tensor-core convolution (b200_conv2d_tc) through the engine, on a B200.

The conv_2d_nchw_fchw nest (reference tests/kernels.py:50-64) is run with
``configure(precision="bf16")``; inputs and weights are pre-rounded to bf16
so every product is exact in fp32 and the deviation from the reference's
sequential f32 chain is accumulation order only.  Bound per output
(K = C*KH*KW terms):

    |got - want| <= 2*K*2^-24 * sum|in*w| + 4*2^-24*|want|

with ``want`` = out0 + conv(in, w) computed in float64.
"""
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # nb, c, f, ho, wo, kh, kw
    (2, 64, 64, 56, 56, 3, 3),      # the ResNet-50 layer of BASELINE configs[2], 2 images
    (1, 16, 32, 20, 12, 3, 3),      # ragged tiles, channels padded to 64
    (3, 128, 32, 17, 24, 3, 3),     # two channel blocks per tap
    (1, 64, 128, 16, 16, 1, 1),     # F = 128, 1x1
    (1, 16, 32, 20, 13, 3, 3),      # Wo = 13: output rows not 16-byte multiples
    (2, 64, 128, 18, 20, 3, 3),     # F = 128 3x3: unmerged 16 x 8 tiling
    (1, 32, 32, 12, 21, 5, 5),      # 5x5 merged into N = 160
    (2, 100, 64, 14, 14, 3, 3),     # C = 100: second channel block zero-padded by the TMA pack
]


def _conv_kernel(nb, c, f, ho, wo, kh, kw):
    import bench_kernels as bk

    hp, wp = ho + kh - 1, wo + kw - 1
    src = f'''
@staged
def conv_t(inp: MemRef[({nb}, {c}, {hp}, {wp}), F32], ker: MemRef[({f}, {c}, {kh}, {kw}), F32],
           out: MemRef[({nb}, {f}, {ho}, {wo}), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), ({nb}, {f}, {ho}, {wo})):
        for ci in range(0, {c}):
            for ki in range(0, {kh}):
                for kj in range(0, {kw}):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]
'''
    return bk._capture_from_source(src, "conv_t", {}, f"{nb}_{c}_{f}_{ho}_{wo}_{kh}_{kw}")


def test_unsupported_filter_count_takes_the_exact_path():
    """F = 48 has no tensor-core instantiation: exact kernel, bit-exact."""
    import torch

    import oracle
    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    fn = _conv_kernel(1, 16, 48, 20, 13, 3, 3)
    g = torch.Generator().manual_seed(3)
    ts = [torch.rand(s, generator=g) * 2 - 1 for s in ((1, 16, 22, 15), (48, 16, 3, 3),
                                                        (1, 48, 20, 13))]
    a1 = [Buffer(tuple(t.shape), "f32", t.numpy().tobytes()) for t in ts]
    a2 = [Buffer(tuple(t.shape), "f32", t.numpy().tobytes()) for t in ts]
    b2.configure(precision="bf16")
    try:
        machine.run(fn.module, "conv_t", a1, engine=b2.engine)
    finally:
        b2.configure(precision="exact")
    assert b2.engine.last_plan[-1][0] == "conv2d_exact"
    oracle.build()
    machine.run(fn.module, "conv_t", a2, engine=oracle)
    assert a1[2].data.tobytes() == a2[2].data.tobytes()


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_conv_tc_through_engine(case):
    import torch
    import torch.nn.functional as Fn

    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    nb, c, f, ho, wo, kh, kw = case
    fn = _conv_kernel(*case)
    g = torch.Generator().manual_seed(7)
    hp, wp = ho + kh - 1, wo + kw - 1
    x = (torch.rand(nb, c, hp, wp, generator=g) * 2 - 1).bfloat16().float()
    w = (torch.rand(f, c, kh, kw, generator=g) * 2 - 1).bfloat16().float()
    o = torch.rand(nb, f, ho, wo, generator=g) * 2 - 1
    args = [Buffer(tuple(t.shape), "f32", t.numpy().tobytes()) for t in (x, w, o)]
    b2.configure(precision="bf16")
    try:
        machine.run(fn.module, "conv_t", args, engine=b2.engine)
    finally:
        b2.configure(precision="exact")
    assert b2.engine.last_plan[-1][0] == "conv2d_tc_bf16", b2.engine.last_plan
    got = torch.frombuffer(args[2].data, dtype=torch.float32).reshape(nb, f, ho, wo).double()
    want = o.double() + Fn.conv2d(x.double(), w.double())
    mag = Fn.conv2d(x.double().abs(), w.double().abs())
    K = c * kh * kw
    bound = 2 * K * 2.0 ** -24 * mag + 4 * 2.0 ** -24 * want.abs() + 1e-30
    bad = ((got - want).abs() > bound).sum().item()
    assert bad == 0, f"{bad} outputs outside the bound"
    # inputs are untouched
    assert torch.equal(torch.frombuffer(args[0].data, dtype=torch.float32).reshape(x.shape), x)


EXACT_CASES = [
    # nb, c, f, ho, wo, dtype
    (2, 64, 64, 56, 56, "F32"),     # the ResNet layer's shape, 2 images (56-wide runs tiles)
    (1, 16, 48, 10, 40, "F32"),     # ragged rows (10 = 2 x 4 + 2), F = 48 < 64
    (1, 12, 30, 9, 37, "F32"),      # F = 30: scalar weight staging; odd width
    (2, 8, 20, 7, 56, "F64"),       # f64 (the reference's desk kernels)
    (1, 20, 16, 13, 20, "F32"),     # narrow: 32-wide tiles
]


@pytest.mark.parametrize("variant", ["auto", "old", "rows", "runs"])
@pytest.mark.parametrize("case", EXACT_CASES, ids=[str(c) for c in EXACT_CASES])
def test_conv_exact_variants_bit_identical(case, variant, monkeypatch):
    """Every variant of b200_conv2d_exact (generic, 32-wide rows, 56-wide
    runs) reproduces the reference's f32 / f64 chain bit for bit."""
    import torch

    import bench_kernels as bk
    import oracle
    import paper_2307_16080_b200 as b2
    from staircase.interp import Buffer, machine

    nb, c, f, ho, wo, dt = case
    if variant != "auto":
        monkeypatch.setenv("B200_CONV_EXACT", variant)
    hp, wp = ho + 2, wo + 2
    src = f'''
@staged
def conv_e(inp: MemRef[({nb}, {c}, {hp}, {wp}), {dt}], ker: MemRef[({f}, {c}, 3, 3), {dt}],
           out: MemRef[({nb}, {f}, {ho}, {wo}), {dt}]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), ({nb}, {f}, {ho}, {wo})):
        for ci in range(0, {c}):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]
'''
    fn = bk._capture_from_source(src, "conv_e", {}, f"{nb}_{c}_{f}_{ho}_{wo}_{dt}")
    tdt, bdt = (torch.float32, "f32") if dt == "F32" else (torch.float64, "f64")
    g = torch.Generator().manual_seed(11)
    ts = [(torch.rand(s, generator=g, dtype=torch.float64) * 2 - 1).to(tdt)
          for s in ((nb, c, hp, wp), (f, c, 3, 3), (nb, f, ho, wo))]
    a1 = [Buffer(tuple(t.shape), bdt, t.numpy().tobytes()) for t in ts]
    a2 = [Buffer(tuple(t.shape), bdt, t.numpy().tobytes()) for t in ts]
    machine.run(fn.module, "conv_e", a1, engine=b2.engine)
    assert b2.engine.last_plan[-1][0] == "conv2d_exact", b2.engine.last_plan
    oracle.build()
    machine.run(fn.module, "conv_e", a2, engine=oracle)
    assert a1[2].data.tobytes() == a2[2].data.tobytes()


@pytest.mark.parametrize("sizes,unroll", [("1, 1, 4, 8", 1), ("1, 2, 8, 7", 3), ("2, 4", 1),
                                          ("1, 1, 2, 2", 3)])
def test_tiled_conv_takes_the_direct_kernel_bit_exact(sizes, unroll):
    """Tiled (and unrolled) conv nests — the sweep's configurations — are
    recognised as convolutions (origin + offset loops per output role) and
    run on the direct exact kernel, bit-identical to the reference."""
    import harness
    import oracle
    import paper_2307_16080_b200 as b2
    from staircase.tuner.search import default_pipeline

    fn = _conv_kernel(2, 16, 8, 16, 28, 3, 3)
    pipe = default_pipeline([int(x) for x in sizes.split(",")], unroll)
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, pipe, "sequential", 4)
    assert b2.engine.last_plan[-1][0] == "conv2d_exact", b2.engine.last_plan
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, pipe, "sequential", 4)
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()
