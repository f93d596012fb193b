"""Tensor-core contraction (b200_gemm_tc, tcgen05) on a real B200.

Inputs are pre-rounded to the kernel's operand type (bf16 / tf32) so every
product is exact in fp32 and the only deviation from the reference's
sequential per-op-rounded f32 chain is accumulation rounding.  Tolerance
(stated here and in DESIGN.md):

    |got - want| <= 2 * K * 2^-24 * sum_k |a_mk * b_kn|  + 1e-30

per output, where ``want`` is the exact (float64) sum of the same rounded
products plus the initial C.  This is the standard γ_K bound for any fp32
summation order (the reference's own chain obeys it too).
"""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def _round(t, kind):
    import torch

    if kind == 0:
        return t.to(torch.bfloat16).to(torch.float32)
    u = t.view(torch.int32)
    u = (u + 0xFFF + ((u >> 13) & 1)) & ~0x1FFF
    return u.view(torch.float32)


def _run(kind, M, N, K, init=0, bias=False, trans_b=False, seed=0, max_ctas=0, variant=0):
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = _round(torch.rand(M, K, device="cuda", generator=g) * 2 - 1, kind)
    if trans_b:
        Bsrc = _round(torch.rand(N, K, device="cuda", generator=g) * 2 - 1, kind)
        sBk, sBn = 1, K
        B = Bsrc.t()
    else:
        Bsrc = _round(torch.rand(K, N, device="cuda", generator=g) * 2 - 1, kind)
        sBk, sBn = N, 1
        B = Bsrc
    C = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
    bvec = torch.rand(N, device="cuda", generator=g) if bias else None
    C0 = C.clone()
    elt = torch.bfloat16 if kind == 0 else torch.float32
    Ap = torch.empty(M, K, dtype=elt, device="cuda")
    Bp = torch.empty(N, K, dtype=elt, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    assert lib.b200_pack_operand(kind, P(A.data_ptr()), K, 1, P(Ap.data_ptr()), M, K, s) == 0
    assert lib.b200_pack_operand(kind, P(Bsrc.data_ptr()), sBn, sBk, P(Bp.data_ptr()),
                                 N, K, s) == 0
    rc = lib.b200_gemm_tc(kind, P(Ap.data_ptr()), P(Bp.data_ptr()), P(C.data_ptr()), N, 1,
                          M, N, K, init, 0.5, P(bvec.data_ptr()) if bias else None, 1,
                          max_ctas, variant, s)
    assert rc == 0
    torch.cuda.synchronize()
    Ad, Bd = A.double(), B.double()
    want = Ad @ Bd + (0.5 if init else C0.double())
    if bias:
        want = want + bvec.double()[None, :]
    mag = Ad.abs() @ Bd.abs()
    err = (C.double() - want).abs()
    bound = 2 * K * 2.0 ** -24 * mag + 4 * 2.0 ** -24 * want.abs() + 1e-30
    return err, bound, Ap, Bp, A, Bsrc


@pytest.mark.parametrize("variant", [1, 2, 3], ids=["cta1", "cta2", "solo"])
@pytest.mark.parametrize("kind", [0, 1], ids=["bf16", "tf32"])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 256), (300, 520, 200),
                                   (1024, 1024, 1024), (2048, 1536, 512)])
def test_gemm_tc_accuracy(kind, shape, variant):
    M, N, K = shape
    if kind == 0 and K % 8:
        pytest.skip("bf16 TMA rows need K % 8 == 0")
    err, bound, *_ = _run(kind, M, N, K, variant=variant)
    bad = (err > bound).sum().item()
    assert bad == 0, f"{bad} outputs outside the bound; max err {err.max().item()}"


@pytest.mark.parametrize("variant", [1, 2, 3], ids=["cta1", "cta2", "solo"])
@pytest.mark.parametrize("kind", [0, 1], ids=["bf16", "tf32"])
def test_gemm_tc_epilogue_modes(kind, variant):
    err, bound, *_ = _run(kind, 512, 512, 128, init=1, bias=True, trans_b=True,
                          variant=variant)
    assert (err > bound).sum().item() == 0


def test_pack_rounding_exact():
    import torch

    err, bound, Ap, Bp, A, Bsrc = _run(0, 128, 256, 64)
    assert torch.equal(Ap.float(), A)
    err, bound, Ap, Bp, A, Bsrc = _run(1, 128, 256, 64)
    assert torch.equal(Ap, A)
    assert torch.equal(Bp, Bsrc.t().contiguous())


@pytest.mark.parametrize("variant", [1, 2, 3], ids=["cta1", "cta2", "solo"])
def test_gemm_tc_few_ctas_persistent_loop(variant):
    # fewer CTAs than tiles: every CTA loops over several tiles (TMEM ping-pong)
    err, bound, *_ = _run(0, 1024, 1024, 256, max_ctas=4, variant=variant)
    assert (err > bound).sum().item() == 0


@pytest.mark.parametrize("kind", [0, 1], ids=["bf16", "tf32"])
def test_pack_paths(kind):
    """row-contiguous, transposed and general-stride packs agree with torch."""
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    src = torch.randn(300, 264, device="cuda")
    elt = torch.bfloat16 if kind == 0 else torch.float32
    for rows, cols, s_row, s_col in [(300, 264, 264, 1), (264, 300, 1, 264),
                                     (150, 132, 528, 2)]:
        dst = torch.empty(rows, cols, dtype=elt, device="cuda")
        assert lib.b200_pack_operand(kind, P(src.data_ptr()), s_row, s_col,
                                     P(dst.data_ptr()), rows, cols, s) == 0
        torch.cuda.synchronize()
        view = torch.as_strided(src, (rows, cols), (s_row, s_col))
        want = _round(view.contiguous(), kind)
        assert torch.equal(dst.float(), want), (rows, cols, s_row, s_col)


@pytest.mark.parametrize("kind", [0, 1], ids=["bf16", "tf32"])
@pytest.mark.parametrize("shape,clusters", [((4096, 4096, 512), 74), ((2560, 2304, 640), 20),
                                            ((1280, 1280, 1024), 7)])
def test_gemm_tc2_split_tail(kind, shape, clusters):
    """partial last wave split along K; run twice to check ticket reset and
    that results are deterministic (bit-identical across launches)."""
    M, N, K = shape
    err, bound, *_ = _run(kind, M, N, K, variant=2, max_ctas=2 * clusters, seed=3)
    assert (err > bound).sum().item() == 0
    err2, _, *_ = _run(kind, M, N, K, variant=2, max_ctas=2 * clusters, seed=3)
    assert (err2 == err).all().item()


@pytest.mark.parametrize("rows", [256, 300])
def test_linear_stack_shadow_bit_identical(rows):
    """Chained Linear lowerings at bf16: the second contraction's A operand
    comes from the first one's epilogue (b200_gemm_tc_shadow) instead of a
    separate pack of H.  Both round the same f32 H to bf16 (RN), so every
    output must be bit-identical to the unshadowed run, H included; the
    second contraction must launch without an A pack."""
    import bench_kernels as bk
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    import harness

    fn = bk.make_linear_stack(rows)
    outs = {}
    for shadow in (False, True):
        args = harness.make_args(fn, seed=3)
        b2.configure(precision="bf16", shadow=shadow)
        try:
            machine.run(fn.module, "linear_stack", args, engine=b2.engine)
        finally:
            b2.configure(precision="exact", shadow=True)
        outs[shadow] = [a.data.tobytes() for a in args]
        plan = list(b2.engine.last_plan)
    assert outs[True] == outs[False]
    assert [p[0] for p in plan] == ["gemm_tc_bf16", "gemm_tc_bf16"]
    assert "C->shadow" in plan[0][-1] and "A<-shadow" in plan[1][-1]


@pytest.mark.parametrize("shape", [(128, 256, 64), (300, 512, 200), (1024, 1024, 1024),
                                   (4096, 4096, 512), (1000, 1024, 1000), (256, 192, 136)])
@pytest.mark.parametrize("mode", ["acc", "init_bias", "shadow"])
def test_gemm_tc_kn_equals_kmajor(shape, mode):
    """b200_gemm_tc_kn (B read MN-major from its K x N layout) computes the
    same products in the same order as the K-major CTA-pair kernel over the
    transposed pack: C (and the bf16 shadow) bitwise equal; tail items with
    narrow N included (split waves)."""
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(5)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    Bkn = (torch.rand(K, N, device="cuda", generator=g) * 2 - 1).bfloat16()
    Bt = Bkn.t().contiguous()
    C0 = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
    bias = torch.rand(N, device="cuda", generator=g)
    init, bptr = (1, bias) if mode == "init_bias" else (0, None)
    P = ctypes.c_void_p
    s = P(torch.cuda.current_stream().cuda_stream)
    outs = []
    for kn in (False, True):
        C = C0.clone()
        c16 = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda") if mode == "shadow" else None
        bp = P(bptr.data_ptr()) if bptr is not None else None
        if kn:
            rc = lib.b200_gemm_tc_kn(0, P(A.data_ptr()), P(Bkn.data_ptr()), P(C.data_ptr()), N,
                                     1, M, N, K, init, 0.25, bp, 1,
                                     P(c16.data_ptr()) if c16 is not None else None,
                                     N if c16 is not None else 0, s)
        elif c16 is not None:
            rc = lib.b200_gemm_tc_shadow(0, P(A.data_ptr()), P(Bt.data_ptr()), P(C.data_ptr()),
                                         N, 1, M, N, K, init, 0.25, bp, 1, P(c16.data_ptr()), N,
                                         s)
        else:
            rc = lib.b200_gemm_tc(0, P(A.data_ptr()), P(Bt.data_ptr()), P(C.data_ptr()), N, 1,
                                  M, N, K, init, 0.25, bp, 1, 0, 2, s)
        assert rc == 0
        torch.cuda.synchronize()
        outs.append((C, c16))
    assert torch.equal(outs[0][0], outs[1][0])
    if mode == "shadow":
        assert torch.equal(outs[0][1], outs[1][1])
        assert torch.equal(outs[1][1], outs[1][0].bfloat16())


def test_gemm_tc_kn_rejects_ragged_n():
    """The MN-major view needs N % 64 == 0; other widths are refused (the
    engine then packs B transposed for b200_gemm_tc)."""
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    P = ctypes.c_void_p
    A = torch.zeros(128, 64, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(64, 72, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(128, 72, device="cuda")
    s = P(torch.cuda.current_stream().cuda_stream)
    rc = lib.b200_gemm_tc_kn(0, P(A.data_ptr()), P(B.data_ptr()), P(C.data_ptr()), 72, 1, 128,
                             72, 64, 0, 0.0, None, 0, None, 0, s)
    assert rc != 0
