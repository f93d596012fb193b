"""The whole-tile exact GEMM kernels (gemm_exact.cu): the TMA-fed default,
the cp.async variant it replaced (B200_GEMM_EXACT_TMA=0) and the general
tiled kernel (B200_GEMM_EXACT_OLD=1) all run the reference's chain — one
__fmul_rn and one __fadd_rn per MAC, k ascending, init and bias in the
reference order — so they must agree bit for bit on every qualifying shape,
padded strides, init and bias included, and match the chain recomputed with
numpy float32 ops on sampled outputs.
"""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(A, B, C, init, bias, env):
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    out = C.clone()
    M, K = A.shape[0], A.shape[1]
    N = B.shape[1]
    P = ctypes.c_void_p
    saved = {k: os.environ.get(k) for k in ("B200_GEMM_EXACT_TMA", "B200_GEMM_EXACT_OLD")}
    os.environ.pop("B200_GEMM_EXACT_TMA", None)
    os.environ.pop("B200_GEMM_EXACT_OLD", None)
    os.environ.update(env)
    try:
        rc = lib.b200_gemm_f32_exact(P(A.data_ptr()), A.stride(0), 1, P(B.data_ptr()),
                                     B.stride(0), 1, P(out.data_ptr()), out.stride(0), 1, M, N,
                                     K, init, ctypes.c_float(0.75),
                                     P(bias.data_ptr()) if bias is not None else None, 1,
                                     P(torch.cuda.current_stream().cuda_stream))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    torch.cuda.synchronize()
    assert rc == 0
    return out


@pytest.mark.parametrize("M,N,K,pad", [(128, 128, 32, 0), (256, 384, 96, 4), (512, 128, 1024, 0),
                                       (384, 256, 160, 8), (1024, 1024, 512, 0)])
@pytest.mark.parametrize("init,use_bias", [(0, False), (1, True), (0, True)])
def test_whole_tile_kernels_agree(M, N, K, pad, init, use_bias):
    import torch

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (torch.rand(M, K + pad, device="cuda", generator=g) * 2 - 1)[:, :K]
    B = (torch.rand(K, N + pad, device="cuda", generator=g) * 2 - 1)[:, :N]
    C = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
    bias = torch.rand(N, device="cuda", generator=g) if use_bias else None
    tma = _gemm(A, B, C, init, bias, {})
    cpa = _gemm(A, B, C, init, bias, {"B200_GEMM_EXACT_TMA": "0"})
    old = _gemm(A, B, C, init, bias, {"B200_GEMM_EXACT_OLD": "1"})
    assert bool((tma == cpa).all()) and bool((tma == old).all())
    a, b, c, t = (x.cpu().numpy() for x in (A, B, C, tma))
    bn = bias.cpu().numpy() if use_bias else None
    rng = np.random.default_rng(K)
    for _ in range(8):
        i, j = int(rng.integers(0, M)), int(rng.integers(0, N))
        acc = np.float32(0.75) if init else np.float32(c[i, j])
        for k in range(K):
            acc = np.float32(acc + np.float32(np.float32(a[i, k]) * np.float32(b[k, j])))
        if use_bias:
            acc = np.float32(acc + np.float32(bn[j]))
        assert t[i, j] == acc


def _gemm_tiled(A, B, C, init, bias, cta, env):
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    out = C.clone()
    P = ctypes.c_void_p
    saved = os.environ.get("B200_GEMM_EXACT_OLD")
    os.environ.pop("B200_GEMM_EXACT_OLD", None)
    os.environ.update(env)
    try:
        rc = lib.b200_gemm_f32_exact_tiled(
            P(A.data_ptr()), A.stride(0), 1, P(B.data_ptr()), B.stride(0), 1, P(out.data_ptr()),
            out.stride(0), 1, A.shape[0], B.shape[1], A.shape[1], init, ctypes.c_float(0.75),
            P(bias.data_ptr()) if bias is not None else None, 1, cta[0], cta[1],
            P(torch.cuda.current_stream().cuda_stream))
    finally:
        if saved is None:
            os.environ.pop("B200_GEMM_EXACT_OLD", None)
        else:
            os.environ["B200_GEMM_EXACT_OLD"] = saved
    torch.cuda.synchronize()
    assert rc == 0
    return out


@pytest.mark.parametrize("cta", [(64, 256), (256, 64), (64, 64)])
@pytest.mark.parametrize("M,N,K,pad", [(256, 256, 32, 0), (512, 768, 96, 4), (768, 512, 320, 8),
                                       (1024, 1024, 512, 0)])
@pytest.mark.parametrize("init,use_bias", [(0, False), (1, True)])
def test_tile_shaped_whole_tile_kernels_agree(cta, M, N, K, pad, init, use_bias):
    """The TMA kernel's 4 x 16 / 16 x 4 / 4 x 4 micro-tile shapes (the CTA
    tiles runtime.cta_tile picks for (4, 16)-, (16, 4)- and small-tiled
    nests) against the general tiled kernel of the same CTA tile and the
    default 128 x 128 TMA kernel: bit for bit."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = (torch.rand(M, K + pad, device="cuda", generator=g) * 2 - 1)[:, :K]
    B = (torch.rand(K, N + pad, device="cuda", generator=g) * 2 - 1)[:, :N]
    C = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
    bias = torch.rand(N, device="cuda", generator=g) if use_bias else None
    tma = _gemm_tiled(A, B, C, init, bias, cta, {})
    old = _gemm_tiled(A, B, C, init, bias, cta, {"B200_GEMM_EXACT_OLD": "1"})
    square = _gemm(A, B, C, init, bias, {})
    assert bool((tma == old).all()) and bool((tma == square).all())
