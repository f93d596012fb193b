"""The TMA-fed exact conv (conv_runs_tma_kernel: row-pair TMA boxes, mbarrier
ring, no CTA-wide barrier) against the cp.async-staged runs kernel it
replaces (B200_CONV_EXACT_TMA=0): the same per-output ci -> ki -> kj chain
of individually rounded products and sums, so the outputs must be
bit-identical — and both bit-identical to the reference's f32 chain
(interp/_evalpy.py:115-127), checked on sampled outputs.
"""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _conv(x, w, o, init, env):
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    nb, c, hp, wp = x.shape
    f, _, kh, kw = w.shape
    ho, wo = hp - kh + 1, wp - kw + 1
    out = o.clone()
    work = torch.empty(c * kh * kw * f, device="cuda")
    I64 = ctypes.c_int64 * 4
    P = ctypes.c_void_p
    old = os.environ.get("B200_CONV_EXACT_TMA")
    os.environ["B200_CONV_EXACT_TMA"] = env
    try:
        rc = lib.b200_conv2d_exact(0, P(x.data_ptr()), I64(*x.stride()), P(w.data_ptr()),
                                   I64(*w.stride()), P(work.data_ptr()), P(out.data_ptr()),
                                   I64(*out.stride()), nb, c, hp, wp, f, ho, wo, kh, kw, init,
                                   ctypes.c_double(0.25),
                                   P(torch.cuda.current_stream().cuda_stream))
    finally:
        if old is None:
            del os.environ["B200_CONV_EXACT_TMA"]
        else:
            os.environ["B200_CONV_EXACT_TMA"] = old
    torch.cuda.synchronize()
    assert rc == 0
    return out


def _chain(x, w, o, init, n, f, h, wcol):
    """The reference chain for one output, numpy float32 ops."""
    acc = np.float32(0.25) if init else np.float32(o[n, f, h, wcol])
    c = x.shape[1]
    for ci in range(c):
        for ki in range(3):
            for kj in range(3):
                p = np.float32(x[n, ci, h + ki, wcol + kj]) * np.float32(w[f, ci, ki, kj])
                acc = np.float32(acc + np.float32(p))
    return acc


@pytest.mark.parametrize("nb,c,f,ho,wo", [
    (2, 64, 64, 56, 56), (3, 13, 64, 20, 40), (1, 8, 128, 33, 34), (2, 30, 68, 10, 50),
    (4, 64, 64, 14, 56), (1, 3, 4, 6, 36),
])
@pytest.mark.parametrize("init", [0, 1])
def test_tma_runs_kernel_equals_cp_async_kernel(nb, c, f, ho, wo, init):
    import torch

    g = torch.Generator(device="cuda").manual_seed(nb * 1000 + c)
    x = torch.rand(nb, c, ho + 2, wo + 2, device="cuda", generator=g) * 2 - 1
    w = torch.rand(f, c, 3, 3, device="cuda", generator=g) * 2 - 1
    o = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
    a = _conv(x, w, o, init, "0")
    b = _conv(x, w, o, init, "1")
    assert bool((a == b).all()), f"max diff {(a - b).abs().max().item()}"
    xn, wn, on, bn = (t.cpu().numpy() for t in (x, w, o, b))
    rng = np.random.default_rng(c)
    for _ in range(6):
        n_, f_, h_, w_ = (int(rng.integers(0, e)) for e in (nb, f, ho, wo))
        assert bn[n_, f_, h_, w_] == _chain(xn, wn, on, init, n_, f_, h_, w_)
