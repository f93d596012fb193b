"""The fused tensor-core conv (b200_conv2d_tc_fused: the NCHW f32 input read
by TMA in whole row pairs and converted to the bf16 patch inside the conv
kernel) against the repack path (b200_pack_conv_input + b200_conv2d_tc).

Both feed the tensor cores the same bf16-rounded patch values in the same
MMA order, so the outputs must be bit-identical — at every batch size,
including the full ResNet batch and several row bands per CTA (the raw-chunk
rings and band order are exercised there), not only at the sizes the engine
routes to the fused kernel (runtime.FUSED_CONV_MAX_IMAGES).
"""
import ctypes

import numpy as np
import pytest

import corpus
import harness

pytestmark = pytest.mark.gpu


def _run_both(nb, c, f, ho, wo, init=0, seed=0):
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    kh = kw = 3
    hp, wp = ho + 2, wo + 2
    cp = -(-c // 64) * 64
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64 * 4
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand(nb, c, hp, wp, device="cuda", generator=g) * 2 - 1
    w = torch.rand(f, c, kh, kw, device="cuda", generator=g) * 2 - 1
    o0 = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
    xp = torch.empty(nb, hp, wp, cp, device="cuda", dtype=torch.bfloat16)
    wt = torch.empty(f, kh * kw * cp, device="cuda", dtype=torch.bfloat16)
    xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*o0.stride())
    runtime.check(lib.b200_pack_conv_weight(P(w.data_ptr()), ws, P(wt.data_ptr()), f, c, kh, kw,
                                            cp, s), "pack weights")
    a, b = o0.clone(), o0.clone()
    runtime.check(lib.b200_pack_conv_input(P(x.data_ptr()), xs, P(xp.data_ptr()), nb, c, hp, wp,
                                           cp, s), "pack input")
    runtime.check(lib.b200_conv2d_tc(P(xp.data_ptr()), P(wt.data_ptr()), P(a.data_ptr()), os_, nb,
                                     cp, hp, wp, f, ho, wo, kh, kw, init, ctypes.c_float(0.5), s),
                  "conv")
    rc = lib.b200_conv2d_tc_fused(P(x.data_ptr()), xs, P(wt.data_ptr()), P(b.data_ptr()), os_, nb,
                                  c, hp, wp, f, ho, wo, kh, kw, init, ctypes.c_float(0.5), s)
    torch.cuda.synchronize()
    return rc, a, b


@pytest.mark.parametrize("nb,c,f,ho,wo", [
    (1, 64, 64, 56, 56), (8, 64, 64, 56, 56), (64, 64, 64, 56, 56), (256, 64, 64, 56, 56),
    (4, 32, 32, 20, 30), (5, 64, 32, 56, 56), (3, 48, 64, 16, 24), (2, 64, 64, 12, 20),
])
@pytest.mark.parametrize("init", [0, 1])
@pytest.mark.parametrize("pair", ["0", "1"])
def test_fused_equals_repack_path(nb, c, f, ho, wo, init, pair, monkeypatch):
    """pair "1": the opt-in CTA-pair variant (B200_CONV_PAIR=1: the band's two
    column tiles as one cta_group::2 MMA, weights split across the pair)."""
    monkeypatch.setenv("B200_CONV_PAIR", pair)
    rc, a, b = _run_both(nb, c, f, ho, wo, init)
    assert rc == 0
    assert bool((a == b).all()), f"max diff {(a - b).abs().max().item()}"


def test_fused_refuses_what_it_cannot_tile():
    """C > 64 (two channel blocks), odd H or W, or three column tiles per
    band: B200_EUNSUPPORTED (-3), and the engine packs instead."""
    for shape in [(2, 100, 64, 16, 24), (2, 64, 64, 15, 24), (2, 64, 64, 16, 64)]:
        rc, _, _ = _run_both(*shape)
        assert rc == -3, shape


def test_engine_routes_small_batches_to_the_fused_kernel(monkeypatch):
    """run() at bf16: a small-batch conv plan uses the weight pack + fused
    kernel; B200_CONV_UNFUSED=1 gives the pack + conv path; the outputs of
    the two runs are bit-identical and the tally is the reference's."""
    import paper_2307_16080_b200 as b2

    fn = corpus.conv_tc_smoke
    outs, plans = [], []
    for unfused in ("0", "1"):
        monkeypatch.setenv("B200_CONV_UNFUSED", unfused)
        with b2.engine.using(precision="bf16", strict=True):
            _, bufs, tally, _ = harness.run_engine(b2.engine, fn, None, "sequential", 8)
        outs.append(np.frombuffer(bufs[-1].data, dtype=np.float32).copy())
        plans.append(list(b2.engine.last_plan))
    assert plans[0][-1][0] == plans[1][-1][0] == "conv2d_tc_bf16"
    assert "input converted in-kernel" in plans[0][-1][-1], plans[0]
    assert "input converted in-kernel" not in str(plans[1][-1]), plans[1]
    assert outs[0].tobytes() == outs[1].tobytes()
