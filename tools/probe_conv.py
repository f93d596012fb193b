"""Dev probe: time the conv tensor-core path stage by stage with CUDA events.

    python tools/probe_conv.py [--shape NB C F HO WO KH KW] [--init 0 1]

Prints pack-input, pack-weight and conv kernel times with the bandwidth /
TFLOP/s each reaches.  Not a bench number (bench.py is); used to A/B kernel
schedules quickly.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, iters):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=7, default=[256, 64, 64, 56, 56, 3, 3])
    ap.add_argument("--init", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    nb, c, f, ho, wo, kh, kw = a.shape
    hp, wp = ho + kh - 1, wo + kw - 1
    cp = -(-c // 64) * 64
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64 * 4
    x = torch.randn(nb, c, hp, wp, device="cuda")
    w = torch.randn(f, c, kh, kw, device="cuda")
    out = torch.zeros(nb, f, ho, wo, device="cuda")
    xp = torch.empty(nb, hp, wp, cp, device="cuda", dtype=torch.bfloat16)
    wt = torch.empty(f, kh * kw * cp, device="cuda", dtype=torch.bfloat16)
    xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*out.stride())

    def pack_in():
        runtime.check(lib.b200_pack_conv_input(P(x.data_ptr()), xs, P(xp.data_ptr()), nb, c, hp,
                                               wp, cp, s), "pack_in")

    def pack_w():
        runtime.check(lib.b200_pack_conv_weight(P(w.data_ptr()), ws, P(wt.data_ptr()), f, c, kh,
                                                kw, cp, s), "pack_w")

    ms = timed(pack_in, a.iters)
    byt = x.numel() * 4 + xp.numel() * 2
    print(f"pack_input  {ms * 1e3:8.1f} us  {byt / ms / 1e6:7.0f} GB/s", flush=True)
    ms = timed(pack_w, a.iters)
    print(f"pack_weight {ms * 1e3:8.1f} us", flush=True)
    flops = 2 * nb * ho * wo * f * c * kh * kw
    for init in a.init:
        def conv():
            runtime.check(lib.b200_conv2d_tc(P(xp.data_ptr()), P(wt.data_ptr()),
                                             P(out.data_ptr()), os_, nb, cp, hp, wp, f, ho, wo,
                                             kh, kw, init, 0.0, s), "conv")
        ms = timed(conv, a.iters)
        byt = xp.numel() * 2 + out.numel() * 4 * (1 if init else 2)
        print(f"conv init={init} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s  "
              f"{byt / ms / 1e6:7.0f} GB/s (algorithmic)", flush=True)
    # correctness spot check against torch (bf16-rounded operands, fp32 accumulate)
    out.zero_()
    runtime.check(lib.b200_conv2d_tc(P(xp.data_ptr()), P(wt.data_ptr()), P(out.data_ptr()),
                                     os_, nb, cp, hp, wp, f, ho, wo, kh, kw, 0, 0.0, s), "conv")
    ref = torch.nn.functional.conv2d(x[:2].bfloat16().float(), w.bfloat16().float())
    err = (out[:2] - ref).abs().max().item()
    print(f"max |err| vs torch on 2 images: {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
