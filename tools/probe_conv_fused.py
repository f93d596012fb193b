"""Dev probe: the fused conv (b200_conv2d_tc_fused: NCHW f32 read and
converted in the kernel) against the repack path (b200_pack_conv_input +
b200_conv2d_tc) — the bf16 patches are the same values, so the outputs must
be bit-identical — and both timed.

    python tools/probe_conv_fused.py NB [C F HO WO]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2307_16080_b200 import runtime

    nb = int(sys.argv[1])
    c, f, ho, wo = (int(v) for v in sys.argv[2:6]) if len(sys.argv) > 5 else (64, 64, 56, 56)
    kh = kw = 3
    lib = runtime.load_library()
    hp, wp = ho + kh - 1, wo + kw - 1
    cp = -(-c // 64) * 64
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64 * 4
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(nb, c, hp, wp, device="cuda", generator=g) * 2 - 1
    w = torch.rand(f, c, kh, kw, device="cuda", generator=g) * 2 - 1
    o0 = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
    xp = torch.empty(nb, hp, wp, cp, device="cuda", dtype=torch.bfloat16)
    wt = torch.empty(f, kh * kw * cp, device="cuda", dtype=torch.bfloat16)
    xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*o0.stride())
    runtime.check(lib.b200_pack_conv_weight(P(w.data_ptr()), ws, P(wt.data_ptr()), f, c, kh, kw,
                                            cp, s), "wpack")
    a, b = o0.clone(), o0.clone()

    def unfused(out):
        runtime.check(lib.b200_pack_conv_input(P(x.data_ptr()), xs, P(xp.data_ptr()), nb, c, hp,
                                               wp, cp, s), "pack")
        runtime.check(lib.b200_conv2d_tc(P(xp.data_ptr()), P(wt.data_ptr()), P(out.data_ptr()),
                                         os_, nb, cp, hp, wp, f, ho, wo, kh, kw, 0,
                                         ctypes.c_float(0.0), s), "conv")

    def fused(out):
        runtime.check(lib.b200_conv2d_tc_fused(P(x.data_ptr()), xs, P(wt.data_ptr()),
                                               P(out.data_ptr()), os_, nb, c, hp, wp, f, ho, wo,
                                               kh, kw, 0, ctypes.c_float(0.0), s), "fused")

    only = os.environ.get("ONLY")
    if only != "fused":
        unfused(a)
        torch.cuda.synchronize()
        print("unfused ran", flush=True)
    if only != "unfused":
        fused(b)
        torch.cuda.synchronize()
        print("fused ran", flush=True)
    if only:
        return
    same = torch.equal(a, b)
    diff = (a - b).abs().max().item()
    times = {}
    for name, fn, out in (("unfused", unfused, a), ("fused", fused, b)):
        for _ in range(3):
            fn(out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn(out)
        e1.record()
        torch.cuda.synchronize()
        times[name] = e0.elapsed_time(e1) / 10
    print(f"nb {nb}: bit-identical {same} (max diff {diff:.3g}); unfused {times['unfused']*1e3:.1f}"
          f" us, fused {times['fused']*1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
