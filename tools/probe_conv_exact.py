"""Dev probe: the bit-exact conv (b200_conv2d_exact) at the ResNet shape
(N=256, C=F=64, 56x56, 3x3), timed with CUDA events; prints a hash of the
output so staging variants (B200_CONV_EXACT_TMA=0/1) can be compared.

    python tools/probe_conv_exact.py [NB [INIT]]    (INIT 0: out += conv, as the bench)
"""
import ctypes
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2307_16080_b200 import runtime

    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    init = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    c = f = 64
    ho = wo = 56
    lib = runtime.load_library()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(nb, c, ho + 2, wo + 2, device="cuda", generator=g) * 2 - 1
    w = torch.rand(f, c, 3, 3, device="cuda", generator=g) * 2 - 1
    out = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
    work = torch.empty(c * 9 * f, device="cuda")
    I64 = ctypes.c_int64 * 4
    P = ctypes.c_void_p
    s = P(torch.cuda.current_stream().cuda_stream)
    xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*out.stride())

    def run():
        runtime.check(lib.b200_conv2d_exact(0, P(x.data_ptr()), xs, P(w.data_ptr()), ws,
                                            P(work.data_ptr()), P(out.data_ptr()), os_, nb, c,
                                            ho + 2, wo + 2, f, ho, wo, 3, 3, init,
                                            ctypes.c_double(0.0), s), "conv")

    run()
    torch.cuda.synchronize()
    h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 2.0 * nb * f * ho * wo * c * 9
    print(f"{ms:.3f} ms {flops / ms / 1e9:.1f} TFLOP/s hash {h}")


if __name__ == "__main__":
    main()
