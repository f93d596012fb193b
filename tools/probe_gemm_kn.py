"""Dev probe: b200_gemm_tc_kn (B K x N, MN-major) vs b200_gemm_tc (B^T packed
K-major) — equality of C and kernel time.

    python tools/probe_gemm_kn.py [--mnk M N K]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mnk", type=int, nargs=3, default=[4096, 4096, 4096])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--kind", type=int, default=0, help="0 bf16, 1 tf32")
    a = ap.parse_args()
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    M, N, K = a.mnk
    P = ctypes.c_void_p
    s = P(torch.cuda.current_stream().cuda_stream)
    kind = a.kind
    if kind == 0:
        A = torch.randn(M, K, device="cuda").bfloat16()
        Bkn = torch.randn(K, N, device="cuda").bfloat16()
    else:   # tf32-representable f32 (low 13 mantissa bits clear)
        def tf32(t):
            return (t.view(torch.int32) & ~0x1FFF).view(torch.float32)
        A = tf32(torch.randn(M, K, device="cuda"))
        Bkn = tf32(torch.randn(K, N, device="cuda"))
    Bt = Bkn.t().contiguous()
    C0 = torch.randn(M, N, device="cuda")
    res = {}
    for name in ("kmajor", "mnmajor"):
        C = C0.clone()

        def go():
            if name == "kmajor":
                rc = lib.b200_gemm_tc(kind, P(A.data_ptr()), P(Bt.data_ptr()), P(C.data_ptr()), N, 1,
                                      M, N, K, 0, 0.0, None, 0, 0, 2, s)
            else:
                rc = lib.b200_gemm_tc_kn(kind, P(A.data_ptr()), P(Bkn.data_ptr()), P(C.data_ptr()),
                                         N, 1, M, N, K, 0, 0.0, None, 0, None, 0, s)
            assert rc == 0, rc

        go()
        torch.cuda.synchronize()
        res[name] = C.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            go()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"{name}: M={M} N={N} K={K} ms={ms:.4f} TFLOP/s={2 * M * N * K / ms / 1e9:.1f}")
    want = C0.double() + A.double() @ Bkn.double()
    for name, C in res.items():
        err = (C.double() - want).abs().max().item()
        print(f"{name}: max |err| vs fp64 = {err:.3e}")
    print("bitwise equal:", torch.equal(res["kmajor"], res["mnmajor"]))


if __name__ == "__main__":
    main()
