"""Dev probe: time b200_gemm_tc variants at 4096^3 with CUDA events.

    python tools/probe_gemm.py [--kind 0|1] [--variant 0|1|2] [--init 0|1] [--mnk M N K]

Prints one line per configuration: kernel ms and TFLOP/s.  Not a bench
number (bench.py is); used to A/B kernel schedules quickly.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", type=int, nargs="+", default=[0])
    ap.add_argument("--variant", type=int, nargs="+", default=[2])
    ap.add_argument("--init", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--mnk", type=int, nargs=3, default=[4096, 4096, 4096])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cublas", action="store_true", help="also time torch.mm (cuBLAS) bf16")
    ap.add_argument("--bias", action="store_true", help="fused bias epilogue")
    ap.add_argument("--shadow", action="store_true", help="also write the bf16 shadow of C")
    a = ap.parse_args()
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    M, N, K = a.mnk
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = ctypes.c_void_p
    C = torch.zeros(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    if a.cublas:
        for dt in (torch.bfloat16,):
            X = torch.randn(M, K, device="cuda").to(dt)
            Y = torch.randn(K, N, device="cuda").to(dt)
            Z = torch.empty(M, N, device="cuda", dtype=dt)
            for _ in range(3):
                torch.mm(X, Y, out=Z)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                torch.mm(X, Y, out=Z)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            print(f"cublas {dt} M={M} N={N} K={K} ms={ms:.4f} TFLOP/s={2*M*N*K/ms/1e9:.1f}",
                  flush=True)
    for kind in a.kind:
        elt = torch.bfloat16 if kind == 0 else torch.float32
        A = torch.randn(M, K, device="cuda").to(elt)
        Bt = torch.randn(N, K, device="cuda").to(elt)
        for variant in a.variant:
            for init in a.init:
                S16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if a.shadow else None

                def go():
                    if a.shadow:
                        rc = lib.b200_gemm_tc_shadow(
                            kind, P(A.data_ptr()), P(Bt.data_ptr()), P(C.data_ptr()), N, 1, M, N,
                            K, init, 0.0, P(bias.data_ptr()) if a.bias else None,
                            1 if a.bias else 0, P(S16.data_ptr()), N, s)
                        assert rc == 0
                        return
                    rc = lib.b200_gemm_tc(kind, P(A.data_ptr()), P(Bt.data_ptr()),
                                          P(C.data_ptr()), N, 1, M, N, K, init, 0.0,
                                          P(bias.data_ptr()) if a.bias else None,
                                          1 if a.bias else 0, 0, variant, s)
                    assert rc == 0
                for _ in range(3):
                    go()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    go()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                print(f"kind={kind} variant={variant} init={init} bias={int(a.bias)} "
                      f"shadow={int(a.shadow)} M={M} N={N} K={K} "
                      f"ms={ms:.4f} TFLOP/s={2*M*N*K/ms/1e9:.1f}", flush=True)


if __name__ == "__main__":
    main()
