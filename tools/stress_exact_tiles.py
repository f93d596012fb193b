"""Dev stress: random whole-tile shapes, paddings, init / bias for every CTA
tile of the exact GEMM (b200_gemm_f32_exact_tiled) against the general
tiled kernel (B200_GEMM_EXACT_OLD=1): bit for bit.

    python tools/stress_exact_tiles.py [cases] [seed]
"""
import ctypes
import os
import random
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16080_b200 import runtime  # noqa: E402


def run(lib, A, B, C, init, bias, cta, old):
    out = C.clone()
    P = ctypes.c_void_p
    if old:
        os.environ["B200_GEMM_EXACT_OLD"] = "1"
    else:
        os.environ.pop("B200_GEMM_EXACT_OLD", None)
    rc = lib.b200_gemm_f32_exact_tiled(
        P(A.data_ptr()), A.stride(0), 1, P(B.data_ptr()), B.stride(0), 1, P(out.data_ptr()),
        out.stride(0), 1, A.shape[0], B.shape[1], A.shape[1], init, ctypes.c_float(-0.25),
        P(bias.data_ptr()) if bias is not None else None, 1, cta[0], cta[1],
        P(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0, rc
    return out


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    lib = runtime.load_library()
    bad = 0
    for c in range(cases):
        cta = rnd.choice([(128, 128), (64, 256), (256, 64), (64, 64)])
        M = cta[0] * rnd.randint(1, 12)
        N = cta[1] * rnd.randint(1, 12)
        K = 32 * rnd.randint(1, 40)
        pad = 4 * rnd.randint(0, 3)
        init, use_bias = rnd.randint(0, 1), rnd.randint(0, 1)
        g = torch.Generator(device="cuda").manual_seed(c)
        A = (torch.rand(M, K + pad, device="cuda", generator=g) * 2 - 1)[:, :K]
        B = (torch.rand(K, N + pad, device="cuda", generator=g) * 2 - 1)[:, :N]
        C = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
        bias = torch.rand(N, device="cuda", generator=g) if use_bias else None
        new = run(lib, A, B, C, init, bias, cta, False)
        ref = run(lib, A, B, C, init, bias, cta, True)
        same = bool((new == ref).all())
        bad += not same
        print(f"case {c}: cta {cta} M {M} N {N} K {K} pad {pad} init {init} bias {use_bias}: "
              f"{'ok' if same else 'MISMATCH'}", flush=True)
    print(f"{cases - bad}/{cases} bit-identical")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
