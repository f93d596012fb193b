"""Dev probe: the exact GEMM through b200_gemm_f32_exact_tiled with each CTA
tile the tile sizes can select (runtime.cta_tile) at 4096^3: time and a
hash of C (every tile shape must give the same bits).

    B200_LIB=... python tools/probe_exact_tiles.py
"""
import ctypes
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16080_b200 import runtime  # noqa: E402

N = int(os.environ.get("N", "4096"))
lib = runtime.load_library()
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(N, N, device="cuda", generator=g) * 2 - 1
B = torch.rand(N, N, device="cuda", generator=g) * 2 - 1
C0 = torch.rand(N, N, device="cuda", generator=g) * 2 - 1
P = ctypes.c_void_p
s = P(torch.cuda.current_stream().cuda_stream)
for cm, cn in ((128, 128), (64, 256), (256, 64), (64, 64)):
    C = C0.clone()

    def run():
        rc = lib.b200_gemm_f32_exact_tiled(P(A.data_ptr()), N, 1, P(B.data_ptr()), N, 1,
                                           P(C.data_ptr()), N, 1, N, N, N, 0, 0.0, None, 0,
                                           cm, cn, s)
        assert rc == 0

    run()
    torch.cuda.synchronize()
    h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:16]
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cta {cm}x{cn}: {ms:.3f} ms {2 * N ** 3 / ms / 1e9:.1f} TFLOP/s hash {h}", flush=True)
