"""Dev probe: b200_gemm_f32_exact at 4096^3 (N=... to change); prints the
time and a hash of C so kernel variants can be checked bit-identical (the
round-2 tile / residency variants measured here are recorded in
csrc/gemm_exact.cu's launch())."""
import ctypes
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16080_b200 import runtime  # noqa: E402

N = int(os.environ.get("N", "4096"))
M = int(os.environ.get("M", str(N)))   # rows of A / C (wave-count experiments)
lib = runtime.load_library()
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
B = torch.rand(N, N, device="cuda", generator=g) * 2 - 1
C0 = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
C = C0.clone()
P = ctypes.c_void_p
s = P(torch.cuda.current_stream().cuda_stream)


def run():
    rc = lib.b200_gemm_f32_exact(P(A.data_ptr()), N, 1, P(B.data_ptr()), N, 1, P(C.data_ptr()),
                                 N, 1, M, N, N, 0, 0.0, None, 0, s)
    assert rc == 0


run()
torch.cuda.synchronize()
h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:16]
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
print(f"{ms:.3f} ms "
      f"{2 * M * N * N / ms / 1e9:.1f} TFLOP/s hash {h}")
