"""Dev probe: host -> device -> host schedules for the exact 4096^3 matmul
(C += A.B with pinned host A, B, C), timed end to end with CUDA events: the
engine's (row, column) blocks (`runtime._gemm_streamed_2d`) against the
same blocks split along K, so a block's first K slice computes while the
rest of its A rows / B columns upload.  C is read once per block (first
slice) and written back after its last slice; every output keeps its full
ascending k chain, so C must come out bit-identical to one whole launch.

    python tools/probe_stream_e2e.py [MP NP KS STREAMS ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2307_16080_b200 import runtime

    lib = runtime.load_library()
    n = 4096
    g = torch.Generator().manual_seed(0)
    hA = (torch.rand(n, n, generator=g) * 2 - 1).pin_memory()
    hB = (torch.rand(n, n, generator=g) * 2 - 1).pin_memory()
    hC0 = (torch.rand(n, n, generator=g) * 2 - 1)
    hC = hC0.clone().pin_memory()
    tA, tB, tC = (torch.empty(n, n, device="cuda") for _ in range(3))
    P = ctypes.c_void_p
    esz = 4
    cur = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    comps = [torch.cuda.Stream() for _ in range(8)]

    def copy2d(dst, src, r0, r1, c0, c1, kind, st):
        runtime.check(lib.b200_copy2d(P(dst.data_ptr() + esz * (r0 * n + c0)), n * esz,
                                      P(src.data_ptr() + esz * (r0 * n + c0)), n * esz,
                                      (c1 - c0) * esz, r1 - r0, kind, P(st.cuda_stream)),
                      "copy2d")

    def run(mp, np_, ks, nstreams):
        rs, cs, kl = n // mp, n // np_, n // ks
        up.wait_stream(cur)
        down.wait_stream(cur)
        comp = comps[:nstreams]
        for c in comp:
            c.wait_stream(cur)
        q = 0
        a_done = set()
        b_done = set()
        if os.environ.get("ORDER") == "row":
            # each row panel's blocks across every column panel in turn
            order = [(i, j) for i in range(mp) for j in range(np_)]
        elif os.environ.get("ORDER") == "zig":
            # pairs of row panels sweep every column panel before the next pair
            order = [(i, j) for i0 in range(0, mp, 2) for j in range(np_)
                     for i in range(i0, min(mp, i0 + 2))]
        else:
            order = [(i, j) for j in range(np_) for i in range(mp)]
        for i, j in order:
            c0, c1 = j * cs, (j + 1) * cs
            if True:
                r0, r1 = i * rs, (i + 1) * rs
                copy2d(tC, hC, r0, r1, c0, c1, 1, up)
                st = comp[q % nstreams]
                q += 1
                for s in range(ks):
                    k0, k1 = s * kl, (s + 1) * kl
                    if (i, s) not in a_done:
                        copy2d(tA, hA, r0, r1, k0, k1, 1, up)
                        a_done.add((i, s))
                    if (j, s) not in b_done:
                        copy2d(tB, hB, k0, k1, c0, c1, 1, up)
                        b_done.add((j, s))
                    ev = torch.cuda.Event()
                    ev.record(up)
                    st.wait_event(ev)
                    if os.environ.get("NOGEMM"):
                        continue
                    rc = lib.b200_gemm_f32_exact_tiled(
                        P(tA[r0, k0:].data_ptr()), n, 1, P(tB[k0, c0:].data_ptr()), n, 1,
                        P(tC[r0, c0:].data_ptr()), n, 1, r1 - r0, c1 - c0, k1 - k0, 0,
                        ctypes.c_float(0.0), None, 0, 128, 128, P(st.cuda_stream))
                    assert rc == 0
                done = torch.cuda.Event()
                done.record(st)
                down.wait_event(done)
                copy2d(hC, tC, r0, r1, c0, c1, 2, down)
        for c in comp:
            cur.wait_stream(c)
        cur.wait_stream(down)

    # reference result: one whole launch
    tA.copy_(hA)
    tB.copy_(hB)
    tC.copy_(hC0)
    assert lib.b200_gemm_f32_exact(P(tA.data_ptr()), n, 1, P(tB.data_ptr()), n, 1,
                                   P(tC.data_ptr()), n, 1, n, n, n, 0, ctypes.c_float(0.0),
                                   None, 0, P(cur.cuda_stream)) == 0
    want = tC.cpu()
    shapes = [tuple(int(v) for v in sys.argv[i:i + 4]) for i in range(1, len(sys.argv), 4)]
    shapes = shapes or [(4, 2, 1, 3), (4, 2, 2, 3), (4, 2, 4, 3), (2, 2, 4, 2), (2, 2, 4, 4),
                        (4, 2, 4, 4), (4, 4, 4, 4), (2, 2, 8, 4)]
    for mp, np_, ks, nst in shapes:
        hC.copy_(hC0)
        run(mp, np_, ks, nst)
        torch.cuda.synchronize()
        same = torch.equal(hC, want)
        times = []
        for _ in range(5):
            hC.copy_(hC0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(mp, np_, ks, nst)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        if os.environ.get("NOGEMM"):
            same = "n/a (copies only)"
        print(f"blocks {mp}x{np_} k-slices {ks} streams {nst}: median {times[2]:.3f} ms "
              f"(min {times[0]:.3f}); {2 * n ** 3 / times[2] / 1e9:.1f} TFLOP/s; "
              f"bit-identical {same}", flush=True)


if __name__ == "__main__":
    main()
