"""Dev probe: the bf16 conv step (input pack + tensor-core conv) over the
whole batch against the same work in image chunks, so a chunk's NHWC bf16
repack is still in L2 when its conv reads it (one stream), or with the next
chunk's pack overlapping the current chunk's conv (two streams).  Outputs
must be bit-identical to the whole-batch run.

    python tools/probe_conv_chunks.py [NB] [CHUNK ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2307_16080_b200 import runtime

    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    chunks = [int(v) for v in sys.argv[2:]] or [64, 32, 16]
    c = f = 64
    ho = wo = 56
    kh = kw = 3
    hp, wp = ho + 2, wo + 2
    cp = 64
    lib = runtime.load_library()
    P = ctypes.c_void_p
    I64 = ctypes.c_int64 * 4
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(nb, c, hp, wp, device="cuda", generator=g) * 2 - 1
    w = torch.rand(f, c, kh, kw, device="cuda", generator=g) * 2 - 1
    o0 = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
    xp = torch.empty(nb, hp, wp, cp, device="cuda", dtype=torch.bfloat16)
    wt = torch.empty(f, kh * kw * cp, device="cuda", dtype=torch.bfloat16)
    xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*o0.stride())
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    runtime.check(lib.b200_pack_conv_weight(P(w.data_ptr()), ws, P(wt.data_ptr()), f, c, kh, kw,
                                            cp, P(main_s.cuda_stream)), "wpack")

    def pack(i0, n, st):
        runtime.check(lib.b200_pack_conv_input(P(x[i0].data_ptr()), xs, P(xp[i0].data_ptr()), n,
                                               c, hp, wp, cp, P(st.cuda_stream)), "pack")

    def conv(out, i0, n, st):
        runtime.check(lib.b200_conv2d_tc(P(xp[i0].data_ptr()), P(wt.data_ptr()),
                                         P(out[i0].data_ptr()), os_, n, cp, hp, wp, f, ho, wo,
                                         kh, kw, 0, ctypes.c_float(0.0), P(st.cuda_stream)),
                      "conv")

    def run(out, chunk, streams):
        if streams == 1:
            for i0 in range(0, nb, chunk):
                n = min(chunk, nb - i0)
                pack(i0, n, main_s)
                conv(out, i0, n, main_s)
            return
        evs = []
        side.wait_stream(main_s)
        for i0 in range(0, nb, chunk):
            n = min(chunk, nb - i0)
            pack(i0, n, side)
            ev = torch.cuda.Event()
            ev.record(side)
            evs.append((i0, n, ev))
        for i0, n, ev in evs:
            main_s.wait_event(ev)
            conv(out, i0, n, main_s)

    ref = o0.clone()
    run(ref, nb, 1)
    torch.cuda.synchronize()
    for chunk in [nb] + chunks:
        for streams in (1, 2):
            if chunk == nb and streams == 2:
                continue
            out = o0.clone()
            run(out, chunk, streams)
            torch.cuda.synchronize()
            same = torch.equal(out, ref)
            for _ in range(3):
                run(out, chunk, streams)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                run(out, chunk, streams)
            e1.record()
            torch.cuda.synchronize()
            print(f"nb {nb} chunk {chunk} streams {streams}: {e0.elapsed_time(e1) / 10 * 1e3:.1f}"
                  f" us  (first run bit-identical to whole batch: {same})", flush=True)


if __name__ == "__main__":
    main()
