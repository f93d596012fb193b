"""Dev stress: random matmul / Linear shapes through run() with the host
copies streamed (row panels, (row, column) blocks with K slices) against the
same run unstreamed, at exact and bf16: buffers and tally bit-identical.
Streaming is forced at any size (runtime.STREAM_MIN_BYTES = 1).

    python tools/stress_stream.py [cases] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

MM = '''
@staged
def mm_s(A: MemRef[({M}, {K}), F32], B: MemRef[({K}, {N}), F32], C: MemRef[({M}, {N}), F32]):
    for i, j in parallel((0, 0), ({M}, {N})):
        for k in range(0, {K}):
            C[i, j] = C[i, j] + A[i, k] * B[k, j]
'''


def main():
    import bench_kernels as bk
    import harness

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import engine, runtime

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    runtime.STREAM_MIN_BYTES = 1
    runtime.STREAM_PANEL_BYTES = 1 << 14
    bad = 0
    for c in range(cases):
        M = rnd.choice([128, 256, 384, 512, 1024, 96, 200, 640])
        N = rnd.choice([256, 512, 768, 1024, 64, 130, 512])
        K = rnd.choice([32, 64, 96, 160, 512, 1000, 48])
        prec = rnd.choice(["exact", "exact", "bf16"])
        tiles = rnd.choice([None, (8, 8), (4, 16), (16, 4), (2, 2)])
        fn = bk._capture_from_source(MM.format(M=M, N=N, K=K), "mm_s", {}, f"{M}_{N}_{K}")
        pipe = (harness._spec(f"scf-parallel-loop-tiling{{sizes=[{tiles[0]}, {tiles[1]}]}}")
                if tiles else None)
        out = []
        for stream in (False, True):
            with engine.using(precision=prec, stream_io=stream):
                _, bufs, tally, _ = harness.run_engine(b2.engine, fn, pipe, "sequential", c)
            out.append(([b.data.tobytes() for b in bufs], tally, list(engine.last_plan),
                        engine.last_staging.panels))
        (w, tw, pw, p0), (g, tg, pg, p1) = out
        same = w == g and tw == tg and pw == pg
        bad += not same
        print(f"case {c}: {M}x{N}x{K} {prec} tiles {tiles}: panels {p1} "
              f"{'equal' if same else 'DIFFERENT'} {pg}", flush=True)
    print(f"{cases - bad}/{cases} streamed runs equal to unstreamed")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
