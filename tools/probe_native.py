"""Dev probe: native-specialised VM programs vs the device interpreter.

    python tools/probe_native.py

Runs nests that no template matches (data-dependent branches, running
recurrences) through the engine with native.ENABLED on and off and prints
device time per run (Session replay, CUDA events) and the speedup.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import bench_kernels as bk  # noqa: E402

SRC = {
    "relu_dot": '''
@staged
def relu_dot(x: MemRef[(8192, 1024), F32], w: MemRef[(1024,), F32], y: MemRef[(8192,), F32]):
    for i in parallel((0,), (8192,)):
        for j in range(1024):
            if x[i, j] > constant(0.0, F32):
                y[i] = y[i] + x[i, j] * w[j]
''',
    "row_scan": '''
@staged
def row_scan(x: MemRef[(16384, 512), F32]):
    for i in parallel((0,), (16384,)):
        for j in range(1, 512):
            x[i, j] = x[i, j] + x[i, j - 1]
''',
}


def main():
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import native

    for name, src in SRC.items():
        fn = bk._capture_from_source(src, name, {}, name)
        times = {}
        for on in (False, True):
            native.ENABLED = on
            import bench

            args = bench.host_inputs(fn, 0)
            sess = b2.Session()
            dev = [sess.tensor(a) for a in args]   # noqa: F841  (stage once)
            rec = sess.record(fn.module, name, args)
            torch.cuda.synchronize()
            for _ in range(3):
                rec.replay()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                rec.replay()
            e1.record()
            torch.cuda.synchronize()
            times[on] = e0.elapsed_time(e1) / 10
            print(f"{name:10s} native={on!s:5s} {times[on]:9.3f} ms  plan={sess.plan}", flush=True)
        print(f"{name:10s} speedup {times[False] / times[True]:.1f}x", flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
