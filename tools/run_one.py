"""Dev driver for profiling: one workload's recorded launch sequence, replayed.

    python tools/run_one.py --workload mm --precision exact [--tiles 8x8] [--reps 3]

Records the engine's plan for the bench workload (bench.Workload) with a
Session and replays it ``reps`` times (no CPU baseline, no e2e): the short
command the ncu recipe wants (B200_PROFILING.md).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mm")
    ap.add_argument("--precision", default="exact")
    ap.add_argument("--tiles", default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import runtime

    torch.cuda.set_device(0)
    lib = runtime.load_library()
    tiles = tuple(int(x) for x in args.tiles.split("x")) if args.tiles else None
    wl = bench.Workload(args.workload, tiles)
    b2.configure(precision=args.precision)
    sess = b2.Session()
    dev = bench.host_inputs(wl.fn)
    rec = sess.record(wl.module, wl.func, dev)
    for _ in range(args.reps):
        rec.replay(lib)
    torch.cuda.synchronize()
    print("plan", sess.plan, "launches per step", rec.launches)


if __name__ == "__main__":
    main()
