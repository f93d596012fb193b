"""Dev probe: where the host time of one end-to-end run goes.

    python tools/profile_e2e.py [workload] [precision]

Runs the bench workload through staircase's run() with host Buffers (as the
bench's e2e leg does), warms twice, then cProfiles 3 runs and prints the top
cumulative entries plus the wall time per run.
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    import torch

    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    name = sys.argv[1] if len(sys.argv) > 1 else "mm"
    wl = bench.Workload(name)
    b2.configure(precision=sys.argv[2] if len(sys.argv) > 2 else wl.default_precision)
    host = bench.host_inputs(wl.fn)
    fn = wl.fn
    for _ in range(2):
        machine.run(fn.module, fn.__name__, host, engine=b2.engine)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        machine.run(fn.module, fn.__name__, host, engine=b2.engine)
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.3f} ms per run (unprofiled)")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        machine.run(fn.module, fn.__name__, host, engine=b2.engine)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)


if __name__ == "__main__":
    main()
