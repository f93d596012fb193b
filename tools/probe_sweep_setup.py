"""Dev probe: where a sweep rank's setup goes (make_inputs, the baseline
run, the resident uploads) for the bench's two targets."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import bench_kernels as bk  # noqa: E402


def main():
    import importlib

    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import sweep
    from staircase.interp import machine

    ref = importlib.import_module("staircase.tuner.search")
    torch.zeros(1, device="cuda")
    Session, _ = sweep._session_class()
    for rep in range(3):
        for fn in (bk.mm_par1024, bk.conv_paper):
            t0 = time.perf_counter()
            inputs = sweep.make_inputs(fn.module, None, 0)
            t1 = time.perf_counter()
            args = ref._copy_args(inputs)
            t2 = time.perf_counter()
            machine.run(fn.module, fn.__name__, args, mode="sequential", engine=b2.engine)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            s = Session(fn.module, b2.engine)
            torch.cuda.synchronize()
            t4 = time.perf_counter()
            print(f"{fn.__name__}: make_inputs {1e3 * (t1 - t0):.1f} ms, copy_args "
                  f"{1e3 * (t2 - t1):.1f}, baseline run {1e3 * (t3 - t2):.1f}, "
                  f"whole Session init {1e3 * (t4 - t3):.1f}", flush=True)
            del s


if __name__ == "__main__":
    main()
