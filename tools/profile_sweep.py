"""Dev probe: where a sweep trial's time goes (cProfile over sweep.search).

    python tools/profile_sweep.py [budget]
"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import bench_kernels as bk  # noqa: E402


def main():
    import torch

    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace

    budget = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    space = ParamSpace(tile_sizes=([1, 2, 4, 8, 16, 32, 64, 128],) * 2,
                       unroll_factors=[1, 2, 4, 8])
    for fn in (bk.mm_par1024, bk.conv_paper):
        sweep.search(fn.module, None, space, budget=4, seed=0, strategy="grid")   # warm
        torch.cuda.synchronize()
        prof = cProfile.Profile()
        timing = {}
        prof.enable()
        sweep.search(fn.module, None, space, budget=budget, seed=0, strategy="grid",
                     timing=timing)
        torch.cuda.synchronize()
        prof.disable()
        print(f"== {fn.__name__}: {budget} trials, trials {timing.get('trials_s'):.3f} s",
              flush=True)
        pstats.Stats(prof).sort_stats(os.environ.get("SORT", "cumulative")).print_stats(int(os.environ.get("TOP", "28")))


if __name__ == "__main__":
    main()
