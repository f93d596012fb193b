"""Dev stress: the B200 sweep's log against the reference tuner's own
search() (run on the C oracle engine) over corpus kernels, strategies,
seeds and budgets — the log (idx, params, cost, status, seed) and the best
trial must be identical.

    python tools/stress_sweep.py [cases] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()


def main():
    import corpus
    import oracle
    from test_sweep import _ref, _space

    from paper_2307_16080_b200 import sweep

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    oracle.build()
    kernels = [corpus.conv_small, corpus.conv_rows, corpus.matmul_par]
    bad = 0
    for c in range(cases):
        fn = rnd.choice(kernels)
        strategy = rnd.choice(["random", "es"])   # the reference strategies
        seed, budget = rnd.randint(0, 10 ** 6), rnd.randint(4, 24)
        best_r, log_r = _ref(fn.module, budget, seed, strategy)
        best, log = sweep.search(fn.module, None, _space(), budget=budget, seed=seed,
                                 strategy=strategy, rank=0, world=1)
        same = log == log_r and best == best_r
        bad += not same
        print(f"case {c}: {fn.__name__} {strategy} seed {seed} budget {budget}: "
              f"{'equal' if same else 'DIFFERENT'}", flush=True)
    print(f"{cases - bad}/{cases} logs equal to the reference")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
