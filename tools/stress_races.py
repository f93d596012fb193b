"""Dev stress: random parallel nests (shared, shifted, strided, transposed and
private writes; reads of written cells) through races.check_races against the
reference's own check_races (baseline/_ref, its CPU simulation): the conflict
lists must be identical, triples and order.

    python tools/stress_races.py [cases] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

PATTERNS = [
    "a[i] = a[i] + b[i, j]",                  # shared across j
    "a[j] = b[i, j]",                          # write-write across i
    "c[i, j] = b[i, j] * constant(2.0, F32)",  # private
    "c[i, j] = c[j, i] + b[i, j]",             # transposed read of written cells
    "a[i + j] = b[i, j]",                      # diagonal collisions
    "c[i, 0] = c[i, 0] + b[i, j]",             # column accumulate
]


def main():
    import bench_kernels as bk
    import harness
    from staircase.interp.races import check_races as ref_check

    from paper_2307_16080_b200 import races

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    bad = 0
    for c in range(cases):
        n, m = rnd.randint(1, 6), rnd.randint(1, 6)
        body = rnd.choice(PATTERNS)
        src = f'''
@staged
def race_r(a: MemRef[({n + m},), F32], b: MemRef[({max(n, m)}, {max(n, m)}), F32],
           c: MemRef[({max(n, m)}, {max(n, m)}), F32]):
    for i, j in parallel((0, 0), ({n}, {m})):
        {body}
'''
        fn = bk._capture_from_source(src, "race_r", {}, f"{n}_{m}_{PATTERNS.index(body)}")
        args = harness.make_args(fn, c)
        want = ref_check(fn.module, fn.__name__, args)
        args = harness.make_args(fn, c)
        got = races.check_races(fn.module, fn.__name__, args)
        same = got == want
        bad += not same
        print(f"case {c}: {n}x{m} {body!r}: {len(want)} conflicts "
              f"{'equal' if same else 'DIFFERENT'}", flush=True)
    print(f"{cases - bad}/{cases} conflict lists equal to the reference")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
