"""Dev stress: random batch sizes and worlds for batch-sharded runs
(shard.run, every rank in turn on this GPU) of the conv and the Linear
stack at exact and bf16: the union of the ranks' rows must equal the
unsharded run bit for bit.

    python tools/stress_shard.py [cases] [seed]
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
    import bench_kernels as bk
    import test_gpu_shard as ts

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    bad = 0
    for c in range(cases):
        kind = rnd.choice(["conv", "ls"])
        prec = rnd.choice(["exact", "bf16"])
        world = rnd.randint(2, 9)   # _union checks a rank moves only its rows
        if kind == "conv":
            nb = rnd.randint(1, 20)
            fn, outs = bk.make_conv(nb), [2]
        else:
            nb = 64 * rnd.randint(1, 8)
            fn, outs = bk.make_linear_stack(nb), [3, 6]
        got, want = ts._union(fn, world, prec)
        same = all(got[k].tobytes() == want[k].tobytes() for k in outs)
        bad += not same
        print(f"case {c}: {kind} batch {nb} world {world} {prec}: "
              f"{'equal' if same else 'DIFFERENT'}", flush=True)
    print(f"{cases - bad}/{cases} unions equal to the unsharded run")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
