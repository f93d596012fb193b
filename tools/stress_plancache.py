"""Dev stress: the region plan cache under a random interleaving of runs —
every harness case (corpus kernel x pipeline x mode) run repeatedly with
fresh seeded inputs in random order, so cached plans are replayed against
new buffers, scalars and neighbours; each run's buffers, tally and error
must equal the C oracle's.

    python tools/stress_plancache.py [runs] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()


def outcome(engine, case, seed):
    import harness

    fn, _, pipe, mode = case
    try:
        _, args, tally, _ = harness.run_engine(engine, fn, pipe, mode, seed)
        return ([a.data.tobytes() if hasattr(a, "data") else a for a in args], tally, None)
    except Exception as exc:   # faults must match too
        return (None, None, (type(exc).__name__, str(exc)))


def main():
    import harness
    import oracle

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import plancache

    runs = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    oracle.build()
    bad = 0
    for r in range(runs):
        case = rnd.choice(harness.CASES)
        seed = rnd.randint(0, 7)
        got = outcome(b2.engine, case, seed)
        want = outcome(oracle, case, seed)
        if got != want:
            bad += 1
            print(f"run {r}: {case[0].__name__} {case[1]} {case[3]} seed {seed}: DIFFERENT",
                  flush=True)
    stats = getattr(plancache, "STATS", None)
    print(f"{runs - bad}/{runs} runs equal to the oracle; cache stats {stats}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
