"""Generate tests/golden/golden.json by running the UNMODIFIED reference executor.

Run in the build container (where /root/reference exists) as

    python tests/golden/make_golden.py

It imports staircase from baseline/_ref (installed from /root/reference by
baseline/install_ref.sh, with the compiled _evalcy engine) and records, for
every corpus kernel and pass-pipeline variant: the seeded inputs' recipe,
the output buffers (raw bytes, base64) and the full 25-slot tally.  The
fixtures travel with the repo; the GPU-side tests read them instead of the
reference.  Inputs are regenerated from ``(seed, recipe)`` by
``tests/harness.py:make_args`` — the same generator this script uses.
"""
import base64
import hashlib
import re
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import corpus  # noqa: E402
import harness  # noqa: E402
from staircase.interp import Buffer, _evalcy, machine  # noqa: E402


def _buf_record(a):
    raw = a.data.tobytes()
    rec = {"dtype": a.dtype, "shape": list(a.shape),
           "sha256": hashlib.sha256(raw).hexdigest()}
    if len(a.data) <= 1024:
        rec["b64"] = base64.b64encode(raw).decode()
    return rec


def _portable(msg):
    # absolute source paths differ between machines; keep the basename
    return re.sub(r"at \S*/([^/\s]+):(\d+)", r"at \1:\2", msg)


def record(fn, variant, pipeline, mode, seed):
    module = harness.transformed(fn, pipeline)
    args = harness.make_args(fn, seed)
    tally_box = {}

    class Tap:
        ExecContext = _evalcy.ExecContext

        @staticmethod
        def run_tape(program, code, regs, tally, ctx):
            out = _evalcy.run_tape(program, code, regs, tally, ctx)
            tally_box["t"] = list(tally)
            return out

    entry = {"kernel": fn.__name__, "variant": variant, "pipeline": pipeline,
             "mode": mode, "seed": seed}
    try:
        results, stats = machine.run(module, fn.__name__, args, mode=mode,
                                     engine=Tap)
    except Exception as exc:  # error parity fixtures
        entry["error"] = type(exc).__name__
        entry["message"] = _portable(str(exc))
        return entry
    entry["tally"] = tally_box["t"]
    entry["stats"] = {"total": stats.total, "arith": stats.arith_ops,
                      "loads": stats.loads, "stores": stats.stores,
                      "bookkeeping": stats.bookkeeping}
    entry["args"] = [_buf_record(a) if isinstance(a, Buffer) else {"scalar": a}
                     for a in args]
    entry["results"] = [r if not isinstance(r, Buffer) else "buffer"
                        for r in results]
    return entry


def main():
    out = []
    for fn, variant, pipeline, mode in harness.CASES:
        for seed in (0, 1):
            out.append(record(fn, variant, pipeline, mode, seed))
    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "staircase 0.1.0 (_evalcy engine, unmodified)",
                   "cases": out}, fh, indent=0)
    print(f"wrote {len(out)} cases to {path}")


if __name__ == "__main__":
    main()
