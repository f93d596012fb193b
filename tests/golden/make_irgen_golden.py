"""Generate tests/golden/irgen.json: random modules run by the UNMODIFIED reference.

Run in the build container (where /root/reference exists) as

    python tests/golden/make_irgen_golden.py

The reference's own random module builder (pkg/tests/irgen.py:
``random_module(seed)`` — nested scf.for / affine.for / scf.if /
scf.parallel, f64 and i64 arithmetic, memref.alloc / alloca *inside* those
blocks, loads and stores with unchecked indices) is imported from
/root/reference; each module is printed with the reference printer (.sir
text), its memref parameters are filled from ``random.Random(seed)``
(U(-2, 2)), and it is run with the reference's compiled executor (_evalcy,
baseline/_ref, sequential mode).  Recorded per seed: the .sir text, the
inputs, the outputs (raw bytes, base64), the 25-slot tally, or the error
type and message.  The GPU box has no /root/reference: the tests parse the
.sir with the reference parser (baseline/_ref) and compare the B200 engine
against these fixtures.
"""
import base64
import json
import os
import random
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()
sys.path.insert(0, "/root/reference/pkg/tests")

import irgen  # noqa: E402  (the reference's generator)
from staircase.interp import Buffer, _evalcy, machine  # noqa: E402
from staircase.ir.core import create_context  # noqa: E402
from staircase.textio import parse_module, print_module  # noqa: E402

SEEDS = range(300)


def _portable(msg):
    return re.sub(r"at \S*/([^/\s]+):(\d+)", r"at \1:\2", msg)


def make_inputs(module, seed):
    func = [op for op in module.body().ops if op.name == "func.func"][0]
    rng = random.Random(seed)
    out = []
    for a in func.body().args:
        n = 1
        for s in a.type.shape:
            n *= s
        out.append(Buffer(tuple(a.type.shape), a.type.element.kind,
                          [rng.uniform(-2.0, 2.0) for _ in range(n)]))
    return func.attributes["sym_name"].value, out


def main():
    cases = []
    for seed in SEEDS:
        # the fixture is the printed module, re-parsed — exactly what the
        # tests run (op locations then read <input>:line in both)
        module = parse_module(print_module(irgen.random_module(seed)), create_context())
        name, args = make_inputs(module, seed)
        ins = [base64.b64encode(a.data.tobytes()).decode() for a in args]
        box = {}

        class Tap:
            ExecContext = _evalcy.ExecContext

            @staticmethod
            def run_tape(program, code, regs, tally, ctx):
                try:
                    return _evalcy.run_tape(program, code, regs, tally, ctx)
                finally:
                    box["t"] = list(tally)

        rec = {"seed": seed, "func": name, "sir": print_module(module),
               "args": [{"shape": list(a.shape), "dtype": a.dtype, "b64": b}
                        for a, b in zip(args, ins)]}
        try:
            machine.run(module, name, args, engine=Tap)
            rec["outputs"] = [base64.b64encode(a.data.tobytes()).decode() for a in args]
            rec["tally"] = box["t"]
        except Exception as exc:   # noqa: BLE001 — the reference's error is the fixture
            rec["error"] = [type(exc).__name__, _portable(str(exc))]
            rec["outputs"] = [base64.b64encode(a.data.tobytes()).decode() for a in args]
            rec["tally"] = box.get("t")
        cases.append(rec)
    with open(os.path.join(HERE, "irgen.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    n_err = sum("error" in c for c in cases)
    n_alloc = sum("memref.alloc" in c["sir"] for c in cases)
    print(f"{len(cases)} modules ({n_err} raising, {n_alloc} with allocs) -> irgen.json")


if __name__ == "__main__":
    main()
