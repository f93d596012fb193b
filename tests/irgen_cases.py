"""Fixtures of tests/golden/irgen.json: the reference's random modules
(pkg/tests/irgen.py) with the reference executor's outcome (test helper)."""
import base64
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "irgen.json")))


def module_and_args(case):
    from staircase.interp import Buffer
    from staircase.textio import parse_module

    from staircase.ir.core import create_context

    module = parse_module(case["sir"], create_context())
    args = []
    for a in case["args"]:
        dt = {"f64": np.float64, "f32": np.float32, "i32": np.int32, "i64": np.int64}[a["dtype"]]
        data = np.frombuffer(base64.b64decode(a["b64"]), dtype=dt).tolist()
        args.append(Buffer(tuple(a["shape"]), a["dtype"], data))
    return module, args


def check(engine, case, exact_fault_tally=False):
    """Run ``case`` through the reference run() on ``engine``; compare the
    outputs (bytes), the 25-slot tally and the error type + message."""
    import re

    from staircase.interp import machine

    module, args = module_and_args(case)
    box = {}

    class Tap:
        ExecContext = engine.ExecContext

        @staticmethod
        def run_tape(program, code, regs, tally, ctx):
            try:
                return engine.run_tape(program, code, regs, tally, ctx)
            finally:
                box["t"] = list(tally)

    err = None
    try:
        machine.run(module, case["func"], args, engine=Tap)
    except Exception as exc:   # noqa: BLE001
        err = [type(exc).__name__, re.sub(r"at \S*/([^/\s]+):(\d+)", r"at \1:\2", str(exc))]
    assert err == case.get("error"), (err, case.get("error"))
    for a, want in zip(args, case["outputs"]):
        assert a.data.tobytes() == base64.b64decode(want), f"seed {case['seed']}: buffer differs"
    # the tally is observable only through the ExecStats of a run that
    # returns (run() raises before folding it): compared for those, and for
    # raising runs only when the engine is the oracle (a restatement of the
    # reference loop, it counts up to the fault too)
    if case.get("tally") is not None and (err is None or exact_fault_tally):
        assert box["t"] == case["tally"], f"seed {case['seed']}: tally differs"
