"""Pin the C oracle (oracle/tape_eval.c) to the reference's golden fixtures.

tests/golden/golden.json was produced by the unmodified reference executor
(_evalcy) via tests/golden/make_golden.py.  The oracle must reproduce every
fixture bit-for-bit: output buffer bytes, the full 25-slot tally, and the
error type/message for the error fixtures.  When the reference itself is
importable (this container and, via baseline/_ref, the GPU box) the oracle
is also compared live against it.
"""
import hashlib
import json
import os
import re

import pytest

import corpus
import harness

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "golden.json")))["cases"]
KERNELS = {fn.__name__: fn for fn in corpus.ALL}


def _portable(msg):
    return re.sub(r"at \S*/([^/\s]+):(\d+)", r"at \1:\2", msg)


def check_against_golden(engine, case):
    fn = KERNELS[case["kernel"]]
    if "error" in case:
        with pytest.raises(Exception) as info:
            harness.run_engine(engine, fn, case["pipeline"], case["mode"], case["seed"])
        assert type(info.value).__name__ == case["error"]
        assert _portable(str(info.value)) == case["message"]
        return
    results, args, tally, stats = harness.run_engine(
        engine, fn, case["pipeline"], case["mode"], case["seed"])
    assert tally == case["tally"]
    for a, rec in zip(args, case["args"]):
        if "sha256" in rec:
            assert hashlib.sha256(a.data.tobytes()).hexdigest() == rec["sha256"], \
                f"{case['kernel']}/{case['variant']} buffer mismatch"
    assert stats.total == case["stats"]["total"]


@pytest.mark.parametrize("case", GOLDEN,
                         ids=[f"{c['kernel']}-{c['variant']}-s{c['seed']}" for c in GOLDEN])
def test_oracle_matches_golden(oracle_engine, case):
    check_against_golden(oracle_engine, case)


@pytest.mark.parametrize("fn", [corpus.matmul_par, corpus.conv_f32, corpus.int_ops,
                                corpus.cond_body])
def test_oracle_matches_live_reference(oracle_engine, ref_engine, fn):
    for seed in (5, 6):
        mode = "sequential"
        r1, a1, t1, _ = harness.run_engine(ref_engine, fn, None, mode, seed)
        r2, a2, t2, _ = harness.run_engine(oracle_engine, fn, None, mode, seed)
        assert t1 == t2
        for x, y in zip(a1, a2):
            assert x.data.tobytes() == y.data.tobytes()
