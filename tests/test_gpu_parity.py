"""Parity of the CUDA path on a real B200 (run with -m gpu via gpurun).

1. Every golden fixture from the unmodified reference (tests/golden) is
   reproduced bit-for-bit through staircase's own run() with the B200
   engine: buffer bytes, the full 25-slot tally, error type and message.
2. Larger seeded cases (shapes that are not tile multiples, transposed
   operands, tiled/unrolled/outlined variants) are compared bit-for-bit with
   the C oracle (oracle/tape_eval.c), itself pinned to the reference.
Tolerance: none — the fp32/f64 paths are bit-exact by construction
(per-op IEEE rounding, reference reduction order).
"""
import pytest

import corpus
import harness
import oracle
from test_oracle import GOLDEN, check_against_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b200():
    import paper_2307_16080_b200 as b2

    return b2.engine


@pytest.mark.parametrize("case", GOLDEN,
                         ids=[f"{c['kernel']}-{c['variant']}-s{c['seed']}" for c in GOLDEN])
def test_golden_on_b200(b200, case):
    check_against_golden(b200, case)


BIG_CASES = [
    (corpus.matmul_odd, None, "sequential"),
    (corpus.matmul_odd, harness.UNROLL2, "sequential"),
    (corpus.matmul_t, None, "sequential"),
    (corpus.matmul_t, harness.TILE416, "worksharing"),
    (corpus.matmul_t, harness.TILE_OUTLINE, "gpu_emulated"),
    (corpus.conv_mid, None, "sequential"),
    (corpus.conv_mid, harness.TILE88, "sequential"),
    (corpus.conv_mid, harness.OUTLINE, "gpu_emulated"),
]


@pytest.mark.parametrize("fn,pipe,mode", BIG_CASES,
                         ids=[f"{f.__name__}-{i}" for i, (f, p, m) in enumerate(BIG_CASES)])
def test_big_vs_oracle(b200, fn, pipe, mode):
    oracle.build()
    for seed in (11, 12):
        _, got, t_got, _ = harness.run_engine(b200, fn, pipe, mode, seed)
        _, want, t_want, _ = harness.run_engine(oracle, fn, pipe, mode, seed)
        assert t_got == t_want
        for g, w in zip(got, want):
            assert g.data.tobytes() == w.data.tobytes()
