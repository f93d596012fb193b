"""The reference's known answers on the B200 (-m gpu).

* the matmul golden IR (pkg/tests/golden/matmul.sir ==
  corpus.matmul_affine, tests/test_known_answers.py) on A = ones(4,16),
  B = ones(16,8), C = zeros(4,8) gives C all 16.0 — at every precision;
* conv on ones (1x1x8x8, 3x3) gives 9.0; through the
  tcgen05 conv (C = F = 64) the same answer is 9 * 64 = 576.0;
* pkg/tests/kernels.py:116 — the reference's conv_oracle equals the B200's
  f64 conv of the golden conv2d IR bit for bit (both accumulate in double
  from 0.0 in ci -> ki -> kj order);
* a map body that stores y and loads y again is bit-exact with
  the oracle (no __restrict__ on aliasing operands).
"""
import numpy as np
import pytest

import corpus
import harness
from test_known_answers import conv_oracle, ones_args

pytestmark = pytest.mark.gpu


def _run(fn, args, precision="exact", pipe=None):
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    b2.configure(precision=precision, strict=precision != "exact")
    try:
        machine.run(harness.transformed(fn, pipe), fn.__name__, args, engine=b2.engine)
    finally:
        b2.configure(precision="exact", strict=False)
    return list(b2.engine.last_plan)


@pytest.mark.parametrize("precision", ["exact", "bf16", "tf32"])
def test_matmul_golden_ones_is_16(precision):
    args = ones_args(corpus.matmul_affine)
    plan = _run(corpus.matmul_affine, args, precision)
    assert set(args[2].data) == {16.0}, plan
    assert plan[-1][0] == {"exact": "gemm_f32_exact", "bf16": "gemm_tc_bf16",
                           "tf32": "gemm_tc_tf32"}[precision]


def test_conv_ones_is_9():
    args = ones_args(corpus.conv_ones8)
    plan = _run(corpus.conv_ones8, args)
    assert set(args[2].data) == {9.0}, plan


@pytest.mark.parametrize("precision", ["exact", "bf16"])
def test_conv_ones_tensor_cores(precision):
    args = ones_args(corpus.conv_ones64)
    plan = _run(corpus.conv_ones64, args, precision)
    assert plan[-1][0] == {"exact": "conv2d_exact", "bf16": "conv2d_tc_bf16"}[precision]
    assert set(args[2].data) == {576.0}


def test_conv_oracle_equals_b200_f64_conv():
    from staircase.interp import Buffer

    args = harness.make_args(corpus.conv2d_desk, 4)
    src = np.array(args[0].data).reshape(args[0].shape)
    flt = np.array(args[1].data).reshape(args[1].shape)
    zero = Buffer(args[2].shape, "f64", [0.0] * int(np.prod(args[2].shape)))
    plan = _run(corpus.conv2d_desk, [args[0], args[1], zero])
    assert plan[-1][0] == "conv2d_exact", plan
    want = conv_oracle(src, flt, args[2].shape)
    assert np.array(zero.data).reshape(args[2].shape).tobytes() == want.tobytes()


def test_store_then_load_map_matches_oracle(oracle_engine):
    fn = corpus.store_then_load
    _, got, t_got, _ = harness.run_engine(__import__("paper_2307_16080_b200").engine, fn, None,
                                          "sequential", 2)
    _, want, t_want, _ = harness.run_engine(oracle_engine, fn, None, "sequential", 2)
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()
