"""The reference's own known answers, CPU side.

The corpus kernels the GPU known-answer tests run (tests/test_gpu_known_answers.py)
ARE the reference's golden IR: printed with the reference's printer they equal
pkg/tests/golden/matmul.sir and conv2d.sir byte for byte (checked here, where
/root/reference exists; the GPU box has no /root/reference).  The oracle
reproduces the answers, and the reference's conv_oracle
(pkg/tests/kernels.py:116-134) restated below agrees with the oracle.
"""
import os

import numpy as np
import pytest

import corpus
from staircase.interp import Buffer, machine

REF_GOLDEN = "/root/reference/pkg/tests/golden"


@pytest.mark.skipif(not os.path.isdir(REF_GOLDEN), reason="reference tree not present")
@pytest.mark.parametrize("fn,name,golden", [(corpus.matmul_affine, "matmul_affine", "matmul"),
                                            (corpus.conv2d_desk, "conv2d_desk", "conv2d")])
def test_corpus_kernel_is_the_reference_golden_ir(fn, name, golden):
    from staircase.textio import print_module

    text = print_module(fn.module).replace(f"@{name}", f"@{golden}")
    with open(os.path.join(REF_GOLDEN, golden + ".sir")) as fh:
        assert text.strip() == fh.read().strip()


def conv_oracle(src, flt, dst_shape):
    """Restatement of the reference's conv_oracle (pkg/tests/kernels.py:116-134):
    direct convolution in plain Python floats, acc from 0.0, ci -> ki -> kj."""
    n_, ci_, hi, wi = src.shape
    co_, _, k, _ = flt.shape
    _, _, ho_, wo_ = dst_shape
    out = np.zeros(dst_shape)
    for n in range(n_):
        for co in range(co_):
            for ho in range(ho_):
                for wo in range(wo_):
                    acc = 0.0
                    for ci in range(ci_):
                        for ki in range(k):
                            for kj in range(k):
                                acc += float(src[n, ci, ho + ki, wo + kj]) * float(
                                    flt[co, ci, ki, kj])
                    out[n, co, ho, wo] = acc
    return out


def ones_args(fn, zero_last=True):
    out = []
    args = fn.func_op.body().args
    for i, a in enumerate(args):
        n = int(np.prod(a.type.shape))
        v = 0.0 if (zero_last and i == len(args) - 1) else 1.0
        out.append(Buffer(tuple(a.type.shape), a.type.element.kind, [v] * n))
    return out


def test_oracle_known_answers(oracle_engine):
    args = ones_args(corpus.matmul_affine)
    machine.run(corpus.matmul_affine.module, "matmul_affine", args, engine=oracle_engine)
    assert set(args[2].data) == {16.0}
    args = ones_args(corpus.conv_ones8)
    machine.run(corpus.conv_ones8.module, "conv_ones8", args, engine=oracle_engine)
    assert set(args[2].data) == {9.0}


def test_conv_oracle_restatement_matches_the_oracle(oracle_engine):
    import harness

    args = harness.make_args(corpus.conv2d_desk, 4)
    src = np.array(args[0].data).reshape(args[0].shape)
    flt = np.array(args[1].data).reshape(args[1].shape)
    zero = Buffer(args[2].shape, "f64", [0.0] * int(np.prod(args[2].shape)))
    machine.run(corpus.conv2d_desk.module, "conv2d_desk", [args[0], args[1], zero],
                engine=oracle_engine)
    want = conv_oracle(src, flt, args[2].shape)
    assert np.array(zero.data).reshape(args[2].shape).tobytes() == want.tobytes()
