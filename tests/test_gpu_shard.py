"""Batch-sharded runs on the B200 (-m gpu): union of shards == unsharded run.

BASELINE configs[2] / [3] shard the batch of the conv and of the Linear
stack across GPUs.  One GPU is available here, so the ranks of
a world run one after another in this process, each through
paper_2307_16080_b200.shard.run on fresh copies of the same global batch;
every rank uploads, computes and writes back only its own rows.  The union
of the ranks' rows must be bit-identical to the unsharded run at the same
precision (every kernel computes each image / row independently of the
partition), and at exact precision also to the reference's f32 chain.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(fn, seed=0):
    import torch
    from staircase.interp import Buffer

    out = []
    for i, a in enumerate(fn.func_op.body().args):
        shape = tuple(a.type.shape)
        g = torch.Generator().manual_seed(seed + i)
        t = torch.rand(shape, generator=g, dtype=torch.float32) * 2 - 1
        out.append(Buffer(shape, "f32", t.numpy().tobytes()))
    return out


def _np(buf):
    return np.frombuffer(buf.data, dtype=np.float32).reshape(buf.shape[0], -1)


def _union(fn, world, precision, check_plan=None):
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import shard

    b2.configure(precision=precision, strict=True)
    try:
        union = None
        for rank in range(world):
            args = _inputs(fn)
            res = shard.run(fn.module, fn.__name__, args, rank=rank, world=world)
            if check_plan:
                check_plan(b2.engine.last_plan)
            st = b2.engine.last_staging
            r0, r1 = res.rows
            if union is None:
                union = [_np(a).copy() for a in args]
            for k, a in enumerate(args):
                if any(a is b for b in res.buffers):
                    union[k][r0:r1] = _np(a)[r0:r1]
            # only this rank's rows moved over PCIe (plus the replicated weights)
            total = sum(_np(a).nbytes for a in args)
            if r1 - r0 < res.batch:
                assert st.h2d_bytes < total
            else:
                assert st.h2d_bytes <= total
        full = _inputs(fn)
        from staircase.interp import machine

        machine.run(fn.module, fn.__name__, full, engine=b2.engine)
    finally:
        b2.configure(precision="exact", strict=False)
    return union, [_np(a) for a in full]


@pytest.mark.parametrize("precision", ["exact", "bf16"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_conv_resnet_shards(world, precision):
    import bench_kernels as bk

    fn = bk.make_conv(256)
    kernel = {"exact": "conv2d_exact", "bf16": "conv2d_tc_bf16"}[precision]

    def plan_ok(plan):
        assert plan[-1][0] == kernel, plan

    got, want = _union(fn, world, precision, plan_ok)
    assert got[2].tobytes() == want[2].tobytes()


@pytest.mark.parametrize("precision", ["exact", "bf16"])
@pytest.mark.parametrize("world", [2, 8])
def test_linear_stack_shards(world, precision):
    import bench_kernels as bk

    fn = bk.make_linear_stack(8192)
    kernel = {"exact": "gemm_f32_exact", "bf16": "gemm_tc_bf16"}[precision]

    def plan_ok(plan):
        assert [p[0] for p in plan] == [kernel, kernel], plan
        assert all({"fill", "bias"} <= set(p[4]) for p in plan), plan

    got, want = _union(fn, world, precision, plan_ok)
    assert got[3].tobytes() == want[3].tobytes()      # h
    assert got[6].tobytes() == want[6].tobytes()      # y


def test_conv_shard_exact_matches_reference_chain():
    """A shard's images at exact precision are the reference's f32 chain."""
    import bench_kernels as bk
    from paper_2307_16080_b200 import shard

    fn = bk.make_conv(16)
    args = _inputs(fn)
    X, W, O0 = (_np(a).reshape(a.shape).copy() for a in args)
    res = shard.run(fn.module, fn.__name__, args, rank=2, world=4)
    assert res.rows == (8, 12)
    O = _np(args[2]).reshape(args[2].shape)
    rng = np.random.default_rng(9)
    n = rng.integers(8, 12, 32)
    f, h, w = rng.integers(0, 64, 32), rng.integers(0, 56, 32), rng.integers(0, 56, 32)
    c = O0[n, f, h, w].astype(np.float32)
    for ci in range(64):
        for ki in range(3):
            for kj in range(3):
                c = (c + (X[n, ci, h + ki, w + kj] * W[f, ci, ki, kj]).astype(np.float32)
                     ).astype(np.float32)
    assert np.array_equal(O[n, f, h, w].view(np.int32), c.view(np.int32))
    # rows outside the shard were not touched
    assert np.array_equal(O[:8], O0[:8]) and np.array_equal(O[12:], O0[12:])


@pytest.mark.parametrize("nb,world", [(13, 4), (7, 3), (3, 5)])
@pytest.mark.parametrize("precision", ["exact", "bf16"])
def test_conv_uneven_and_empty_shards(nb, world, precision):
    """Batches the world does not divide, and more ranks than images (the
    reference's chunking [total w / W, total (w + 1) / W) leaves some ranks
    no rows): the union is still the unsharded run, bit for bit."""
    import bench_kernels as bk

    fn = bk.make_conv(nb)
    got, want = _union(fn, world, precision)
    assert got[2].tobytes() == want[2].tobytes()
