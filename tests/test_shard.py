"""Batch-sharded runs (paper_2307_16080_b200.shard) on CPU.

Each rank runs the same module on the same global batch, restricted to the
contiguous batch rows the worksharing rule assigns it (reference
interp/_evalpy.py:279); the union of the ranks' rows must be bit-identical
to the unsharded run (the reference executor / the oracle pinned to it),
including unequal chunks.  The device kernels are replaced by the CPU
simulator (tests/vm_sim.py); the world-2 test runs two gloo processes and
gathers the rows with shard.gather.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import conftest  # noqa: F401  (spawned workers re-import this module: shim first)
import corpus
import harness
from vm_sim import SimBackend


def _np(buf):
    return np.frombuffer(buf.data, dtype={"f32": np.float32, "f64": np.float64}[buf.dtype])


def _sharded_union(fn, world, seed=3):
    from paper_2307_16080_b200 import shard

    out = None
    rows_seen = []
    for rank in range(world):
        args = harness.make_args(fn, seed)
        res = shard.run(fn.module, fn.__name__, args, rank=rank, world=world,
                        backend=SimBackend())
        assert res.rows == shard.chunk(res.batch, rank, world)
        rows_seen.append(res.rows)
        if out is None:
            out = [np.array(_np(a)).reshape(a.shape[0], -1) if hasattr(a, "data") else a
                   for a in args]
        for k, a in enumerate(args):
            if hasattr(a, "data") and any(a is b for b in res.buffers):
                r0, r1 = res.rows
                out[k][r0:r1] = _np(a).reshape(a.shape[0], -1)[r0:r1]
    return out, rows_seen


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])   # 7 > 4 images: empty shards
@pytest.mark.parametrize("fn", [corpus.conv_mid, corpus.matmul_t, corpus.conv_f32],
                         ids=["conv_mid", "matmul_t", "conv_f32"])
def test_union_of_shards_is_the_unsharded_run(fn, world, oracle_engine):
    got, rows = _sharded_union(fn, world)
    # contiguous, disjoint, covering
    assert rows[0][0] == 0 and all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    want_args = harness.make_args(fn, 3)
    from staircase.interp import machine

    machine.run(fn.module, fn.__name__, want_args, engine=oracle_engine)
    for g, w in zip(got, want_args):
        if hasattr(w, "data"):
            assert g.tobytes() == _np(w).tobytes()


def test_linear_stack_shards_keep_fusion():
    """The Linear stack (fill / contraction / bias per layer) on a shard of
    its rows: still two fused contractions, and rows identical to the
    unsharded run."""
    import bench_kernels as bk
    from paper_2307_16080_b200 import engine, shard
    from vm_sim import SimEngine

    fn = bk.make_linear_stack(8)
    args = harness.make_args(fn, 1)
    res = shard.run(fn.module, fn.__name__, args, rank=1, world=2, backend=SimBackend())
    plan = engine.last_plan
    assert [p[0] for p in plan] == ["contract_exact", "contract_exact"], plan
    assert res.rows == (4, 8)
    assert [b.shape for b in res.buffers] == [(8, 4096), (8, 1024)]   # h, y
    full = harness.make_args(fn, 1)
    from staircase.interp import machine

    machine.run(fn.module, fn.__name__, full, engine=SimEngine())
    for k in (3, 6):
        got = _np(args[k]).reshape(8, -1)[4:8]
        want = _np(full[k]).reshape(8, -1)[4:8]
        assert got.tobytes() == want.tobytes()


def test_unshardable_regions_raise():
    from paper_2307_16080_b200 import shard
    from paper_2307_16080_b200.host import errors

    E = errors()
    # sequential (affine.for) nests and a loop-carried triangle: no batch loop
    for fn in (corpus.matmul_affine, corpus.triangle):
        args = harness.make_args(fn, 0)
        with pytest.raises(E.ModeUnsupported):
            shard.run(fn.module, fn.__name__, args, rank=0, world=2, backend=SimBackend())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import conftest  # noqa: F401
    import torch.distributed as dist

    import corpus
    import harness
    from paper_2307_16080_b200 import shard
    from vm_sim import SimBackend

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        fn = corpus.conv_mid
        args = harness.make_args(fn, 5)
        res = shard.run(fn.module, fn.__name__, args, backend=SimBackend())
        got = shard.gather(res)
        np.save(os.path.join(out_dir, f"r{rank}.npy"),
                np.frombuffer(args[2].data, dtype=np.float32))
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(repr((res.rank, res.world, res.rows, got)))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_gather_equals_unsharded(oracle_engine):
    import torch.multiprocessing as mp
    from staircase.interp import machine

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        outs = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(2)]
        meta = [eval(open(os.path.join(d, f"r{r}.txt")).read()) for r in range(2)]
    assert [m[:3] for m in meta] == [(0, 2, (0, 2)), (1, 2, (2, 4))]
    assert all(m[3] == 2 * 8 * 32 * 32 * 4 for m in meta)   # the other rank's 2 images
    fn = corpus.conv_mid
    want = harness.make_args(fn, 5)
    machine.run(fn.module, fn.__name__, want, engine=oracle_engine)
    for o in outs:   # after the gather every rank holds the whole batch
        assert o.tobytes() == np.frombuffer(want[2].data, dtype=np.float32).tobytes()
