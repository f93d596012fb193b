"""bench.py's multi-rank plumbing on CPU (gloo, world size 2).

The driver launches `bench.py --gpus N` under torch.distributed.run, one rank
per GPU over NCCL; besides shard.gather (tests/test_shard.py) the only
collectives are the timing max-over-ranks and one all-gather of per-rank
checksums.  Here the same helpers run over gloo with two CPU
processes: the conv / Linear-stack workloads are the global batch (sharded
by paper_2307_16080_b200.shard at run time, contiguous halves), max_over_ranks
returns the slowest rank's time on every rank, and gather_checksums returns
every rank's value in rank order.
"""
import os
import socket
import tempfile

import conftest  # noqa: F401  (spawned workers re-import this module: shim first)


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

    import bench

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from paper_2307_16080_b200 import shard

        conv, ls = bench.Workload("conv"), bench.Workload("ls")
        t = bench.max_over_ranks(1.0 + rank, world)
        sums = bench.gather_checksums(10.0 * rank + 0.5, world)
        bench.barrier(world)
        nb = conv.fn.func_op.body().args[0].type.shape[0]
        rows = ls.fn.func_op.body().args[0].type.shape[0]
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(repr((shard.chunk(nb, rank, world), conv.flops,
                           shard.chunk(rows, rank, world), t, sums,
                           conv.sharded, bench.Workload("mm").sharded)))
    finally:
        dist.destroy_process_group()


def test_two_rank_helpers_over_gloo():
    import torch.multiprocessing as mp

    import bench

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [eval(open(os.path.join(d, f"r{r}.txt")).read()) for r in range(2)]
    assert [r[0] for r in res] == [(0, 128), (128, 256)]          # contiguous image halves
    assert [r[2] for r in res] == [(0, 32768), (32768, 65536)]    # contiguous row halves
    for _, flops, _, t, sums, conv_sharded, mm_sharded in res:
        assert flops == 2.0 * 256 * 64 * 56 * 56 * 64 * 9        # the global batch's work
        assert t == 2.0                                  # the slowest rank, on every rank
        assert sums == [0.5, 10.5]                       # rank order
        assert (conv_sharded, mm_sharded) == (True, False)
