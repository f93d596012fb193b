"""bench.py's multi-rank plumbing on CPU (gloo, world size 2).

The driver launches `bench.py --gpus N` under torch.distributed.run, one rank
per GPU over NCCL; the only collectives are the timing max-over-ranks and one
all-gather of per-rank checksums.  Here the same helpers run over
gloo with two CPU processes: batch shards of the conv / Linear-stack
workloads partition the batch exactly, max_over_ranks returns the slowest
rank's time on every rank, and gather_checksums returns every rank's value in
rank order.
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
        conv, ls = bench.Workload("conv", world), bench.Workload("ls", world)
        t = bench.max_over_ranks(1.0 + rank, world)
        sums = bench.gather_checksums(10.0 * rank + 0.5, world)
        bench.barrier(world)
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(repr((conv.shapes()[0][0], conv.flops, ls.shapes()[0][0], t, sums,
                           conv.scaling, bench.Workload("mm", world).scaling)))
    finally:
        dist.destroy_process_group()


def test_two_rank_helpers_over_gloo():
    import torch.multiprocessing as mp

    import bench

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [eval(open(os.path.join(d, f"r{r}.txt")).read()) for r in range(2)]
    full = bench.Workload("conv", 1)
    for nb, flops, rows, t, sums, conv_scaling, mm_scaling in res:
        assert nb == 128 and 2 * flops == full.flops      # the batch split exactly in two
        assert rows == 32768
        assert t == 2.0                                  # the slowest rank, on every rank
        assert sums == [0.5, 10.5]                       # rank order
        assert (conv_scaling, mm_scaling) == ("strong", "weak")
