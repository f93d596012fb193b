"""Batch-sharded execution of one staircase run over the GPUs of a node.

The reference parallelises a run with *worksharing* (reference
interp/_evalpy.py:276-300): each top-level (depth-0) ``scf.parallel`` loop's
iteration space is cut into contiguous chunks ``[total*w/W,
total*(w+1)/W)`` (:279), one per worker, over shared memory.  Here the
workers are processes, one per GPU (torch.distributed, NCCL), and the
memory is not shared: every rank holds the run's arguments as host Buffers
(the same global batch), executes the chunk of every depth-0 parallel nest
that the same rule assigns it — applied to the batch (outermost) dimension,
which equals the reference's flattened chunks whenever W divides the batch,
as at every BASELINE config — and copies only its own rows of the batch
buffers in and out.  There is no collective on the data path;
``gather()`` is an optional NCCL all-gather of the outputs' rows, timed on
its own.

A run shards when every region of the entry function is a depth-0 parallel
nest whose first loop (the batch loop, 0 .. B step 1) indexes the leading
dimension of each buffer it touches *in that loop's iteration* — the
*batch buffers* — and writes no other buffer (weights and biases are read
only, i.e. replicated).  Then row b of every batch buffer depends only on
rows b of the others, so each rank's rows are exactly those of the
unsharded run (tests/test_shard.py: the union of the shards is bit-identical
to the unsharded run).  Anything else raises ``ModeUnsupported``.

    from paper_2307_16080_b200 import shard
    res = shard.run(module, "conv", args)          # rank / world from torch.distributed
    res.rows                                       # this rank's batch rows [r0, r1)
    shard.gather(res)                              # all ranks' rows into every rank's Buffers
"""
from __future__ import annotations

from .host import errors as _errors
from .lift import Aff, Par


def chunk(total, rank, world):
    """[lo, hi): worker ``rank``'s contiguous share of ``total`` iterations
    (reference interp/_evalpy.py:279)."""
    return total * rank // world, total * (rank + 1) // world


class Shard:
    """One rank's view of a sharded run: which rows of which buffers."""

    def __init__(self, rank, world):
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world {world}")
        self.rank, self.world = rank, world
        self.batch = None        # B: the batch extent (first region fixes it)
        self.rows = None         # (r0, r1) = chunk(B, rank, world)
        self.buffers = {}        # id(Buffer) -> Buffer: the batch buffers
        self.written = set()     # ids of the batch buffers some region writes
        self.regions = 0

    def restrict(self, region, accesses, stage):
        """Validate ``region`` for sharding and restrict its batch loop to
        this rank's rows (mutates the loop's bounds before any planning)."""
        E = _errors()
        top = region.tree[0] if len(region.tree) == 1 else None
        if not isinstance(top, Par) or not top.vars:
            raise E.ModeUnsupported("sharded run: every region must be one depth-0 "
                                    "scf.parallel nest (the batch loop)")
        v = top.vars[0]
        st = v.static()
        if st is None or st[0] != 0 or st[1] != 1:
            raise E.ModeUnsupported("sharded run: the batch loop must run 0 .. B step 1")
        B = st[2]
        if self.batch is None:
            self.batch = B
            self.rows = chunk(B, self.rank, self.world)
        elif B != self.batch:
            raise E.ModeUnsupported(f"sharded run: batch extent {B} != {self.batch} of an "
                                    f"earlier region")
        batch_slots, other = set(), []
        for a in accesses:
            lead = a.idx[0] if a.idx else None
            if isinstance(lead, Aff) and v.id in lead.t:
                if lead.c != 0 or lead.t != {v.id: 1} or region.buffers[a.slot].shape[0] != B:
                    raise E.ModeUnsupported(f"sharded run: {region.buffers[a.slot]!r} is not "
                                            f"indexed [b, ...] by the batch loop")
                batch_slots.add(a.slot)
            elif a.offset is None or v.id in a.offset.t:
                raise E.ModeUnsupported(f"sharded run: an access to {region.buffers[a.slot]!r} "
                                        f"moves with the batch loop off its leading index")
            else:
                other.append(a)
        for a in other:
            if a.slot in batch_slots:
                raise E.ModeUnsupported(f"sharded run: {region.buffers[a.slot]!r} is also "
                                        f"accessed outside its batch row")
            if a.write:
                raise E.ModeUnsupported(f"sharded run: writes {region.buffers[a.slot]!r}, "
                                        f"which is not a batch buffer")
        for a in accesses:
            if a.write:
                self.written.add(id(region.buffers[a.slot]))
        for slot in batch_slots:
            buf = region.buffers[slot]
            self.buffers[id(buf)] = buf
            stage_rows = getattr(stage, "rows", None)
            if stage_rows is not None:
                stage_rows[id(buf)] = self.rows
        r0, r1 = self.rows
        v.lb, v.ub = Aff(r0), Aff(r1)
        self.regions += 1


class ShardResult:
    """What shard.run returns: the reference run()'s (results, stats) plus
    this rank's rows and the batch buffers."""

    def __init__(self, results, stats, shard, args, staging=None):
        self.results, self.stats = results, stats
        self.staging = staging   # the run's device copies (runtime.Staging) or None
        self.rank, self.world = shard.rank, shard.world
        self.rows = shard.rows
        self.batch = shard.batch
        # the batch buffers the run writes (its outputs; gather() moves these)
        self.buffers = [b for b in args if id(b) in shard.buffers and id(b) in shard.written]


def _dist():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def run(module, func, args, rank=None, world=None, mode="sequential", backend=None):
    """Run ``func`` of ``module`` on this rank's batch shard.

    ``rank`` / ``world`` default to torch.distributed's (or 0 / 1).  Returns
    a ShardResult; the Buffers hold this rank's rows of every batch buffer
    after the run (other rows keep their host contents)."""
    from staircase.interp import machine

    from . import engine

    if rank is None or world is None:
        rank, world = _dist()
    sh = Shard(rank, world)

    class _Eng:
        ExecContext = engine.ExecContext

        @staticmethod
        def run_tape(program, code, regs, tally, ctx):
            return engine.run_tape(program, code, regs, tally, ctx, backend=backend, shard=sh)

    results, stats = machine.run(module, func, args, mode=mode, engine=_Eng)
    return ShardResult(results, stats, sh, args, engine.last_staging)


def gather(res, group=None, to_host=True):
    """All-gather every batch buffer's rows over the ranks — one NCCL
    all_gather per buffer on the GPUs (gloo on CPU) — so each rank holds the
    whole batch: the unsharded run's result.  On the GPU path the rows are
    gathered into the run's device copies (device to device over NVLink);
    ``to_host`` then writes them back to the host Buffers.  Unequal chunks
    are padded to the largest.  Returns the bytes this rank received."""
    import numpy as np
    import torch
    import torch.distributed as dist

    if res.world == 1:
        return 0
    use_cuda = dist.get_backend(group) == "nccl"
    bounds = [chunk(res.batch, r, res.world) for r in range(res.world)]
    most = max(hi - lo for lo, hi in bounds)
    r0, r1 = res.rows
    got = 0
    for buf in res.buffers:
        dt = np.dtype({"f32": np.float32, "f64": np.float64, "i32": np.int32,
                       "i64": np.int64}[buf.dtype])
        host = torch.from_numpy(np.frombuffer(buf.data, dtype=dt)).view(buf.shape[0], -1)
        ent = res.staging.dev.get(id(buf)) if (use_cuda and res.staging is not None) else None
        full = ent[1].view(buf.shape[0], -1) if ent is not None and ent[0] is buf else None
        if full is None:
            full = host.to("cuda") if use_cuda else host
        width = full.shape[1]
        mine = torch.zeros(most, width, dtype=full.dtype, device=full.device)
        mine[:r1 - r0].copy_(full[r0:r1])
        out = torch.empty(res.world * most, width, dtype=full.dtype, device=full.device)
        if use_cuda:
            dist.all_gather_into_tensor(out, mine, group=group)
        else:
            dist.all_gather(list(out.chunk(res.world)), mine, group=group)
        for r, (lo, hi) in enumerate(bounds):
            if r != res.rank:
                full[lo:hi].copy_(out[r * most:r * most + hi - lo])
                got += (hi - lo) * width * dt.itemsize
        if to_host and full.data_ptr() != host.data_ptr():
            host.copy_(full)
    return got


__all__ = ["chunk", "run", "gather", "Shard", "ShardResult"]
