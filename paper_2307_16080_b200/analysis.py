"""Region analysis: accesses, static bounds, the parallel band, the static tally.

Given a lifted region (lift.py) this decides how the GPU may execute it
without changing any observable result of the reference's sequential
semantics (staircase/interp/_evalpy.py:81-331):

* **chain** — the perfectly nested prefix of loop-like nodes (scf.for,
  affine.for, scf.parallel dims, gpu.launch grid/block dims) whose bodies
  hold only pure scalar ops besides the next chain node, with static bounds.
* **band** — the subset of chain variables distributed over GPU threads.
  A set B is legal when, for every buffer the region writes, every access
  to it has an affine offset, all accesses share the same coefficients on
  B, and B-points map to pairwise disjoint location sets (a mixed-radix
  injectivity check against the span of the non-B remainder).  Then each
  B-point's iterations touch locations no other B-point reads or writes, so
  running B-points concurrently and everything else in original order is
  equivalent to the reference's sequential execution — including
  ``scf.parallel`` loops that *do* race (they simply do not enter the band
  and execute in reference order).
* **bounds** — if every access is affine and its per-dimension index range
  over the iteration domain lies inside the buffer extents, no OutOfBounds
  can occur and the kernel runs unchecked.  Otherwise the region runs
  *checked*: sequentially on one GPU thread, which reproduces the first
  faulting access (and the partial writes before it) exactly like the
  reference.
* **tally** — the per-opcode counters of ``run_tape`` (tally[op] += 1 per
  executed instruction, tally[-1] per loop-body entry / parallel point /
  gpu thread; _evalpy.py:87,145,150,265,327) computed analytically when the
  region's control flow is static, else counted on the device.
"""
from __future__ import annotations

from .lift import (BOOKKEEPING, CAST, CMPF, CMPI, CONST, BINF, BINI, GPUID, JUMP,
                   IF_FALSE, LAUNCH, LOAD, LOOP_INIT_A, LOOP_INIT_S, LOOP_NEXT_I,
                   LOOP_NEXT_R, LOOP_TEST_I, LOOP_TEST_R, N_OPCODES, PARALLEL, RETURN_GPU,
                   PURE_OPS, STORE, EMPTY, Aff, If, Ins, Launch, Loop, Par,
                   aff_range, prod, var_range)


# leaves allowed beside a chain loop: pure scalar ops and the kernel's
# gpu.return (a no-op for memory; counted in the tally like any leaf)
CHAIN_LEAVES = PURE_OPS | {RETURN_GPU}


class Access:
    __slots__ = ("slot", "idx", "offset", "write", "loc", "node")

    def __init__(self, slot, idx, offset, write, loc, node):
        self.slot = slot        # buffer slot in region.buffers
        self.idx = idx          # tuple of Aff|None per dim
        self.offset = offset    # Aff (row-major element offset) or None
        self.write = write
        self.loc = loc
        self.node = node


def _iter_nodes(nodes):
    for n in nodes:
        yield n
        if isinstance(n, (Loop, Par, Launch)):
            yield from _iter_nodes(n.body)
        elif isinstance(n, If):
            yield from _iter_nodes(n.then)
            yield from _iter_nodes(n.els)


def collect_accesses(region):
    out = []
    for n in _iter_nodes(region.tree):
        if isinstance(n, Ins) and n.op in (LOAD, STORE):
            buf = region.env.get(n.b)
            if buf is None:
                from .lift import Unsupported
                raise Unsupported("memref operand is not a function argument")
            slot = region.buf_slot[id(buf)]
            idx = tuple(region.sym.get(v) if isinstance(region.sym.get(v), Aff) else None
                        for v in n.idx)
            off = None
            if all(i is not None for i in idx) and len(idx) == len(buf.shape):
                off = Aff(0)
                for i, s in zip(idx, buf.strides):
                    off = off + i.scale(s)
            out.append(Access(slot, idx, off, n.op == STORE, n.loc, n))
    return out


def statically_in_bounds(region, accesses):
    """True iff no access can go out of bounds (exact for affine indices)."""
    memo = {}   # variable ranges, shared by every index of the region
    for a in accesses:
        buf = region.buffers[a.slot]
        if len(a.idx) != len(buf.shape):
            return False
        for i, extent in zip(a.idx, buf.shape):
            if i is None:
                return False
            r = aff_range(region, i, memo)
            if r is None:
                return False
            if r is EMPTY or r[1] < r[0]:
                break   # the access never executes
            if r[0] < 0 or r[1] >= extent:
                return False
    return True


# -- chain & band ----------------------------------------------------------------


class ChainLink:
    """One chain level: a node plus its variables (1 for loops, n for par/launch)."""

    __slots__ = ("node", "vars", "pure")

    def __init__(self, node, vars_, pure):
        self.node = node
        self.vars = vars_
        self.pure = pure        # pure Ins leaves in this node's body (duplicated per thread)


def chain_of(region):
    """The perfectly nested, statically bounded prefix of loop-like nodes."""
    links = []
    seq = region.tree
    while True:
        loops = [n for n in seq if not isinstance(n, Ins)]
        leaves = [n for n in seq if isinstance(n, Ins)]
        if len(loops) != 1 or any(x.op not in CHAIN_LEAVES for x in leaves):
            break
        node = loops[0]
        if isinstance(node, Loop):
            vars_ = [node.var]
        elif isinstance(node, (Par, Launch)):
            vars_ = list(node.vars)
        else:
            break
        if any(v.static() is None for v in vars_):
            break
        # a non-terminal position of the loop in its block would need the
        # pure ops after it to run after the whole nest; they are pure and
        # unobservable, so order does not matter.
        links.append(ChainLink(node, vars_, leaves))
        seq = node.body
    return links, seq


def _mixed_radix_injective(terms, span):
    """terms: list of (|coef*step|, trip).  True iff sum(coef_i * t_i) + r,
    t_i in [0, trip_i), r in [0, span], is injective in (t, r) classes."""
    acc = span
    for g, trip in sorted(terms):
        if trip <= 1:
            continue
        if g == 0 or g <= acc:
            return False
        acc += g * (trip - 1)
    return True


def band_ok(region, accesses, band_ids, written, memo=None):
    if memo is None:
        memo = {}
    for slot in written:
        accs = [a for a in accesses if a.slot == slot]
        if any(a.offset is None for a in accs):
            return False
        coefs = None
        lo = hi = None
        for a in accs:
            c = tuple(a.offset.t.get(v, 0) for v in band_ids)
            if coefs is None:
                coefs = c
            elif c != coefs:
                return False
            rest = Aff(a.offset.c, {k: v for k, v in a.offset.t.items()
                                    if k not in band_ids})
            r = aff_range(region, rest, memo)
            if r is None:
                return False
            if r is EMPTY:
                continue
            lo = r[0] if lo is None else min(lo, r[0])
            hi = r[1] if hi is None else max(hi, r[1])
        if coefs is None or lo is None:
            continue
        terms = []
        for vid, c in zip(band_ids, coefs):
            lb, st, trip = region.vars[vid].static()
            terms.append((abs(c * st), trip))
        if not _mixed_radix_injective(terms, hi - lo):
            return False
    return True


def choose_band(region, links, accesses):
    """The chain variables to distribute over GPU threads: greedily, in nest
    order, every variable whose addition keeps the band provably race-free
    — repeated until nothing changes, since a tiled nest's origin loop
    (passes/tiling.py:56-80) is only provable once the offset loop of the
    other dimension is in the band.  Returned in nest order."""
    written = sorted({a.slot for a in accesses if a.write})
    order = [v.id for link in links for v in link.vars]
    memo = {}   # variable ranges: fixed for the region, shared by every trial band
    band = []
    changed = True
    while changed:
        changed = False
        for vid in order:
            if vid in band:
                continue
            trial = sorted(band + [vid], key=order.index)
            if band_ok(region, accesses, trial, written, memo):
                band = trial
                changed = True
    return band


# -- static tally ---------------------------------------------------------------


def _loop_ops(node):
    if node.scf:
        return LOOP_INIT_S, LOOP_TEST_R, LOOP_NEXT_R
    return LOOP_INIT_A, LOOP_TEST_I, LOOP_NEXT_I


def static_tally(nodes, mult=1, tally=None):
    """Exact counts for statically bounded, branch-free trees, else None."""
    if tally is None:
        tally = [0] * (N_OPCODES + 1)
    for n in nodes:
        if isinstance(n, Ins):
            tally[n.op] += mult
        elif isinstance(n, Loop):
            s = n.var.static()
            if s is None:
                return None
            trip = s[2]
            i_op, t_op, n_op = _loop_ops(n)
            tally[i_op] += mult
            tally[t_op] += mult * (trip + 1)
            tally[n_op] += mult * trip
            tally[BOOKKEEPING] += mult * trip
            if trip and static_tally(n.body, mult * trip, tally) is None:
                return None
        elif isinstance(n, Par):
            stat = [v.static() for v in n.vars]
            if any(s is None for s in stat):
                return None
            pts = prod(s[2] for s in stat)
            tally[PARALLEL] += mult
            tally[BOOKKEEPING] += mult * pts
            if pts and static_tally(n.body, mult * pts, tally) is None:
                return None
        elif isinstance(n, Launch):
            stat = [v.static() for v in n.vars]
            if any(s is None for s in stat):
                return None
            pts = prod(s[2] for s in stat)
            tally[LAUNCH] += mult
            tally[BOOKKEEPING] += mult * pts
            if pts and static_tally(n.body, mult * pts, tally) is None:
                return None
        elif isinstance(n, If):
            return None
    return tally


def chain_tally(links):
    """Counts contributed by the chain levels themselves (loops + pure ops)."""
    tally = [0] * (N_OPCODES + 1)
    mult = 1
    for link in links:
        node = link.node
        # link.pure are the node's siblings: they run once per parent-body entry
        for leaf in link.pure:
            tally[leaf.op] += mult
        if isinstance(node, Loop):
            trip = node.var.static()[2]
            i_op, t_op, n_op = _loop_ops(node)
            tally[i_op] += mult
            tally[t_op] += mult * (trip + 1)
            tally[n_op] += mult * trip
            tally[BOOKKEEPING] += mult * trip
            mult *= trip
        else:
            pts = prod(v.static()[2] for v in link.vars)
            tally[PARALLEL if isinstance(node, Par) else LAUNCH] += mult
            tally[BOOKKEEPING] += mult * pts
            mult *= pts
    return tally, mult


def invalid_steps(region):
    """True if some loop/parallel step is <= 0 where the reference raises."""
    for v in region.vars:
        if v.kind in ("for", "par") and v.step is not None and v.step.is_const() \
                and v.step.c <= 0:
            return True
    return False


__all__ = ["collect_accesses", "statically_in_bounds", "chain_of", "choose_band",
           "static_tally", "chain_tally", "Access", "ChainLink", "invalid_steps",
           "var_range"]
