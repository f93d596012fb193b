"""Race check of ``scf.parallel`` bodies: static-affine proof first.

The reference's ``check_races(module, func, args)`` (staircase/interp/
races.py:20-97) simulates the whole program sequentially on copies of the
arguments in ``gpu_emulated`` mode, recording which iteration of each
outermost ``scf.parallel`` touches every buffer address, and returns the
conflicting ``(point, point, address)`` triples.  At the paper's sizes that
simulation is hours of Python.

``check_races`` here has the same signature and result.  It runs the program
once through the B200 engine (on copies, ``gpu_emulated``) and decides every
region on the device side:

1. *static proof*: the engine's band analysis (analysis.band_ok — the test
   that decides which loops run on parallel GPU threads) shows the
   iteration variables of each outermost parallel race-free: every written
   buffer accessed through affine offsets with identical coefficients on
   them, distinct iterations mapped to disjoint location sets.  No conflict.
2. *device recorder* (record_region): for a region whose outermost parallel
   is not proven — a genuine race, non-affine but data-independent indices
   (y[i*i]) — one GPU thread per parallel point replays the point's address
   stream and three passes of shadow-memory atomics reproduce the
   reference recorder's conflict list, in its order.
3. anything else (indices computed from loaded data, parallels inside
   sequential loops, memref.alloc) falls back to the reference's own
   simulation, whose exact list is returned.
"""
from __future__ import annotations

from .host import ensure_staircase


def _outermost_pars(nodes, inside=False):
    """Par nodes not nested in another Par (Launch / Loop / If ancestors ok)."""
    from .lift import If, Launch, Loop, Par

    for n in nodes:
        if isinstance(n, Par):
            if not inside:
                yield n
            yield from _outermost_pars(n.body, True)
        elif isinstance(n, (Loop, Launch)):
            yield from _outermost_pars(n.body, inside)
        elif isinstance(n, If):
            yield from _outermost_pars(n.then, inside)
            yield from _outermost_pars(n.els, inside)


def region_race_free(region, accesses):
    """True iff every outermost parallel of the region is proven race-free."""
    from . import analysis

    for par in _outermost_pars(region.tree):
        ids = [v.id for v in par.vars]
        if any(region.vars[i].static() is None for i in ids):
            return False
        inside = {id(n) for n in analysis._iter_nodes(par.body)}
        accs = [a for a in accesses if id(a.node) in inside]
        written = sorted({a.slot for a in accs if a.write})
        if not analysis.band_ok(region, accs, ids, written):
            return False
    return True


def _data_independent(region):
    """No loaded value flows into an address, a branch or a loop bound: the
    region's access stream is a function of its loop variables and host
    scalars alone (so it can be replayed without the data, in parallel)."""
    from .analysis import _iter_nodes
    from .lift import LOAD, STORE, If, Ins, Launch, Loop, Par

    ins = [n for n in _iter_nodes(region.tree) if isinstance(n, Ins)]
    tainted = {n.dst for n in ins if n.op == LOAD}
    changed = True
    while changed:
        changed = False
        for n in ins:
            if n.dst is not None and n.dst not in tainted and n.op != LOAD and \
                    (n.a in tainted or n.b in tainted):
                tainted.add(n.dst)
                changed = True
    for n in _iter_nodes(region.tree):
        if isinstance(n, Ins) and n.op in (LOAD, STORE) and any(i in tainted for i in n.idx):
            return False
        if isinstance(n, If) and n.cond in tainted:
            return False
        if isinstance(n, Loop) and n.scf and {n.lb, n.ub, n.step} & tainted:
            return False
        if isinstance(n, Par) and set(n.lbs + n.ubs + n.steps) & tainted:
            return False
        if isinstance(n, Launch) and set(n.grid + n.block) & tainted:
            return False
    return True


def recordable(region, accesses, labels):
    """The device recorder reproduces the reference's conflicts for a region
    whose only outermost parallel is its top node (one execution of it),
    without memref.alloc, with data-independent addresses, over argument
    buffers only.  (Indices not provably in bounds are checked during the
    replay; a fault sends the program to the reference simulation, which
    raises it.)"""
    from . import analysis
    from .lift import Par

    if len(region.tree) != 1 or not isinstance(region.tree[0], Par):
        return False
    par = region.tree[0]
    if any(v.static() is None for v in par.vars) or region.has_alloc:
        return False
    if any(id(b) not in labels for b in region.buffers):
        return False
    if analysis.invalid_steps(region):
        return False
    return _data_independent(region)


def record_region(region, accesses, labels, cap=1 << 20):
    """The reference recorder's conflicts (interp/races.py:20-76) for one
    outermost scf.parallel, computed on the GPU.

    One thread per parallel point replays the point's access stream
    (native.vm_source(record=True): addresses only, no data).  Pass 0
    records per element the first writing point W and first reading point
    R1 (atomicMin), pass 1 the first reading point other than R1, R2; pass
    2 emits, per access of point q in program order, exactly the conflicts
    the sequential recorder reports at that access — read: (W, q) if W < q;
    write: (W, q) if W < q, then (R1, q), (R2, q) for readers before q (the
    recorder keeps two readers per address).  Sorting the events by (point,
    access number, kind) restores the recorder's detection order.  Returns
    [(point, point, (label, offset))] with duplicates kept for the caller's
    global dedup, or None when the replay faulted (out of bounds)."""
    import ctypes

    import numpy as np

    from . import analysis, jit, native, runtime, vmcode

    torch = runtime.torch_mod()
    lib = runtime.load_library()
    par = region.tree[0]
    links, remainder = analysis.chain_of(region)
    band = [v.id for v in par.vars]
    checked = not analysis.statically_in_bounds(region, accesses)
    prog = vmcode.encode(region, links, remainder, band, False, checked=checked,
                         max_regs=None)   # the recorder is always native code
    env_regs = [v for v in region.env if region.kind[v] != "buf"]
    src, name, _ = native.vm_source(prog, region.buffers, env_regs, record=True)
    fn = jit.compile_kernel(src, name)
    big = np.iinfo(np.int64).max
    shadows = []
    for b in region.buffers:
        n = 1
        for d in b.shape:
            n *= d
        shadows.append([torch.full((max(1, n),), big, dtype=torch.int64, device="cuda")
                        for _ in range(3)])
    sh = torch.tensor([t.data_ptr() for trio in shadows for t in trio] or [0],
                      dtype=torch.int64, device="cuda")
    ptrs = torch.zeros(max(1, len(region.buffers)), dtype=torch.int64, device="cuda")
    env = torch.tensor(prog.init_vals or [0], dtype=torch.int64, device="cuda")
    err = torch.zeros(ctypes.sizeof(runtime.B200VmError), dtype=torch.uint8, device="cuda")
    nev = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    grid = native.grid_of(prog)

    def launch(pass_id, ev, capacity):
        vals = [ctypes.c_void_p(ptrs.data_ptr()), ctypes.c_void_p(env.data_ptr()),
                ctypes.c_void_p(sh.data_ptr()), ctypes.c_void_p(ev.data_ptr()),
                ctypes.c_void_p(nev.data_ptr()), ctypes.c_int64(capacity),
                ctypes.c_int32(pass_id), ctypes.c_void_p(err.data_ptr())]
        argv = (ctypes.c_void_p * len(vals))(
            *[ctypes.cast(ctypes.byref(v), ctypes.c_void_p) for v in vals])
        runtime.check(lib.b200_jit_launch(ctypes.c_void_p(fn), grid, 1, 1, native.THREADS, 1,
                                          1, 0, argv, stream), "race recorder")

    ev = torch.empty(6 * cap, dtype=torch.int64, device="cuda")
    launch(0, ev, cap)
    if checked and int(err[:4].view(torch.int32).item()) != 0:
        return None   # an out-of-bounds access: the reference simulation raises it
    launch(1, ev, cap)
    launch(2, ev, cap)
    n = int(nev.item())
    if n > cap:   # more events than room: once more with exactly enough
        cap = n
        ev = torch.empty(6 * cap, dtype=torch.int64, device="cuda")
        nev.zero_()
        launch(2, ev, cap)
        n = int(nev.item())
    e = ev[:6 * n].view(n, 6).cpu().numpy()
    order = np.lexsort((e[:, 2], e[:, 1], e[:, 0]))
    geo = [v.static() for v in par.vars]

    def point(q):
        idx = []
        for lb, st, trip in reversed(geo):
            idx.append(lb + st * (q % trip))
            q //= trip
        return tuple(reversed(idx))

    name_of = [labels[id(b)] for b in region.buffers]
    return [(point(int(e[i, 3])), point(int(e[i, 0])), (name_of[int(e[i, 4])], int(e[i, 5])))
            for i in order]


def check_races(module, func_name, args, engine=None):
    """The reference's check_races result (interp/races.py:78-97), computed
    without simulating the program on the CPU whenever possible.

    ``engine`` (default: the B200 engine) runs the program once on copies of
    ``args`` (``gpu_emulated``, like the reference); every region is then
    either proven race-free statically (region_race_free), or — on the GPU
    engine — its conflicts are recorded on the device (record_region),
    in the reference recorder's order.  Regions neither can handle (data-
    dependent addresses, parallels inside sequential loops, allocs) fall back
    to the reference's own simulation of the whole program.
    """
    ensure_staircase()
    from staircase.interp import Buffer, machine
    from staircase.interp.races import check_races as reference_check

    from . import engine as b2engine

    eng = engine or b2engine
    device = eng is b2engine
    copies = [a.copy() if isinstance(a, Buffer) else a for a in args]
    labels = {id(v): f"arg{i}" for i, v in enumerate(copies) if isinstance(v, Buffer)}
    found, fallback = [], []

    def hook(r, acc):
        if region_race_free(r, acc):
            return
        got = record_region(r, acc, labels) if device and recordable(r, acc, labels) else None
        if got is None:
            fallback.append(True)
        else:
            found.extend(got)

    try:
        with b2engine.region_hook(hook):
            machine.run(module, func_name, copies, mode="gpu_emulated", engine=eng)
    except Exception:
        fallback.append(True)   # let the reference reproduce whatever happened
    if fallback:
        return reference_check(module, func_name, args)
    out, seen = [], set()
    for c in found:
        if c not in seen:
            seen.add(c)
            out.append(c)
    return out


__all__ = ["check_races", "region_race_free", "record_region", "recordable"]
