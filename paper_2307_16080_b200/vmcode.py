"""Encode a region's per-thread program for the device tape VM (csrc/vm.cu).

The VM is the generic execution tier: it runs any lifted region exactly
like the reference's ``run_tape`` (staircase/interp/_evalpy.py:81-331), one
band point per GPU thread.  Band loops are removed from the program — their
induction registers are bound from the thread index before the program
starts — while every other loop, branch, load, store and arithmetic op is
executed in reference order inside the thread.  ``scf.parallel`` and
``gpu.launch_func`` nodes that are not in the band are lowered to ordinary
nested loops in row-major / (bx,by,bz,tx,ty,tz) order.

Word format (int32): ``op | (tally_tag + 1) << 8 | flags << 16`` followed
by operands.  ``tally_tag`` is the reference opcode whose counter the
instruction increments when the program is run in counting mode
(-1 = not counted; the chain part is counted analytically on the host).
All floating values live in 64-bit registers as doubles, exactly like the
reference's Python floats; f32 arithmetic is rounded per operation with
``__f*_rn`` intrinsics (no FMA contraction).
"""
from __future__ import annotations

import struct

from .lift import (ALLOC, BINF, BINI, CALL, CAST, CMPF, CMPI, CONST, DEALLOC, GPUID, JUMP,
                   RETURN, LAUNCH, LOAD, LOOP_INIT_A, LOOP_INIT_S, LOOP_NEXT_I,
                   LOOP_NEXT_R, LOOP_TEST_I, LOOP_TEST_R, PARALLEL, RETURN_GPU,
                   STORE, IF_FALSE, If, Ins, Launch, Loop, Par, Unsupported)

# VM opcodes (csrc/vm.cu)
V_END, V_CONST, V_BINF, V_BINI, V_CMPF, V_CMPI, V_CAST, V_LOAD, V_STORE, V_MOV, \
    V_TEST, V_NEXT, V_JUMP, V_IFF, V_PCHECK, V_NOP, V_ZERO = range(17)

DTYPE_CODE = {"f32": 0, "f64": 1, "i32": 2, "i64": 3}
MAX_REGS = 256


def _split64(bits):
    lo = bits & 0xFFFFFFFF
    hi = (bits >> 32) & 0xFFFFFFFF
    return [lo - (1 << 32) if lo >= 1 << 31 else lo,
            hi - (1 << 32) if hi >= 1 << 31 else hi]


def value_bits(v):
    """64-bit register image of a host scalar (double bits or int64)."""
    if isinstance(v, float):
        return struct.unpack("<q", struct.pack("<d", v))[0]
    return int(v)


class VMProgram:
    __slots__ = ("words", "init_regs", "init_vals", "n_regs", "band", "locs",
                 "count")

    def __init__(self):
        self.words = []
        self.init_regs = []
        self.init_vals = []
        self.n_regs = 0
        self.band = []       # list of (vreg, lb, step, trip)
        self.locs = []
        self.count = False


class _Enc:
    def __init__(self, region, band_ids, count, checked):
        self.r = region
        self.band = set(band_ids)
        self.count = count
        self.checked = checked
        self.p = VMProgram()
        self.w = self.p.words
        self.n_regs = region.n_vregs
        self.consts = {}
        self.loc_ids = {}

    # -- helpers
    def head(self, op, tag, flags=0):
        t = tag if (self.count and tag is not None) else -1
        self.w.append(op | ((t + 1) << 8) | (flags << 16))

    def const_reg(self, value):
        key = (type(value), value)
        if key not in self.consts:
            reg = self.n_regs
            self.n_regs += 1
            self.consts[key] = reg
            self.p.init_regs.append(reg)
            self.p.init_vals.append(value_bits(value))
        return self.consts[key]

    def temp_reg(self):
        reg = self.n_regs
        self.n_regs += 1
        return reg

    def loc(self, loc):
        if loc is None:
            return -1
        k = id(loc)
        if k not in self.loc_ids:
            self.loc_ids[k] = len(self.p.locs)
            self.p.locs.append(loc)
        return self.loc_ids[k]

    # -- emission
    def leaf(self, n, tag_on=True):
        op = n.op
        tag = op if tag_on else None
        if op == CONST:
            self.head(V_CONST, tag)
            self.w.append(n.dst)
            self.w.extend(_split64(value_bits(n.value)))
        elif op == BINF:
            self.head(V_BINF, tag, n.sub | (int(n.f32) << 2))
            self.w.extend([n.dst, n.a, n.b])
        elif op == BINI:
            self.head(V_BINI, tag, n.sub | (int(n.f32) << 2))
            self.w.extend([n.dst, n.a, n.b])
        elif op == CMPF:
            self.head(V_CMPF, tag, n.sub)
            self.w.extend([n.dst, n.a, n.b])
        elif op == CMPI:
            self.head(V_CMPI, tag, n.sub)
            self.w.extend([n.dst, n.a, n.b])
        elif op == CAST:
            self.head(V_CAST, tag, int(n.f32))
            self.w.extend([n.dst, n.a])
        elif op in (LOAD, STORE):
            buf = self.r.env[n.b]
            slot = self.r.buf_slot[id(buf)]
            rank = len(n.idx)
            if rank != len(buf.shape) or rank > 8:
                raise Unsupported("memref access rank mismatch")
            flags = rank | (int(self.checked) << 4) | (DTYPE_CODE[buf.dtype] << 5)
            self.head(V_LOAD if op == LOAD else V_STORE, tag, flags)
            self.w.append(n.dst if op == LOAD else n.a)
            self.w.append(slot)
            self.w.extend(n.idx)
            self.w.append(self.loc(n.loc))
        elif op == GPUID:
            self.head(V_MOV, tag)
            self.w.extend([n.dst, n.a])
        elif op in (JUMP, DEALLOC, RETURN_GPU, CALL, RETURN):
            self.head(V_NOP, tag)
        elif op == ALLOC:
            # fresh zero-filled scratch (lift._leaf): V_ZERO slot, elements
            buf = n.value
            size = 1
            for d in buf.shape:
                size *= d
            if size >= 1 << 31:
                raise Unsupported("memref.alloc too large for the VM")
            self.head(V_ZERO, tag, DTYPE_CODE[buf.dtype])
            self.w.extend([self.r.buf_slot[id(buf)], size])
        else:
            raise Unsupported(f"VM cannot encode opcode {op}")

    def loop(self, iv, lb_reg, ub_reg, step_reg, body_fn, tags, bk, chk):
        """Emit MOV/TEST/body/NEXT; tags = (init, test, next) or None."""
        ti, tt, tn = tags if tags else (None, None, None)
        self.head(V_MOV, ti)
        self.w.extend([iv, lb_reg])
        head_pc = len(self.w)
        self.head(V_TEST, tt, int(bk and self.count and tags is not None))
        self.w.extend([iv, ub_reg, -1])
        patch = len(self.w) - 1
        body_fn()
        self.head(V_NEXT, tn, int(chk))
        self.w.extend([iv, step_reg, head_pc])
        self.w[patch] = len(self.w)

    def block(self, nodes, tag_on):
        for n in nodes:
            self.node(n, tag_on)

    def node(self, n, tag_on):
        if isinstance(n, Ins):
            self.leaf(n, tag_on)
        elif isinstance(n, Loop):
            if n.scf:
                lb, ub, st = n.lb, n.ub, n.step
                tags = (LOOP_INIT_S, LOOP_TEST_R, LOOP_NEXT_R)
            else:
                lb, ub, st = (self.const_reg(int(n.lb)), self.const_reg(int(n.ub)),
                              self.const_reg(int(n.step)))
                tags = (LOOP_INIT_A, LOOP_TEST_I, LOOP_NEXT_I)
            self.loop(n.var.vreg, lb, ub, st, lambda: self.block(n.body, tag_on),
                      tags if tag_on else None, bk=True, chk=n.scf)
        elif isinstance(n, Par):
            self.head(V_NOP, PARALLEL if tag_on else None)
            self.head(V_PCHECK, None, len(n.steps))
            self.w.extend(n.steps)
            self._nest(list(zip(n.vars, n.lbs, n.ubs, n.steps)),
                       lambda: self.block(n.body, tag_on), tag_on)
        elif isinstance(n, Launch):
            self.head(V_NOP, LAUNCH if tag_on else None)
            zero, one = self.const_reg(0), self.const_reg(1)
            dims = [(v, zero, ext, one) for v, ext in zip(n.vars, n.grid + n.block)]
            self._nest(dims, lambda: self.block(n.body, tag_on), tag_on)
        elif isinstance(n, If):
            self.head(V_IFF, IF_FALSE if tag_on else None)
            self.w.extend([n.cond, -1])
            patch = len(self.w) - 1
            self.block(n.then, tag_on)
            if n.has_jump:
                self.head(V_JUMP, JUMP if tag_on else None)
                self.w.append(-1)
                jpatch = len(self.w) - 1
                self.w[patch] = len(self.w)
                self.block(n.els, tag_on)
                self.w[jpatch] = len(self.w)
            else:
                self.w[patch] = len(self.w)
        else:
            raise Unsupported(f"VM cannot encode {type(n).__name__}")

    def _nest(self, dims, body_fn, tag_on):
        """Row-major nested loops; one bookkeeping count per point."""
        if not dims:
            body_fn()
            return
        (var, lb, ub, st), rest = dims[0], dims[1:]
        innermost = not rest
        self.head(V_MOV, None)
        self.w.extend([var.vreg, lb])
        head_pc = len(self.w)
        self.head(V_TEST, None, int(innermost and tag_on and self.count))
        self.w.extend([var.vreg, ub, -1])
        patch = len(self.w) - 1
        self._nest(rest, body_fn, tag_on)
        self.head(V_NEXT, None, 0)
        self.w.extend([var.vreg, st, head_pc])
        self.w[patch] = len(self.w)


def encode(region, links, remainder, band_ids, count, checked, max_regs=MAX_REGS):
    """Build the VM program for ``region`` with ``band_ids`` bound per thread.

    ``links``/``remainder`` come from analysis.chain_of.  Chain levels are
    emitted untagged (their counts are added analytically); the remainder is
    tagged when ``count`` is set.  ``max_regs``: the register file of the
    tier that will run it — the interpreter's MAX_REGS, or None for the
    native tier (native.py: registers become scalars, no limit).
    """
    e = _Enc(region, band_ids, count, checked)

    def emit_chain(i):
        if i == len(links):
            e.block(remainder, True)
            return
        link = links[i]
        node = link.node
        for leaf in link.pure:
            e.leaf(leaf, tag_on=False)
        if isinstance(node, Loop):
            var = node.var
            if var.id in e.band:
                emit_chain(i + 1)
            else:
                lb, st, trip = var.static()
                e.loop(var.vreg, e.const_reg(lb), e.const_reg(lb + st * trip),
                       e.const_reg(st), lambda: emit_chain(i + 1), None,
                       bk=False, chk=False)
        else:
            dims = []
            for var in link.vars:
                if var.id in e.band:
                    continue
                lb, st, trip = var.static()
                dims.append((var, e.const_reg(lb), e.const_reg(lb + st * trip),
                             e.const_reg(st)))
            e._nest(dims, lambda: emit_chain(i + 1), False)

    emit_chain(0)
    e.head(V_END, None)
    p = e.p
    p.n_regs = e.n_regs
    if max_regs is not None and p.n_regs > max_regs:
        raise Unsupported(f"region needs {p.n_regs} VM registers (max {max_regs} without "
                          f"the native tier)")
    # initial register images: environment scalars
    for v, val in region.env.items():
        kind = region.kind[v]
        if kind == "buf":
            continue
        p.init_regs.append(v)
        p.init_vals.append(value_bits(val))
    for vid in band_ids:
        var = region.vars[vid]
        lb, st, trip = var.static()
        p.band.append((var.vreg, lb, st, trip))
    p.count = count
    return p
