"""Lift a region of a staircase tape into a loop tree with affine indices.

The reference executes a flat instruction tape (staircase/interp/tape.py:20-45,
compiled by ``_Compiler`` at tape.py:101-274).  The B200 engine offloads every
top-level loop nest, ``scf.parallel`` and ``gpu.launch_func`` of that tape as
one *region*.  This module turns such a region back into structure:

- loops (LOOP_INIT/TEST/NEXT triples, tape.py:233-250) become ``Loop`` nodes,
- ``PARALLEL`` sub-tapes (tape.py:264-274) become ``Par`` nodes whose register
  file is merged into the region's virtual register space through the
  capture list,
- ``LAUNCH`` (tape.py:217-223) becomes a ``Launch`` node over the kernel tape,
- ``IF_FALSE``/``JUMP`` pairs (tape.py:252-262) become ``If`` nodes,
- every other instruction stays a leaf ``Ins`` with renamed registers.

Because tape registers are SSA (one defining instruction each), every index
register has a single symbolic value: an affine form over the region's
iteration variables, a constant, or "data" (unknown).  Registers defined
outside the region are concrete host values (``env``) at offload time.
"""
from __future__ import annotations

import math

# opcodes (staircase/interp/tape.py:20-45)
CONST, BINF, BINI, CMPF, CMPI, CAST, LOAD, STORE, ALLOC, DEALLOC = range(10)
LOOP_INIT_S, LOOP_INIT_A, LOOP_TEST_R, LOOP_TEST_I, LOOP_NEXT_R, LOOP_NEXT_I = range(10, 16)
JUMP, IF_FALSE, PARALLEL, CALL, RETURN, LAUNCH, GPUID, RETURN_GPU = range(16, 24)
N_OPCODES = 24
BOOKKEEPING = N_OPCODES  # tally[-1]

PURE_OPS = frozenset({CONST, BINF, BINI, CMPF, CMPI, CAST, GPUID})


class Unsupported(Exception):
    """Region shape the device backend does not execute (→ ModeUnsupported)."""


# -- affine forms ---------------------------------------------------------------


class Aff:
    """c + sum(coef * var) with integer coefficients; vars are Var ids."""

    __slots__ = ("c", "t")

    def __init__(self, c=0, t=None):
        self.c = int(c)
        self.t = {k: v for k, v in (t or {}).items() if v}

    @staticmethod
    def var(vid):
        return Aff(0, {vid: 1})

    def is_const(self):
        return not self.t

    def __add__(self, o):
        t = dict(self.t)
        for k, v in o.t.items():
            t[k] = t.get(k, 0) + v
        return Aff(self.c + o.c, t)

    def __sub__(self, o):
        t = dict(self.t)
        for k, v in o.t.items():
            t[k] = t.get(k, 0) - v
        return Aff(self.c - o.c, t)

    def scale(self, k):
        return Aff(self.c * k, {v: c * k for v, c in self.t.items()})

    def __eq__(self, o):
        return isinstance(o, Aff) and self.c == o.c and self.t == o.t

    def __hash__(self):
        return hash((self.c, tuple(sorted(self.t.items()))))

    def __repr__(self):
        parts = [f"{c}*v{k}" for k, c in sorted(self.t.items())]
        return "Aff(" + " + ".join([str(self.c)] + parts) + ")"


# -- tree -----------------------------------------------------------------------


class Var:
    """An iteration variable: a loop iv, a parallel dim or a gpu id."""

    __slots__ = ("id", "vreg", "lb", "ub", "step", "kind", "node")

    def __init__(self, vid, vreg, kind):
        self.id = vid
        self.vreg = vreg
        self.kind = kind      # "for" | "par" | "gpu"
        self.lb = self.ub = self.step = None   # Aff (may reference outer vars)
        self.node = None

    def static(self):
        """(lb, step, trip) when all three are constants, else None."""
        if self.lb is None or not (self.lb.is_const() and self.ub.is_const()
                                   and self.step.is_const()):
            return None
        lb, ub, st = self.lb.c, self.ub.c, self.step.c
        if st <= 0:
            return None
        trip = max(0, -(-(ub - lb) // st))
        return lb, st, trip


class Ins:
    """A leaf instruction with registers renamed into the region's vregs.

    ``op`` is the tape opcode; fields follow tape.py:20-45 with registers
    replaced by vregs.  ``buf`` is the vreg of the memref operand.
    """

    __slots__ = ("op", "dst", "a", "b", "sub", "f32", "idx", "loc", "value", "srcs")

    def __init__(self, op):
        self.op = op
        self.dst = self.a = self.b = self.sub = None
        self.f32 = False
        self.idx = ()
        self.loc = None
        self.value = None
        self.srcs = ()


class Loop:
    __slots__ = ("var", "scf", "lb", "ub", "step", "body")

    def __init__(self, var, scf, lb, ub, step, body):
        self.var = var
        self.scf = scf          # True: scf.for (LOOP_*_R), False: affine.for (*_I)
        self.lb, self.ub, self.step = lb, ub, step   # vreg (scf) or int (affine)
        self.body = body


class Par:
    __slots__ = ("vars", "lbs", "ubs", "steps", "body")

    def __init__(self, vars_, lbs, ubs, steps, body):
        self.vars = vars_
        self.lbs, self.ubs, self.steps = lbs, ubs, steps   # vregs
        self.body = body


class Launch:
    __slots__ = ("vars", "grid", "block", "body", "loc", "key")

    def __init__(self, vars_, grid, block, body, loc, key):
        self.vars = vars_          # 6 Vars: bx, by, bz, tx, ty, tz
        self.grid, self.block = grid, block   # vregs
        self.body = body
        self.loc = loc
        self.key = key


class If:
    __slots__ = ("cond", "then", "els", "has_jump")

    def __init__(self, cond, then, els, has_jump):
        self.cond = cond
        self.then = then
        self.els = els
        self.has_jump = has_jump   # an else-skip JUMP executes after `then`


class Region:
    """A lifted region: tree + vreg metadata + iteration variables."""

    def __init__(self):
        self.n_vregs = 0
        self.vars = []          # Var by id
        self.var_of_vreg = {}   # vreg -> Var
        self.env = {}           # vreg -> host value (scalar or Buffer), defined outside
        self.sym = {}           # vreg -> Aff | float | None (symbolic value)
        self.kind = {}          # vreg -> "int" | "f32" | "f64" | "buf" | "bool"
        self.tree = []
        self.buffers = []       # distinct host Buffers referenced
        self.buf_slot = {}      # id(Buffer) -> slot
        self.has_if = False
        self.has_alloc = False
        self.has_launch = False
        self.outer = []         # (outer tape register, vreg) in first-read order

    def new_vreg(self):
        v = self.n_vregs
        self.n_vregs += 1
        return v

    def new_var(self, vreg, kind):
        var = Var(len(self.vars), vreg, kind)
        self.vars.append(var)
        self.var_of_vreg[vreg] = var
        return var


class _Frame:
    """Register renaming for one tape (function body, sub-tape or kernel)."""

    def __init__(self, region, parent_map=None):
        self.region = region
        self.map = dict(parent_map or {})

    def get(self, reg):
        v = self.map.get(reg)
        if v is None:
            raise Unsupported(f"register r{reg} used before definition in region")
        return v

    def define(self, reg):
        v = self.region.new_vreg()
        self.map[reg] = v
        return v


def lift_region(program, code, start, end, regs):
    """Lift ``code[start:end]`` of a tape whose live register file is ``regs``.

    Registers referenced but not defined inside the region are bound to their
    current host values (scalars or Buffers) — the environment.
    """
    from staircase.interp.buffer import Buffer  # host framework type

    region = Region()
    frame = _Frame(region)

    # Bind every outer register that currently holds a value; the region's
    # own definitions shadow them (SSA: no redefinition).
    env_map = {}
    for r, val in enumerate(regs):
        if val is None:
            continue
        env_map[r] = val
    frame.env_regs = env_map

    def outer(reg):
        if reg in frame.map:
            return frame.map[reg]
        if reg not in env_map:
            raise Unsupported(f"register r{reg} has no value at region entry")
        v = region.new_vreg()
        frame.map[reg] = v
        val = env_map[reg]
        region.env[v] = val
        region.outer.append((reg, v))
        if isinstance(val, Buffer):
            region.kind[v] = "buf"
            if id(val) not in region.buf_slot:
                region.buf_slot[id(val)] = len(region.buffers)
                region.buffers.append(val)
        elif isinstance(val, bool):
            region.kind[v] = "int"
        elif isinstance(val, float):
            region.kind[v] = "float"
        else:
            region.kind[v] = "int"
        return v

    frame.get = outer
    region.tree = _lift_block(program, code, start, end, frame, region)
    return region


def _lift_block(program, code, start, end, fr, region):
    out = []
    pc = start
    while pc < end:
        ins = code[pc]
        op = ins[0]
        if op in (LOOP_INIT_S, LOOP_INIT_A):
            test = code[pc + 1]
            if test[0] not in (LOOP_TEST_R, LOOP_TEST_I):
                raise Unsupported("malformed loop head")
            loop_end = test[3]
            nxt = code[loop_end - 1]
            if nxt[0] not in (LOOP_NEXT_R, LOOP_NEXT_I) or nxt[3] != pc + 1:
                raise Unsupported("malformed loop tail")
            scf = op == LOOP_INIT_S
            if scf:
                lb, ub, step = fr.get(ins[2]), fr.get(test[2]), fr.get(nxt[2])
            else:
                lb, ub, step = ins[2], test[2], nxt[2]
            ivreg = fr.define(ins[1])
            region.kind[ivreg] = "int"
            var = region.new_var(ivreg, "for")
            body = _lift_block(program, code, pc + 2, loop_end - 1, fr, region)
            node = Loop(var, scf, lb, ub, step, body)
            var.node = node
            out.append(node)
            pc = loop_end
            continue
        if op == IF_FALSE:
            region.has_if = True
            target = ins[2]
            cond = fr.get(ins[1])
            if target - 1 > pc and code[target - 1][0] == JUMP and \
                    code[target - 1][1] > target:
                skip = code[target - 1][1]
                then = _lift_block(program, code, pc + 1, target - 1, fr, region)
                els = _lift_block(program, code, target, skip, fr, region)
                out.append(If(cond, then, els, True))
                pc = skip
            else:
                then = _lift_block(program, code, pc + 1, target, fr, region)
                out.append(If(cond, then, [], False))
                pc = target
            continue
        if op == JUMP:
            if ins[1] != end:
                raise Unsupported("unstructured jump")
            out.append(Ins(JUMP))
            pc += 1
            continue
        if op == PARALLEL:
            sub = ins[1]
            lbs = tuple(fr.get(r) for r in ins[2])
            ubs = tuple(fr.get(r) for r in ins[3])
            steps = tuple(fr.get(r) for r in ins[4])
            sf = _Frame(region)
            for o, i in sub.captures:
                sf.map[i] = fr.get(o)
            vars_ = []
            for r in sub.index_regs:
                v = sf.define(r)
                region.kind[v] = "int"
                vars_.append(region.new_var(v, "par"))
            body = _lift_block(program, sub.code, 0, len(sub.code), sf, region)
            node = Par(vars_, lbs, ubs, steps, body)
            for v in vars_:
                v.node = node
            out.append(node)
            pc += 1
            continue
        if op == LAUNCH:
            region.has_launch = True
            kernel = program.funcs[ins[1]]
            grid = tuple(fr.get(r) for r in ins[2])
            block = tuple(fr.get(r) for r in ins[3])
            kf = _Frame(region)
            for dst, src in zip(kernel.arg_regs, ins[4]):
                kf.map[dst] = fr.get(src)
            vars_ = []
            for d in range(6):
                v = region.new_vreg()
                region.kind[v] = "int"
                vars_.append(region.new_var(v, "gpu"))
            kf.gpu_vars = vars_
            body = _lift_block(program, kernel.code, 0, len(kernel.code), kf, region)
            node = Launch(vars_, grid, block, body, ins[5], ins[1])
            for v in vars_:
                v.node = node
            out.append(node)
            pc += 1
            continue
        if op == CALL:
            out.extend(_inline_call(program, ins, fr, region))
            pc += 1
            continue
        if op == RETURN:
            raise Unsupported("return inside a loop region")
        out.append(_leaf(ins, fr, region))
        pc += 1
    return out


MAX_INLINE = 8


def _inline_call(program, ins, fr, region):
    """func.call inside a loop region, inlined (reference _evalpy.py:216-223:
    a fresh register file for the callee, its RETURN operands copied to the
    caller's result registers).  The CALL and the callee's RETURN stay in the
    tree as tally-only leaves (the reference counts both).  Callees with a
    RETURN anywhere but at the end, or nested deeper than MAX_INLINE
    (recursion), are not lifted."""
    depth = getattr(fr, "depth", 0)
    if depth >= MAX_INLINE:
        raise Unsupported("func.call nesting too deep inside a loop region")
    callee = program.funcs[ins[2]]
    ccode = callee.code
    if not ccode or ccode[-1][0] != RETURN or any(c[0] == RETURN for c in ccode[:-1]):
        raise Unsupported("a callee with an early return inside a loop region")
    cf = _Frame(region)
    cf.depth = depth + 1
    for dst, src in zip(callee.arg_regs, ins[3]):
        cf.map[dst] = fr.get(src)
    body = _lift_block(program, ccode, 0, len(ccode) - 1, cf, region)
    for dst, r in zip(ins[1], ccode[-1][1]):
        fr.map[dst] = cf.get(r)
    return [Ins(CALL)] + body + [Ins(RETURN)]


def _leaf(ins, fr, region):
    op = ins[0]
    n = Ins(op)
    if op == CONST:
        n.dst = fr.define(ins[1])
        n.value = ins[2]
        region.kind[n.dst] = "float" if isinstance(ins[2], float) else "int"
    elif op == BINF:
        n.a, n.b = fr.get(ins[3]), fr.get(ins[4])
        n.dst = fr.define(ins[1])
        n.sub = ins[2]
        n.f32 = bool(ins[5])
        region.kind[n.dst] = "f32" if n.f32 else "f64"
    elif op == BINI:
        n.a, n.b = fr.get(ins[3]), fr.get(ins[4])
        n.dst = fr.define(ins[1])
        n.sub = ins[2]
        n.f32 = ins[5] == "i32"      # reused as the i32-wrap flag
        region.kind[n.dst] = "int"
    elif op in (CMPF, CMPI):
        n.a, n.b = fr.get(ins[3]), fr.get(ins[4])
        n.dst = fr.define(ins[1])
        n.sub = ins[2]
        region.kind[n.dst] = "int"
    elif op == CAST:
        n.a = fr.get(ins[2])
        n.dst = fr.define(ins[1])
        n.f32 = ins[3] == "i32"
        region.kind[n.dst] = "int"
    elif op == LOAD:
        n.b = fr.get(ins[2])
        n.idx = tuple(fr.get(r) for r in ins[3])
        n.dst = fr.define(ins[1])
        n.loc = ins[4]
        region.kind[n.dst] = "data"
    elif op == STORE:
        n.a = fr.get(ins[1])
        n.b = fr.get(ins[2])
        n.idx = tuple(fr.get(r) for r in ins[3])
        n.loc = ins[4]
    elif op == ALLOC:
        # memref.alloc inside a loop: a fresh zero-filled Buffer every time it
        # executes (reference _evalpy.py:209-210).  It becomes a region
        # scratch buffer that the VM zero-fills at this instruction; the
        # engine runs such regions on one thread (no band), so one scratch
        # buffer is exactly the reference's sequence of fresh buffers.
        from staircase.interp.buffer import Buffer

        region.has_alloc = True
        buf = Buffer(ins[2], ins[3])
        n.dst = fr.define(ins[1])
        n.value = buf
        region.env[n.dst] = buf
        region.kind[n.dst] = "buf"
        region.buf_slot[id(buf)] = len(region.buffers)
        region.buffers.append(buf)
    elif op == DEALLOC:
        n.a = fr.get(ins[1])
    elif op == GPUID:
        gv = getattr(fr, "gpu_vars", None)
        if gv is None:
            raise Unsupported("gpu id outside a launch")
        n.dst = fr.define(ins[1])
        n.sub = ins[2] + (3 if ins[3] else 0)
        n.a = gv[n.sub].vreg
        region.kind[n.dst] = "int"
    elif op == RETURN_GPU:
        pass
    else:
        raise Unsupported(f"opcode {op} inside a loop region")
    return n


# -- symbolic evaluation ----------------------------------------------------------


def evaluate(region):
    """Fill ``region.sym`` (vreg -> Aff | float | None) and var domains."""
    sym = region.sym
    for v, val in region.env.items():
        k = region.kind[v]
        if k == "int":
            sym[v] = Aff(int(val))
        elif k == "float":
            sym[v] = float(val)
        else:
            sym[v] = None
    for var in region.vars:
        sym[var.vreg] = Aff.var(var.id)
    _eval_block(region.tree, region)


def _aff(region, v):
    s = region.sym.get(v)
    return s if isinstance(s, Aff) else None


def _eval_block(nodes, region):
    sym = region.sym
    for n in nodes:
        if isinstance(n, Ins):
            op = n.op
            if op == CONST:
                sym[n.dst] = n.value if isinstance(n.value, float) else Aff(int(n.value))
            elif op == BINI:
                a, b = _aff(region, n.a), _aff(region, n.b)
                r = None
                if a is not None and b is not None and not n.f32:
                    if n.sub == 0:
                        r = a + b
                    elif n.sub == 1:
                        r = a - b
                    elif a.is_const():
                        r = b.scale(a.c)
                    elif b.is_const():
                        r = a.scale(b.c)
                sym[n.dst] = r
            elif op == CAST:
                sym[n.dst] = None if n.f32 else _aff(region, n.a)
            elif op == GPUID:
                sym[n.dst] = Aff.var(region.var_of_vreg[n.a].id)
            elif n.dst is not None:
                sym[n.dst] = None
        elif isinstance(n, Loop):
            var = n.var
            if n.scf:
                var.lb, var.ub, var.step = (_aff(region, n.lb), _aff(region, n.ub),
                                            _aff(region, n.step))
            else:
                var.lb, var.ub, var.step = Aff(n.lb), Aff(n.ub), Aff(n.step)
            if var.lb is None or var.ub is None or var.step is None:
                var.lb = var.ub = var.step = None
            _eval_block(n.body, region)
        elif isinstance(n, Par):
            for var, lb, ub, st in zip(n.vars, n.lbs, n.ubs, n.steps):
                var.lb, var.ub, var.step = _aff(region, lb), _aff(region, ub), _aff(region, st)
                if var.lb is None or var.ub is None or var.step is None:
                    var.lb = var.ub = var.step = None
            _eval_block(n.body, region)
        elif isinstance(n, Launch):
            for d, var in enumerate(n.vars):
                ext = _aff(region, (n.grid + n.block)[d])
                var.lb, var.ub, var.step = Aff(0), ext, Aff(1)
                if ext is None:
                    var.lb = var.ub = var.step = None
            _eval_block(n.body, region)
        elif isinstance(n, If):
            _eval_block(n.then, region)
            _eval_block(n.els, region)


# -- intervals ----------------------------------------------------------------------


def var_range(region, var, memo=None):
    """Inclusive [lo, hi] of an iteration variable's values, or None."""
    if memo is None:
        memo = {}
    if var.id in memo:
        return memo[var.id]
    memo[var.id] = None   # cycle guard
    if var.lb is None:
        return None
    lb = aff_range(region, var.lb, memo)
    ub = aff_range(region, var.ub, memo)
    st = aff_range(region, var.step, memo)
    if lb is None or ub is None or st is None or st[0] <= 0:
        return None
    lo = lb[0]
    hi = ub[1] - 1
    if var.step.is_const() and var.lb.is_const() and var.ub.is_const():
        trip = max(0, -(-(var.ub.c - var.lb.c) // var.step.c))
        hi = var.lb.c + (trip - 1) * var.step.c
    r = (lo, hi) if hi >= lo else EMPTY
    memo[var.id] = r
    return r


EMPTY = (1, 0)   # an empty inclusive range: the access never executes


def aff_range(region, aff, memo=None):
    """Inclusive [lo, hi] of an affine form over its vars' domains.

    Returns None when a domain is unknown and EMPTY when some domain is
    empty (the access is never executed).
    """
    lo = hi = aff.c
    for vid, c in aff.t.items():
        r = var_range(region, region.vars[vid], memo)
        if r is None:
            return None
        if r[1] < r[0]:
            return EMPTY
        if c > 0:
            lo += c * r[0]
            hi += c * r[1]
        else:
            lo += c * r[1]
            hi += c * r[0]
    return lo, hi


def walk(nodes):
    """Yield (node, enclosing_vars) for every node, pre-order."""
    stack = [(nodes, ())]
    while stack:
        seq, encl = stack.pop()
        for n in seq:
            yield n, encl
            if isinstance(n, Loop):
                stack.append((n.body, encl + (n.var,)))
            elif isinstance(n, (Par, Launch)):
                stack.append((n.body, encl + tuple(n.vars)))
            elif isinstance(n, If):
                stack.append((n.then, encl))
                stack.append((n.els, encl))


def prod(xs):
    return math.prod(xs)
