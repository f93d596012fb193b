"""Per-region plan cache: repeated runs skip lifting, analysis and matching.

staircase's run() verifies and compiles the module on every call
(reference interp/machine.py:94-115) and hands the engine a new tape each
time, so the engine would lift (lift.py), analyse (analysis.py) and match
(templates.py) every region again — host work that dominates small runs
(the Linear(32,32) lowering: ~0.5 ms per run for 66 kFLOP).  A region's plan
depends only on

* the region's instructions (and those of any callee / launched kernel),
* the values of the scalar registers it reads from outside (loop bounds,
  constants passed as arguments), bit for bit,
* the geometry of the Buffers it reads (shape, strides, dtype) and which of
  them are the same Buffer (aliasing),
* the engine settings (precision, fusion, shadows) and the run mode,

never on buffer contents.  The key is exactly that; a hit rebinds the cached
plan — a ContractMatch / MapMatch template or a VM program — to this run's
Buffers and scalars.  Sharded runs (shard.py) and race checks (races.py) are
not cached.  B200_PLAN_CACHE=0 disables the cache.
"""
from __future__ import annotations

import struct
from collections import OrderedDict

from .lift import CALL, LAUNCH, PARALLEL

MAX_PLANS = 512
_PLANS = OrderedDict()    # (region key, env key) -> (Plan, Shell)
_OUTER = {}               # region key -> outer registers the region reads
STATS = {"hits": 0, "misses": 0}


class Plan:
    """A region's execution decision, independent of the Buffers it binds."""

    __slots__ = ("kind", "st", "written", "item", "chain", "entry", "checked", "slots")

    def __init__(self, kind, st, written, item, chain=None, entry=None, checked=False):
        self.kind = kind          # "contract" | "map" | "vm"
        self.st = st              # static tally (or None: counted on the device)
        self.written = sorted(written)   # buffer slots the region writes
        self.item = item          # ContractMatch | MapMatch | VMProgram
        self.chain = chain        # chain tally of a counting VM program
        self.entry = entry        # engine.last_plan entry of a VM plan
        self.checked = checked
        self.slots = None         # operand buffer slots of item (put())


class _Bound:
    """What execution needs of a lifted region, bound to one run."""

    __slots__ = ("buffers", "env", "kind", "buf_slot")


class Shell:
    """Where a region's Buffers and scalars come from: outer registers, or
    the region's own scratch buffers (memref.alloc inside the region)."""

    __slots__ = ("slot_src", "env_src", "kind")

    def __init__(self, r):
        reg_of = {}
        for reg, v in r.outer:
            reg_of[v] = reg
        by_buf = {}
        for reg, v in r.outer:
            if r.kind.get(v) == "buf":
                by_buf.setdefault(id(r.env[v]), reg)
        self.slot_src = [("reg", by_buf[id(b)]) if id(b) in by_buf else ("own", b)
                         for b in r.buffers]
        self.env_src = {v: ("reg", reg_of[v]) if v in reg_of else ("own", val)
                        for v, val in r.env.items()}
        self.kind = dict(r.kind)


def bind(shell, regs):
    b = _Bound()
    b.buffers = [regs[x] if how == "reg" else x for how, x in shell.slot_src]
    b.env = {v: regs[x] if how == "reg" else x for v, (how, x) in shell.env_src.items()}
    b.kind = shell.kind
    b.buf_slot = {id(buf): k for k, buf in enumerate(b.buffers)}
    return b


# -- keys -----------------------------------------------------------------------

def _fp(code):
    """A hashable fingerprint of a tape slice (SubTape bodies inlined)."""
    try:
        hash(code)
        return code
    except TypeError:
        pass
    out = []
    for ins in code:
        if ins[0] == PARALLEL:
            sub = ins[1]
            out.append((PARALLEL, (_fp(sub.code), sub.n_regs, tuple(sub.index_regs),
                                   tuple(sub.captures))) + tuple(ins[2:]))
        else:
            out.append(ins)
    return tuple(out)


def _callees(program, code, seen):
    for ins in code:
        if ins[0] in (CALL, LAUNCH):
            name = ins[2] if ins[0] == CALL else ins[1]
            if name not in seen:
                seen[name] = None
                f = program.funcs[name]
                seen[name] = (_fp(f.code), f.n_regs, tuple(f.arg_regs))
                _callees(program, f.code, seen)
        elif ins[0] == PARALLEL:
            _callees(program, ins[1].code, seen)


def region_key(program, code, start, end):
    body = code[start:end]
    seen = {}
    _callees(program, body, seen)
    return (_fp(body), tuple(sorted(seen.items())))


def _env(regs, outer):
    out = []
    first = {}
    for k, reg in enumerate(outer):
        v = regs[reg]
        if isinstance(v, float):
            out.append(("f", struct.pack("<d", v)))
        elif isinstance(v, (bool, int)):
            out.append(("i", int(v), isinstance(v, bool)))
        elif hasattr(v, "shape") and hasattr(v, "strides"):
            alias = first.setdefault(id(v), k)
            out.append(("b", tuple(v.shape), tuple(v.strides), v.dtype, alias))
        else:
            return None
    return tuple(out)


def lookup_key(rkey, regs):
    outer = _OUTER.get(rkey)
    if outer is None:
        return None
    env = _env(regs, outer)
    return None if env is None else (rkey, env)


def get(key):
    if key is None:
        return None
    hit = _PLANS.get(key)
    if hit is None:
        STATS["misses"] += 1
        return None
    _PLANS.move_to_end(key)
    STATS["hits"] += 1
    return hit


def put(rkey, regs, r, plan):
    outer = tuple(reg for reg, _ in r.outer)
    env = _env(regs, outer)
    if env is None:
        return
    _OUTER[rkey] = outer
    slot = {id(b): k for k, b in enumerate(r.buffers)}
    if plan.kind == "contract":
        g = plan.item
        plan.slots = (slot[id(g.A)], slot[id(g.B)], slot[id(g.C)])
    elif plan.kind == "map":
        plan.slots = [slot[id(b)] for b in plan.item.buffers]
    _PLANS[(rkey, env)] = (plan, Shell(r))
    while len(_PLANS) > MAX_PLANS:
        _PLANS.popitem(last=False)


def clear():
    _PLANS.clear()
    _OUTER.clear()


# -- rebinding ----------------------------------------------------------------------

def _clone(obj):
    new = object.__new__(type(obj))
    for k in type(obj).__slots__:
        if hasattr(obj, k):
            setattr(new, k, getattr(obj, k))
    return new


def rebind_contract(g0, r, slots=None):
    g = _clone(g0)
    a, b, c = slots
    g.A, g.B, g.C = r.buffers[a], r.buffers[b], r.buffers[c]
    return g


def rebind_map(m0, r, slots=None):
    m = _clone(m0)
    m.buffers = [r.buffers[k] for k in slots]
    return m


__all__ = ["Plan", "region_key", "lookup_key", "get", "put", "bind", "clear", "STATS"]
