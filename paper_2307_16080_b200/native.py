"""Native execution of device-VM programs: the VM word stream specialised to CUDA C.

The device tape VM (csrc/vm.cu) is the generic tier: any lifted region runs
there exactly like the reference's ``run_tape`` (interp/_evalpy.py:81-331),
one band point per thread, but every instruction pays a dispatch.  This
module turns a region's VM program (vmcode.encode) into a
straight CUDA C kernel, compiled once per program by NVRTC (csrc/jit.cu):

* every VM instruction becomes the statement the VM would execute for it,
  with the same helpers and the same rounding (``__f*_rn`` / ``__d*_rn``,
  floats held as doubles, i32 wrap) — so results, tally counts and faults
  are the VM's, instruction for instruction;
* register numbers, opcodes, flags, buffer ranks / strides / dtypes, band
  geometry and program constants are compile-time constants, so the
  dispatch switch, the register array and the generic indexing disappear
  (registers become scalars; jumps become gotos; loops with constant
  bounds are visible to the optimiser);
* values that change between runs — buffer base pointers and host scalars
  (region environment) — are kernel arguments, so the same nest shape with
  new data reuses the compiled kernel.

B200_NATIVE=0 keeps the interpreter (for A/B comparisons).
"""
from __future__ import annotations

import ctypes
import math
import os

from . import jit
from .vmcode import (V_BINF, V_BINI, V_CAST, V_CMPF, V_CMPI, V_CONST, V_END, V_IFF,
                     V_JUMP, V_LOAD, V_MOV, V_NEXT, V_NOP, V_PCHECK, V_STORE, V_TEST,
                     V_ZERO)

ENABLED = os.environ.get("B200_NATIVE", "1") != "0"
KTALLY = 25
THREADS = 128

_FOPS = ["__fadd_rn", "__fsub_rn", "__fmul_rn", "__fdiv_rn"]
_DOPS = ["__dadd_rn", "__dsub_rn", "__dmul_rn", "__ddiv_rn"]
_CTYPE = {0: "float", 1: "double", 2: "int", 3: "long long"}

_PRELUDE = r"""
typedef unsigned long long u64;
typedef long long i64;
struct VmErr { int code; int slot; i64 index; i64 extent; i64 loc; };
__device__ __forceinline__ double AF(u64 v) { return __longlong_as_double((i64)v); }
__device__ __forceinline__ u64 FA(double d) { return (u64)__double_as_longlong(d); }
__device__ __forceinline__ u64 W32(u64 v) { return (u64)(i64)(int)(unsigned)v; }
__device__ __forceinline__ void report(VmErr *e, int code, int slot, i64 idx, i64 ext,
                                       i64 loc) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->slot = slot; e->index = idx; e->extent = ext; e->loc = loc;
  }
}
"""


def available():
    return ENABLED and jit.available()


def _u64(lo, hi):
    return ((hi & 0xFFFFFFFF) << 32) | (lo & 0xFFFFFFFF)


def _decode(words):
    """(pc, op, tag, flags, operands) for every instruction of the stream."""
    out = []
    pc = 0
    n = len(words)
    while pc < n:
        w = words[pc] & 0xFFFFFFFF
        op, tag, fl = w & 0xFF, ((w >> 8) & 0xFF) - 1, (w >> 16) & 0xFFFF
        if op == V_END or op == V_NOP:
            size = 1
        elif op in (V_CONST, V_BINF, V_BINI, V_CMPF, V_CMPI, V_TEST, V_NEXT):
            size = 4
        elif op in (V_CAST, V_MOV, V_IFF):
            size = 3
        elif op in (V_LOAD, V_STORE):
            size = 4 + (fl & 15)
        elif op == V_JUMP:
            size = 2
        elif op == V_PCHECK:
            size = 1 + fl
        elif op == V_ZERO:
            size = 3
        else:
            raise ValueError(f"unknown VM opcode {op} at {pc}")
        out.append((pc, op, tag, fl, words[pc + 1:pc + size]))
        pc += size
    return out


_RECORD = r"""
// race recorder (races.py): per buffer element, the first writing point W,
// the first reading point R1 and the first reading point other than R1, R2
// (INT64_MAX = none); pass 0 fills W / R1, pass 1 R2, pass 2 emits the
// reference recorder's conflicts (interp/races.py:52-76) as events
// (point, sequence, kind, other point, slot, offset)
__device__ __forceinline__ void emit_ev(i64 *EV, u64 *NEV, i64 cap, i64 q, i64 seq, i64 kind,
                                        i64 other, i64 slot, i64 off) {
  const u64 k = atomicAdd(NEV, 1ULL);
  if ((i64)k < cap) {
    i64 *e = EV + 6 * k;
    e[0] = q; e[1] = seq; e[2] = kind; e[3] = other; e[4] = slot; e[5] = off;
  }
}
__device__ __forceinline__ void rec(int pass, int slot, i64 off, int wr, i64 q, i64 seq,
                                    i64 *const *SH, i64 *EV, u64 *NEV, i64 cap) {
  i64 *W = SH[3 * slot], *R1 = SH[3 * slot + 1], *R2 = SH[3 * slot + 2];
  if (pass == 0) {
    if (wr) atomicMin((long long *)&W[off], (long long)q);
    else atomicMin((long long *)&R1[off], (long long)q);
    return;
  }
  if (pass == 1) {
    if (!wr && R1[off] != q) atomicMin((long long *)&R2[off], (long long)q);
    return;
  }
  const i64 w = W[off];
  if (w < q) emit_ev(EV, NEV, cap, q, seq, 0, w, slot, off);
  if (wr) {
    const i64 r1 = R1[off], r2 = R2[off];
    if (r1 < q) emit_ev(EV, NEV, cap, q, seq, 1, r1, slot, off);
    if (r2 < q) emit_ev(EV, NEV, cap, q, seq, 2, r2, slot, off);
  }
}
"""


def vm_source(prog, buffers, env_regs, record=False):
    """CUDA C for a VMProgram over ``buffers`` (slot order).

    ``env_regs``: the init registers holding host values (loaded from the
    kernel's ``env`` argument, in prog.init_regs order); every other init
    register is a program constant and is embedded.  Returns (source,
    kernel name, env list of (reg, index into init_vals)).

    ``record``: the race recorder variant (races.py): loads and stores only
    report their addresses to ``rec`` (point = the band index, in
    row-major order) — valid for programs whose addresses and control flow
    do not depend on loaded data, which races.py checks.
    """
    count = prog.count and not record
    name = "b200_vm_record" if record else "b200_vm_native"
    used = set()
    insts = _decode(prog.words)
    for _, op, _, fl, a in insts:
        if op in (V_CONST, V_BINF, V_BINI, V_CMPF, V_CMPI, V_CAST, V_MOV):
            used.update(a[:1] if op == V_CONST else a[:3] if op != V_CAST and op != V_MOV
                        else a[:2])
        elif op in (V_LOAD, V_STORE):
            used.add(a[0])
            used.update(a[2:2 + (fl & 15)])
        elif op in (V_TEST, V_NEXT):
            used.update(a[:2])
        elif op == V_IFF:
            used.add(a[0])
        elif op == V_PCHECK:
            used.update(a[:fl])
    used.update(b[0] for b in prog.band)
    targets = set()
    for pc, op, _, _, a in insts:
        if op in (V_TEST, V_NEXT):
            targets.add(a[2])
        elif op == V_JUMP:
            targets.add(a[0])
        elif op == V_IFF:
            targets.add(a[1])
    consts, env = [], []
    envset = set(env_regs)
    for k, (reg, val) in enumerate(zip(prog.init_regs, prog.init_vals)):
        if reg in envset:
            env.append((reg, k))
        else:
            consts.append((reg, val))
    # Constants that reach a float operation are read from a __constant__
    # table instead of embedded: ptxas folds an f32 sub.rn of two immediates
    # without round-to-nearest-even at an exact tie (measured: 0x3f065226 -
    # 0x4027a8c1 folded to 0xc0061437, the hardware FADD gives 0xc0061438),
    # and the reference rounds every operation at run time.  The table is
    # mutable module memory, so nothing can fold through it.  Integer
    # constants (bounds, strides) stay literal for the optimiser.
    fregs = set()
    for _, op, _, _, a in insts:
        if op == V_BINF:
            fregs.update(a[1:3])
    grew = True
    while grew:   # through register copies
        grew = False
        for _, op, _, _, a in insts:
            if op == V_MOV and a[0] in fregs and a[1] not in fregs:
                fregs.add(a[1])
                grew = True
    table = []

    def kslot(val):
        table.append(val & 0xFFFFFFFFFFFFFFFF)
        return len(table) - 1

    if record:
        L = [_PRELUDE, _RECORD,
             f'extern "C" __global__ void __launch_bounds__({THREADS}) {name}(',
             "    void *const *__restrict__ P, const i64 *__restrict__ ENV, i64 *const *SH,"
             " i64 *EV, u64 *NEV, const i64 CAP, const int PASS, VmErr *__restrict__ ERR) {"]
    else:
        L = [_PRELUDE, f'extern "C" __global__ void __launch_bounds__({THREADS}) {name}(',
             "    void *const *__restrict__ P, const i64 *__restrict__ ENV, u64 *__restrict__ TALLY,"
             " VmErr *__restrict__ ERR) {"]
    regs = sorted(used | {r for r, _ in consts} | {r for r, _ in env})
    L.append("  u64 " + ", ".join(f"R{r} = 0" for r in regs) + ";" if regs else "")
    if count:
        L.append("  u64 " + ", ".join(f"c{i} = 0" for i in range(KTALLY)) + ";")
    for reg, k in env:
        L.append(f"  const u64 E{reg} = (u64)ENV[{k}];")
    total = math.prod(b[3] for b in prog.band) if prog.band else 1
    L.append(f"  for (i64 pt = (i64)blockIdx.x * {THREADS} + threadIdx.x; pt < {total}LL;"
             f" pt += (i64)gridDim.x * {THREADS}) {{")
    if record:
        L.append("    i64 seq = 0;")
    for reg, val in consts:
        if reg in fregs:
            L.append(f"    R{reg} = KC[{kslot(val)}];")
        else:
            L.append(f"    R{reg} = 0x{val & 0xFFFFFFFFFFFFFFFF:x}ULL;")
    for reg, _ in env:
        L.append(f"    R{reg} = E{reg};")
    if prog.band:
        L.append("    i64 rem = pt;")
        for (reg, lb, st, trip) in reversed(prog.band):
            L.append(f"    R{reg} = (u64)({lb}LL + {st}LL * (rem % {trip}LL)); rem /= {trip}LL;")
    for pc, op, tag, fl, a in insts:
        line = []
        if pc in targets:
            line.append(f"L{pc}:;")
        if count and tag >= 0:
            line.append(f"c{tag}++;")
        if op == V_CONST and a[0] in fregs:
            line.append(f"R{a[0]} = KC[{kslot(_u64(a[1], a[2]))}];")
        else:
            line.append(_stmt(pc, op, fl, a, buffers, count, record))
        L.append("    " + " ".join(line))
    L.append("  next_point:;")
    L.append("  }")
    L.append("fault:;")
    if count:
        L.append("  {")
        L.append("    const unsigned lane = threadIdx.x & 31;")
        for i in range(KTALLY):
            L.append(f"    {{ u64 v = c{i}; for (int o = 16; o > 0; o >>= 1) "
                     f"v += __shfl_down_sync(0xffffffffu, v, o); "
                     f"if (lane == 0 && v) atomicAdd(&TALLY[{i}], v); }}")
        L.append("  }")
    L.append("}")
    if table:
        at = next(i for i, x in enumerate(L) if x.startswith('extern "C" __global__'))
        L.insert(at, "__constant__ unsigned long long KC[%d] = {%s};" % (
            len(table), ", ".join(f"0x{v:x}ULL" for v in table)))
    return "\n".join(L) + "\n", name, env


def _stmt(pc, op, fl, a, buffers, count, record=False):
    if op == V_END:
        return "goto next_point;"
    if op == V_NOP:
        return ";"
    if op == V_CONST:
        return f"R{a[0]} = 0x{_u64(a[1], a[2]):x}ULL;"
    if op == V_BINF:
        f = fl & 3
        if fl & 4:
            return (f"R{a[0]} = FA((double){_FOPS[f]}((float)AF(R{a[1]}), "
                    f"(float)AF(R{a[2]})));")
        return f"R{a[0]} = FA({_DOPS[f]}(AF(R{a[1]}), AF(R{a[2]})));"
    if op == V_BINI:
        sym = "+-*"[fl & 3]
        e = f"(R{a[1]} {sym} R{a[2]})"
        return f"R{a[0]} = {'W32(' + e + ')' if fl & 4 else e};"
    if op == V_CMPF:
        x, y = f"AF(R{a[1]})", f"AF(R{a[2]})"
        c = fl & 7
        expr = {0: f"{x} == {y}", 1: f"({x} == {x}) && ({y} == {y}) && ({x} != {y})",
                2: f"{x} < {y}", 3: f"{x} <= {y}", 4: f"{x} > {y}"}.get(c, f"{x} >= {y}")
        return f"R{a[0]} = ({expr}) ? 1ULL : 0ULL;"
    if op == V_CMPI:
        x, y = f"(i64)R{a[1]}", f"(i64)R{a[2]}"
        sym = {0: "==", 1: "!=", 2: "<", 3: "<=", 4: ">"}.get(fl & 7, ">=")
        return f"R{a[0]} = ({x} {sym} {y}) ? 1ULL : 0ULL;"
    if op == V_CAST:
        return f"R{a[0]} = {'W32(R' + str(a[1]) + ')' if fl & 1 else 'R' + str(a[1])};"
    if op in (V_LOAD, V_STORE):
        rank, checked, dt = fl & 15, (fl >> 4) & 1, (fl >> 5) & 3
        reg, slot = a[0], a[1]
        idx = a[2:2 + rank]
        loc = a[2 + rank]
        buf = buffers[slot]
        parts = []
        terms = []
        for k, ir in enumerate(idx):
            if checked:
                parts.append(f"if ((i64)R{ir} < 0 || (i64)R{ir} >= {buf.shape[k]}LL) "
                             f"{{ report(ERR, 1, {slot}, (i64)R{ir}, {buf.shape[k]}LL, {loc}); "
                             f"goto fault; }}")
            terms.append(f"(i64)R{ir} * {buf.strides[k]}LL")
        off = " + ".join(terms) if terms else "0"
        if record:
            parts.append(f"rec(PASS, {slot}, {off}, {int(op == V_STORE)}, pt, seq++, SH, EV, NEV,"
                         f" CAP);")
            if op == V_LOAD:
                parts.append(f"R{reg} = 0;")
            return "{ " + " ".join(parts) + " }"
        T = _CTYPE[dt]
        p = f"(({T} *)P[{slot}])[{off}]"
        if op == V_LOAD:
            if dt == 0:
                v = f"FA((double){p})"
            elif dt == 1:
                v = f"FA({p})"
            else:
                v = f"(u64)(i64){p}"
            parts.append(f"R{reg} = {v};")
        else:
            if dt == 0:
                v = f"(float)AF(R{reg})"
            elif dt == 1:
                v = f"AF(R{reg})"
            elif dt == 2:
                v = f"(int)(unsigned)R{reg}"
            else:
                v = f"(i64)R{reg}"
            parts.append(f"{p} = {v};")
        return "{ " + " ".join(parts) + " }"
    if op == V_MOV:
        return f"R{a[0]} = R{a[1]};"
    if op == V_TEST:
        bk = "c24++; " if (count and fl & 1) else ""
        return f"if ((i64)R{a[0]} >= (i64)R{a[1]}) goto L{a[2]}; {bk}"
    if op == V_NEXT:
        chk = (f"if ((i64)R{a[1]} <= 0) {{ report(ERR, 2, -1, (i64)R{a[1]}, 0, -1); "
               f"goto fault; }} ") if fl & 1 else ""
        return f"{chk}R{a[0]} = (u64)((i64)R{a[0]} + (i64)R{a[1]}); goto L{a[2]};"
    if op == V_JUMP:
        return f"goto L{a[0]};"
    if op == V_IFF:
        return f"if (!R{a[0]}) goto L{a[1]};"
    if op == V_PCHECK:
        conds = " || ".join(f"(i64)R{r} <= 0" for r in a[:fl]) or "false"
        return f"if ({conds}) {{ report(ERR, 3, -1, 0, 0, -1); goto fault; }}"
    if op == V_ZERO:   # memref.alloc in the region: zero-fill its scratch buffer
        T = _CTYPE[fl & 3]
        return f"for (i64 z = 0; z < {a[1]}LL; ++z) (({T} *)P[{a[0]}])[z] = 0;"
    raise ValueError(f"unknown VM opcode {op}")


class NativeLaunch:
    """A compiled program plus the argument block of one launch (kept for replay)."""

    def __init__(self, fn, grid, ptr_table, env_vals, tally, err):
        self.fn = fn
        self.grid = grid
        self.vals = [ctypes.c_void_p(ptr_table), ctypes.c_void_p(env_vals),
                     ctypes.c_void_p(tally), ctypes.c_void_p(err)]
        self.argv = (ctypes.c_void_p * 4)(
            *[ctypes.cast(ctypes.byref(v), ctypes.c_void_p) for v in self.vals])


def grid_of(prog):
    total = math.prod(b[3] for b in prog.band) if prog.band else 1
    return max(1, min((total + THREADS - 1) // THREADS, 148 * 16))


__all__ = ["available", "vm_source", "NativeLaunch", "grid_of", "ENABLED"]
