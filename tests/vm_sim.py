"""CPU simulator of the device backend — TEST INFRASTRUCTURE ONLY.

Executes the exact artefacts the engine hands to libb200k.so (VM programs
from vmcode.py, GemmMatch descriptors from templates.py) with the device
kernels' semantics, so the whole host pipeline (lift → analysis → band →
encode → tally) is tested on CPU against the reference's golden fixtures
before any GPU time is spent.  The product never imports this module.
"""
import struct

import numpy as np

V_END, V_CONST, V_BINF, V_BINI, V_CMPF, V_CMPI, V_CAST, V_LOAD, V_STORE, V_MOV, \
    V_TEST, V_NEXT, V_JUMP, V_IFF, V_PCHECK, V_NOP, V_ZERO = range(17)

_NP = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}


def _f32(x):
    return float(np.float32(x))


def _wrap32(v):
    return ((int(v) + (1 << 31)) % (1 << 32)) - (1 << 31)


def _wrap64(v):
    return ((int(v) + (1 << 63)) % (1 << 64)) - (1 << 63)


def _bits_to_val(bits):
    return bits


class SimBackend:
    def __init__(self):
        self.dev = {}
        self.dirty = set()
        self.launches = []

    def arr(self, buf):
        ent = self.dev.get(id(buf))
        if ent is None:
            a = np.frombuffer(buf.data, dtype=_NP[buf.dtype]).copy()
            ent = (buf, a)
            self.dev[id(buf)] = ent
        return ent[1]

    def read(self, buf, off):
        v = self.arr(buf)[off]
        return float(v) if buf.dtype[0] == "f" else int(v)

    def write(self, buf, off, v):
        self.arr(buf)[off] = v
        self.dirty.add(id(buf))

    def mark_dirty(self, buf):
        self.dirty.add(id(buf))

    def flush(self):
        for k in list(self.dirty):
            if k not in self.dev:
                continue
            buf, a = self.dev[k]
            np.frombuffer(buf.data, dtype=_NP[buf.dtype])[:] = a
        self.dirty.clear()

    def contract(self, g, precision="exact", init=0, init_value=0.0, bias=None, bias_base=0,
                 bias_stride=0, shadow_out=False, shadow_in=False, last_writer=False):
        # bf16 shadows only exist on the tensor-core path, and host-copy
        # pipelining is a staging detail: nothing to model
        assert precision == "exact", "the simulator models the exact path only"
        self.launches.append("contract")
        A, B, C = self.arr(g.A), self.arr(g.B), self.arr(g.C)
        a_m, a_k, b_k, b_n, c_m, c_n = g.tables
        dt = np.float32 if g.dtype == "f32" else np.float64
        coff = c_m[:, None] + c_n[None, :]
        acc = np.full(coff.shape, init_value, dtype=dt) if init else C[coff].astype(dt)
        for k in range(g.K):
            a = A[a_m + a_k[k]].astype(dt)[:, None]
            b = B[b_k[k] + b_n].astype(dt)[None, :]
            acc = (acc + (a * b).astype(dt)).astype(dt)
        if bias is not None:
            bv = self.arr(bias)[bias_base + bias_stride * np.arange(g.N)].astype(dt)
            acc = (acc + bv[None, :]).astype(dt)
        C[coff] = acc
        return ["contract_exact"]

    def map(self, m, last_writer=False):
        """b200_map_f32 semantics: every box point runs the program in order."""
        self.launches.append(("map", m.kind, m.vector))
        arrs = [self.arr(b) for b in m.buffers]
        grids = np.meshgrid(*[np.arange(t) for t in m.trips], indexing="ij")
        offs = [base + sum(c * g.reshape(-1) for c, g in zip(coefs, grids))
                for base, coefs in zip(m.bases, m.coefs)]
        regs = {}
        pc = 0
        with np.errstate(all="ignore"):
            while pc < len(m.prog):
                w = m.prog[pc]
                op, dst, a, b = w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, (w >> 24) & 0xFF
                if op == 0:
                    regs[dst] = arrs[a][offs[a]].astype(np.float32)
                    pc += 1
                elif op == 1:
                    regs[dst] = np.float32(m.consts[a])
                    pc += 1
                elif op == 2:
                    f = m.prog[pc + 1]
                    x, y = np.float32(regs[a]), np.float32(regs[b])
                    regs[dst] = [x + y, x - y, x * y, x / y][f].astype(np.float32)
                    pc += 2
                else:
                    arrs[a][offs[a]] = regs[dst]
                    pc += 1
        return ["map_f32"]

    def vm(self, r, prog, checked):
        self.launches.append(("vm", len(prog.band), checked))
        bufs = [(self.arr(b), b) for b in r.buffers]
        w = prog.words
        cnt = [0] * 25
        init = dict(zip(prog.init_regs, prog.init_vals))
        trips = [b[3] for b in prog.band]
        total = 1
        for t in trips:
            total *= t
        for pt in range(total):
            R = {}
            for k, v in init.items():
                R[k] = v
            rem = pt
            for (reg, lb, st, trip) in reversed(prog.band):
                t = rem % trip
                rem //= trip
                R[reg] = lb + st * t
            fault = self._exec(w, R, bufs, cnt, prog.count)
            if fault is not None:
                return None, fault
        return (cnt if prog.count else None), None

    @staticmethod
    def _f(R, r):
        v = R[r]
        return struct.unpack("<d", struct.pack("<q", v))[0] if isinstance(v, int) and \
            not isinstance(v, bool) and _is_bits(v) else v

    def _exec(self, w, R, bufs, cnt, count):
        pc = 0

        def F(r):
            v = R[r]
            return v if isinstance(v, float) else struct.unpack("<d", struct.pack("<q", _wrap64(v)))[0]

        def I(r):
            v = R[r]
            return v if isinstance(v, int) else struct.unpack("<q", struct.pack("<d", v))[0]

        while True:
            word = w[pc]
            op = word & 0xFF
            tag = ((word >> 8) & 0xFF) - 1
            fl = (word >> 16) & 0xFFFF
            if count and tag >= 0:
                cnt[tag] += 1
            if op == V_END:
                return None
            if op == V_CONST:
                lo, hi = w[pc + 2] & 0xFFFFFFFF, w[pc + 3] & 0xFFFFFFFF
                R[w[pc + 1]] = _wrap64(lo | (hi << 32))
                pc += 4
            elif op == V_BINF:
                a, b = F(w[pc + 2]), F(w[pc + 3])
                f = fl & 3
                if fl & 4:
                    a32, b32 = np.float32(a), np.float32(b)
                    with np.errstate(all="ignore"):
                        r = [a32 + b32, a32 - b32, a32 * b32, a32 / b32][f]
                    r = float(np.float32(r))
                else:
                    with np.errstate(all="ignore"):
                        r = float([np.float64(a) + b, np.float64(a) - b, np.float64(a) * b,
                                   np.float64(a) / np.float64(b)][f])
                R[w[pc + 1]] = r
                pc += 4
            elif op == V_BINI:
                a, b = I(w[pc + 2]), I(w[pc + 3])
                f = fl & 3
                r = a + b if f == 0 else (a - b if f == 1 else a * b)
                R[w[pc + 1]] = _wrap32(r) if fl & 4 else _wrap64(r)
                pc += 4
            elif op == V_CMPF:
                a, b = F(w[pc + 2]), F(w[pc + 3])
                p = fl & 7
                r = [a == b, (a == a and b == b and a != b), a < b, a <= b, a > b, a >= b][p]
                R[w[pc + 1]] = int(r)
                pc += 4
            elif op == V_CMPI:
                a, b = I(w[pc + 2]), I(w[pc + 3])
                r = [a == b, a != b, a < b, a <= b, a > b, a >= b][fl & 7]
                R[w[pc + 1]] = int(r)
                pc += 4
            elif op == V_CAST:
                v = I(w[pc + 2])
                R[w[pc + 1]] = _wrap32(v) if fl & 1 else v
                pc += 3
            elif op in (V_LOAD, V_STORE):
                rank, checked = fl & 15, (fl >> 4) & 1
                slot = w[pc + 2]
                arr, buf = bufs[slot]
                off = 0
                for k in range(rank):
                    i = I(w[pc + 3 + k])
                    if checked and (i < 0 or i >= buf.shape[k]):
                        return (1, slot, i, buf.shape[k], w[pc + 3 + rank])
                    off += i * buf.strides[k]
                reg = w[pc + 1]
                if op == V_LOAD:
                    v = arr[off]
                    R[reg] = float(v) if buf.dtype[0] == "f" else int(v)
                else:
                    v = R[reg]
                    if buf.dtype[0] == "f":
                        arr[off] = F(reg)
                    elif buf.dtype == "i32":
                        arr[off] = _wrap32(I(reg))
                    else:
                        arr[off] = I(reg)
                pc += 4 + rank
            elif op == V_MOV:
                R[w[pc + 1]] = R[w[pc + 2]]
                pc += 3
            elif op == V_TEST:
                if I(w[pc + 1]) >= I(w[pc + 2]):
                    pc = w[pc + 3]
                else:
                    if count and (fl & 1):
                        cnt[24] += 1
                    pc += 4
            elif op == V_NEXT:
                step = I(w[pc + 2])
                if (fl & 1) and step <= 0:
                    return (2, -1, step, 0, -1)
                R[w[pc + 1]] = I(w[pc + 1]) + step
                pc = w[pc + 3]
            elif op == V_JUMP:
                pc = w[pc + 1]
            elif op == V_IFF:
                pc = pc + 3 if I(w[pc + 1]) else w[pc + 2]
            elif op == V_PCHECK:
                nd = fl
                for k in range(nd):
                    if I(w[pc + 1 + k]) <= 0:
                        return (3, -1, 0, 0, -1)
                pc += 1 + nd
            elif op == V_ZERO:
                bufs[w[pc + 1]][0][:w[pc + 2]] = 0
                pc += 3
            else:
                pc += 1


def _is_bits(v):
    return True


class SimEngine:
    """Engine-protocol object that runs the real engine on the simulator."""

    def __init__(self):
        from paper_2307_16080_b200 import engine

        self._engine = engine
        self.ExecContext = engine.ExecContext
        self.last = None

    def run_tape(self, program, code, regs, tally, ctx):
        be = SimBackend()
        self.last = be
        return self._engine.run_tape(program, code, regs, tally, ctx, backend=be)
