"""TEST INFRASTRUCTURE — the CPU oracle for the B200 backend.

This package is the parity checker.  It is imported only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg, never by
the product package ``paper_2307_16080_b200``.

``oracle`` is itself a staircase *engine*: it exposes ``ExecContext`` and
``run_tape`` exactly like the reference's ``_evalpy`` / ``_evalcy``
(``staircase/interp/machine.py:105-112``), so a test can run the same
captured module through ``staircase.interp.machine.run(..., engine=oracle)``
and compare buffers and the tally with the B200 engine.  The arithmetic is
done by ``tape_eval.c`` (a plain-C restatement of
``staircase/interp/_evalpy.py:81-331``, compiled with -ffp-contract=off).

Parity of the oracle itself is pinned by ``tests/test_oracle.py`` against
the golden fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the unmodified reference executor.
"""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile tape_eval.c into liboracle.so (gcc, -ffp-contract=off)."""
    import subprocess

    src = os.path.join(_HERE, "tape_eval.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared",
             "-fPIC", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.orc_run.restype = ctypes.c_int
        lib.orc_free_table.restype = None
        _lib = lib
    return _lib


class OrcBuf(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int64),
                ("rank", ctypes.c_int64), ("shape", ctypes.c_int64 * 8),
                ("strides", ctypes.c_int64 * 8)]


_DT = {"f32": 0, "f64": 1, "i32": 2, "i64": 3}
_DT_NAME = {v: k for k, v in _DT.items()}
_NP = {0: np.float32, 1: np.float64, 2: np.int32, 3: np.int64}


def _bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


class _Encoder:
    """Flattens a TapeProgram (funcs, parallel sub-tapes, kernels)."""

    def __init__(self, program):
        self.program = program
        self.tapes = []          # list of (code, n_regs, arg_regs)
        self.ids = {}            # id(code tuple) -> tape index
        self.keep = []
        self.func_ids = {}
        self.locs = []
        self.loc_ids = {}
        for name, ft in program.funcs.items():
            self.func_ids[name] = self._tape(ft.code, ft.n_regs, ft.arg_regs)

    def _tape(self, code, n_regs, arg_regs) -> int:
        key = id(code)
        if key in self.ids:
            return self.ids[key]
        idx = len(self.tapes)
        self.ids[key] = idx
        self.keep.append(code)
        self.tapes.append((code, n_regs, tuple(arg_regs)))
        return idx

    def _loc(self, loc) -> int:
        if loc is None:
            return -1
        k = id(loc)
        if k not in self.loc_ids:
            self.loc_ids[k] = len(self.locs)
            self.locs.append(loc)
        return self.loc_ids[k]

    def encode(self):
        words = []
        ins_off = []
        info = []
        t = 0
        # tapes may be appended while encoding (sub-tapes): loop by index
        while t < len(self.tapes):
            code, n_regs, arg_regs = self.tapes[t]
            first = len(ins_off)
            for ins in code:
                ins_off.append(len(words))
                words.extend(self._ins(ins))
            arg_off = len(words)
            words.extend(arg_regs)
            info.extend([first, len(code), n_regs, arg_off])
            t += 1
        return (np.asarray(words, dtype=np.int64),
                np.asarray(info, dtype=np.int64),
                np.asarray(ins_off, dtype=np.int64))

    def _ins(self, ins):
        op = ins[0]
        if op == 0:
            v = ins[2]
            if isinstance(v, float):
                return [0, ins[1], 1, _bits(v)]
            return [0, ins[1], 0, int(v)]
        if op in (1,):
            return [1, ins[1], ins[2], ins[3], ins[4], int(bool(ins[5]))]
        if op == 2:
            return [2, ins[1], ins[2], ins[3], ins[4], int(ins[5] == "i32")]
        if op in (3, 4):
            return [op, ins[1], ins[2], ins[3], ins[4]]
        if op == 5:
            return [5, ins[1], ins[2], int(ins[3] == "i32")]
        if op in (6, 7):
            idx = list(ins[3])
            return [op, ins[1], ins[2], len(idx), *idx, self._loc(ins[4])]
        if op == 8:
            shape = list(ins[2])
            return [8, ins[1], _DT[ins[3]], len(shape), *shape]
        if op == 9:
            return [9, ins[1]]
        if op in (10, 11):
            return [op, ins[1], ins[2]]
        if op in (12, 13, 14, 15):
            return [op, ins[1], ins[2], ins[3]]
        if op == 16:
            return [16, ins[1]]
        if op == 17:
            return [17, ins[1], ins[2]]
        if op == 18:
            sub = ins[1]
            sid = self._tape(sub.code, sub.n_regs, ())
            nd = len(ins[2])
            caps = [r for pair in sub.captures for r in pair]
            return [18, sid, nd, *ins[2], *ins[3], *ins[4],
                    len(sub.captures), *caps, *sub.index_regs]
        if op == 19:
            callee = self.func_ids[ins[2]]
            return [19, callee, len(ins[3]), *ins[3], len(ins[1]), *ins[1]]
        if op in (20, 23):
            return [op, len(ins[1]), *ins[1]]
        if op == 21:
            kern = self.func_ids[ins[1]]
            return [21, kern, *ins[2], *ins[3], len(ins[4]), *ins[4],
                    self._loc(ins[5])]
        if op == 22:
            return [22, ins[1], ins[2], int(bool(ins[3]))]
        raise ValueError(f"oracle cannot encode opcode {op}")


class ExecContext:
    """Same fields as the reference's ExecContext (_evalpy.py:61-71)."""

    __slots__ = ("mode", "workers", "recorder", "gpu_ids", "depth")

    def __init__(self, mode="sequential", workers=1, recorder=None):
        self.mode = mode
        self.workers = workers
        self.recorder = recorder
        self.gpu_ids = None
        self.depth = 0


def _errors():
    import importlib

    return importlib.import_module("staircase.errors")


def run_tape(program, code, regs, tally, ctx):
    """Engine-protocol entry (machine.py:112) backed by tape_eval.c."""
    lib = _load()
    from staircase.interp.buffer import Buffer

    enc = _Encoder(program)
    entry = enc.ids.get(id(code))
    ftape = None
    for ft in program.funcs.values():
        if ft.code is code:
            ftape = ft
    if entry is None:
        entry = enc._tape(code, len(regs), ())
    words, info, ins_off = enc.encode()

    # buffer table: every Buffer in the seeded register file
    table = []
    buf_ids = {}
    keep = []
    slots = (ctypes.c_int64 * max(1, len(regs)))()
    fslots = ctypes.cast(slots, ctypes.POINTER(ctypes.c_double))
    for r, v in enumerate(regs):
        if v is None:
            continue
        if isinstance(v, Buffer):
            if id(v) not in buf_ids:
                buf_ids[id(v)] = len(table)
                table.append(v)
            slots[r] = buf_ids[id(v)]
        elif isinstance(v, float):
            fslots[r] = v
        else:
            slots[r] = int(v)
    n_bufs = len(table)
    ctable = (OrcBuf * max(1, n_bufs))()
    for k, b in enumerate(table):
        addr, _ = b.data.buffer_info()
        ctable[k].data = addr
        ctable[k].dtype = _DT[b.dtype]
        ctable[k].rank = len(b.shape)
        for d, (s, st) in enumerate(zip(b.shape, b.strides)):
            ctable[k].shape[d] = s
            ctable[k].strides[d] = st
        keep.append(b.data)

    rets = (ctypes.c_int64 * 16)()
    n_rets = ctypes.c_int64(0)
    ctally = (ctypes.c_int64 * len(tally))()
    status = (ctypes.c_int64 * 5)()
    out_table = ctypes.POINTER(OrcBuf)()
    out_n = ctypes.c_int64(0)
    p64 = ctypes.POINTER(ctypes.c_int64)
    lib.orc_run(words.ctypes.data_as(p64), info.ctypes.data_as(p64),
                ins_off.ctypes.data_as(p64), ctypes.c_int64(entry),
                ctable, ctypes.c_int64(n_bufs), slots, rets,
                ctypes.byref(n_rets), ctally,
                ctypes.c_int64(1 if ctx.mode == "gpu_emulated" else 0),
                status, ctypes.byref(out_table), ctypes.byref(out_n))
    for i in range(len(tally)):
        tally[i] += ctally[i]

    all_bufs = list(table)
    for k in range(n_bufs, out_n.value):
        cb = out_table[k]
        shape = tuple(cb.shape[d] for d in range(cb.rank))
        n = int(np.prod(shape))
        arr = np.ctypeslib.as_array(
            ctypes.cast(cb.data, ctypes.POINTER(ctypes.c_byte)),
            shape=(n * np.dtype(_NP[cb.dtype]).itemsize,)).view(_NP[cb.dtype])
        all_bufs.append(Buffer(shape, _DT_NAME[cb.dtype], arr.tolist()))
    lib.orc_free_table(out_table, ctable, ctypes.c_int64(n_bufs), out_n)

    err = status[0]
    if err:
        errors = _errors()
        if err == 1:
            idx, extent, bufno, loc = status[1], status[2], status[3], status[4]
            loc = enc.locs[loc] if loc >= 0 else None
            where = f" at {loc.file}:{loc.line}" if loc else ""
            raise errors.OutOfBounds(
                f"index {idx} out of bounds for extent {extent} of "
                f"{all_bufs[bufno]!r}{where}")
        if err == 2:
            raise errors.InvalidBound("loop step must be positive at runtime")
        if err == 3:
            loc = status[4]
            loc = enc.locs[loc] if loc >= 0 else None
            where = f" at {loc.file}:{loc.line}" if loc else ""
            raise errors.ModeUnsupported(
                f"gpu.launch_func needs gpu_emulated mode, not "
                f"{ctx.mode!r}{where}")
        raise RuntimeError(f"oracle failed with status {err}")
    if n_rets.value < 0:
        return None
    kinds = [t.kind for t in ftape.result_types] if ftape is not None else []
    out = []
    rets_f = ctypes.cast(rets, ctypes.POINTER(ctypes.c_double))
    for k in range(n_rets.value):
        kind = kinds[k] if k < len(kinds) else "index"
        if kind in ("f32", "f64"):
            out.append(rets_f[k])
        elif kind == "memref":
            out.append(all_bufs[rets[k]])
        else:
            out.append(int(rets[k]))
    return tuple(out)


__all__ = ["ExecContext", "run_tape", "build"]
