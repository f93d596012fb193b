"""The B200 engine: a drop-in for staircase's CPU tape evaluators.

Plug-in point (reference pkg/src/staircase/interp/machine.py:26-34,105-112):

    eng = engine or _engine
    ctx = eng.ExecContext(mode, workers)
    rets = eng.run_tape(program, tape.code, regs, tally, ctx)

This module provides ``ExecContext`` and ``run_tape`` with the same
signatures, ownership and error behaviour as ``_evalpy``/``_evalcy``
(interp/_evalpy.py:61-232): memref Buffers are mutated in place, ``tally``
is incremented exactly as the reference increments it, and faults raise
``staircase.errors`` types with the reference's messages.

Execution model: the top level of the entry tape is walked on the host —
that is only scalar bookkeeping (constants, index arithmetic, branches on
scalars, calls, returns) and single-element loads/stores.  Every loop nest,
``scf.parallel`` and ``gpu.launch_func`` found there is a *region*: it is
lifted (lift.py), analysed (analysis.py), matched against the kernel
templates (templates.py) and executed on the GPU, either by a specialised
kernel (contraction, pointwise map) or by the device tape VM (csrc/vm.cu).
Specialised plans are queued while only pure host scalar work separates
them and are fused across regions (fusion.py) before launch — e.g. the
Linear lowering's fill/copy/contraction/bias become one GEMM with an init
value and a bias epilogue.  Nothing in a region runs on the CPU; there is
no fallback.

Install globally (the tuner calls run() without engine=, search.py:170,190):

    import paper_2307_16080_b200 as b2
    b2.install()          # sets staircase.interp.machine._engine
"""
from __future__ import annotations

import contextlib
import math
import os
import threading

from . import analysis, fusion, plancache, templates, vmcode
from .host import errors as _errors
from .lift import (ALLOC, BINF, BINI, CALL, CAST, CMPF, CMPI, CONST, DEALLOC, IF_FALSE,
                   JUMP, LAUNCH, LOAD, LOOP_INIT_A, LOOP_INIT_S, PARALLEL, RETURN,
                   RETURN_GPU, STORE, Launch, Unsupported, evaluate, lift_region)
from .runtime import DeviceBackend


def _vm_reg_limit():
    """Register limit of the tier VM programs run on: none when the native
    tier is on (native.py: registers become scalars), else the interpreter's
    register file (csrc/vm.cu)."""
    from . import native

    return None if native.available() else vmcode.MAX_REGS


ENGINE_NAME = "b200"

# Execution knobs.  Process-wide defaults come from the environment and
# configure(); using(...) overrides them for the calling thread only, so
# concurrent callers (threads, the tuner) never see each other's settings.
#
# precision: contraction arithmetic.  "exact" (default): fp32 per-op
#   rounding on the FP32 pipes, bit-identical to the reference.  "f32x3": f32
#   operands split into tf32 hi + lo parts, three tf32 products per term on
#   the tensor cores — fp32-accurate (within rel 1e-5 of the reference,
#   tests/test_gpu_f32x3.py), not bit-identical.  "tf32" / "bf16": operands
#   rounded to tf32 / bf16 and contracted on the tcgen05 tensor cores with
#   fp32 accumulation (tolerance: DESIGN.md, tests/tcbound.py).
# fuse: cross-region fusion of queued plans (B200_FUSE=0 disables, A/B tests).
# shadow: bf16 shadows of contraction outputs read as the next contraction's
#   A (fusion.plan_shadows; B200_SHADOW=0 disables).
# stream_io: row-panel pipelining of the host copies of large contractions /
#   convs (runtime.Staging.stream_rows; B200_STREAM_IO=0 disables).
# strict: a bf16 / tf32 request a contraction cannot honour (no strided GEMM
#   view, unaligned K, conv shape outside the tcgen05 kernel) runs exact f32
#   with a runtime.PrecisionFallback warning; strict makes it
#   PrecisionUnavailable.
# plan_cache: per-region plan cache (plancache.py): a repeated run of the
#   same tape region with the same scalar values and buffer geometry skips
#   lifting, analysis and matching (B200_PLAN_CACHE=0 disables).
_defaults = {
    "precision": os.environ.get("B200_PRECISION", "exact"),
    "fuse": os.environ.get("B200_FUSE", "1") != "0",
    "shadow": os.environ.get("B200_SHADOW", "1") != "0",
    "stream_io": os.environ.get("B200_STREAM_IO", "1") != "0",
    "strict": os.environ.get("B200_STRICT", "0") == "1",
    "plan_cache": os.environ.get("B200_PLAN_CACHE", "1") != "0",
}
# per-thread state: using() overrides, the last run's plan and device copies,
# the race checker's region hook
_tls = threading.local()
# module attributes kept for callers that read them (engine.PRECISION, ...):
# each resolves to the calling thread's effective value (PEP 562)
_KNOB_ATTRS = {"PRECISION": "precision", "FUSE": "fuse", "SHADOW": "shadow",
               "STREAM_IO": "stream_io", "STRICT": "strict", "PLAN_CACHE": "plan_cache"}


def _validated(kw):
    bad = set(kw) - set(_defaults)
    if bad:
        raise TypeError(f"unknown engine setting(s) {sorted(bad)}")
    out = {}
    for k, v in kw.items():
        if v is None:
            continue
        if k == "precision":
            from .runtime import PRECISIONS

            if v not in PRECISIONS:
                raise ValueError(f"unknown precision {v!r}")
            out[k] = v
        else:
            out[k] = bool(v)
    return out


def settings():
    """The calling thread's effective settings (a fresh dict)."""
    eff = dict(_defaults)
    eff.update(getattr(_tls, "overrides", None) or {})
    return eff


def configure(precision=None, fuse=None, shadow=None, strict=None, stream_io=None,
              plan_cache=None):
    """Set the process-wide defaults for subsequent runs (threads inside a
    using() block keep their overrides)."""
    _defaults.update(_validated(dict(precision=precision, fuse=fuse, shadow=shadow,
                                     strict=strict, stream_io=stream_io,
                                     plan_cache=plan_cache)))
    return {k: _defaults[k] for k in ("precision", "fuse", "shadow", "strict")}


@contextlib.contextmanager
def using(**kw):
    """Override settings for the calling thread inside the block:

        with engine.using(precision="bf16", strict=True):
            machine.run(module, "matmul", args, engine=engine)
    """
    prev = getattr(_tls, "overrides", None)
    _tls.overrides = {**(prev or {}), **_validated(kw)}
    try:
        yield settings()
    finally:
        _tls.overrides = prev


@contextlib.contextmanager
def region_hook(fn):
    """Call ``fn(region, accesses)`` for every region this thread's runs lift
    (races.check_races' static proof)."""
    prev = getattr(_tls, "region_hook", None)
    _tls.region_hook = fn
    try:
        yield
    finally:
        _tls.region_hook = prev


def __getattr__(name):
    if name in _KNOB_ATTRS:
        return settings()[_KNOB_ATTRS[name]]
    if name == "last_plan":     # kernel choice of this thread's last run
        return getattr(_tls, "last_plan", [])
    if name == "last_staging":
        return getattr(_tls, "last_staging", None)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


class ExecContext:
    """Per-run execution knobs (same slots as interp/_evalpy.py:61-71)."""

    __slots__ = ("mode", "workers", "recorder", "gpu_ids", "depth")

    def __init__(self, mode="sequential", workers=1, recorder=None):
        self.mode = mode
        self.workers = workers
        self.recorder = recorder
        self.gpu_ids = None
        self.depth = 0


def _to_f32(x):
    import struct

    try:
        return struct.unpack("<f", struct.pack("<f", x))[0]
    except OverflowError:
        return math.copysign(math.inf, x)


def _wrap(v, dtype):
    span, half = (1 << 32, 1 << 31) if dtype == "i32" else (1 << 64, 1 << 63)
    return (int(v) + half) % span - half


def _where(loc):
    return f" at {loc.file}:{loc.line}" if loc else ""


class _Run:
    """One run() call: host walk of the entry tape + device regions."""

    def __init__(self, program, ctx, backend=None, shard=None):
        self.program = program
        self.ctx = ctx
        self.cfg = settings()
        self.hook = getattr(_tls, "region_hook", None)
        self.be = (backend if backend is not None
                   else DeviceBackend(stream_io=self.cfg["stream_io"]))
        self.plan = []
        self.shard = shard    # shard.Shard: run only this rank's batch rows
        self.pending = []     # queued MapItem / ContractItem, program order

    # -- host walk (mirrors interp/_evalpy.py:81-232 for top-level scalars) --
    def exec_tape(self, code, regs, tally):
        E = _errors()
        n = len(code)
        pc = 0
        while pc < n:
            ins = code[pc]
            op = ins[0]
            if op in (LOOP_INIT_S, LOOP_INIT_A):
                end = code[pc + 1][3]
                self.region(code, pc, end, regs, tally)
                pc = end
                continue
            if op in (PARALLEL, LAUNCH):
                self.region(code, pc, pc + 1, regs, tally)
                pc += 1
                continue
            if op in (LOAD, STORE):
                self.flush_pending()   # the host touches device data
            tally[op] += 1
            if op == CONST:
                regs[ins[1]] = ins[2]
            elif op == BINF:
                a, b, f = regs[ins[3]], regs[ins[4]], ins[2]
                if f == 0:
                    r = a + b
                elif f == 1:
                    r = a - b
                elif f == 2:
                    r = a * b
                else:
                    r = _fdiv(a, b)
                regs[ins[1]] = _to_f32(r) if ins[5] else r
            elif op == BINI:
                a, b, f = regs[ins[3]], regs[ins[4]], ins[2]
                r = a + b if f == 0 else (a - b if f == 1 else a * b)
                regs[ins[1]] = _wrap(r, ins[5])
            elif op == CMPF:
                regs[ins[1]] = _cmpf(ins[2], regs[ins[3]], regs[ins[4]])
            elif op == CMPI:
                regs[ins[1]] = _cmpi(ins[2], regs[ins[3]], regs[ins[4]])
            elif op == CAST:
                v = regs[ins[2]]
                regs[ins[1]] = _wrap(v, "i32") if ins[3] == "i32" else v
            elif op == LOAD:
                buf = regs[ins[2]]
                off = self._offset(buf, [regs[r] for r in ins[3]], ins[4], E)
                regs[ins[1]] = self.be.read(buf, off)
            elif op == STORE:
                buf = regs[ins[2]]
                off = self._offset(buf, [regs[r] for r in ins[3]], ins[4], E)
                v = regs[ins[1]]
                if buf.dtype[0] == "i":
                    v = _wrap(v, buf.dtype)
                self.be.write(buf, off, v)
            elif op == ALLOC:
                from staircase.interp.buffer import Buffer

                regs[ins[1]] = Buffer(ins[2], ins[3])
            elif op == DEALLOC:
                pass
            elif op == IF_FALSE:
                if not regs[ins[1]]:
                    pc = ins[2]
                    continue
            elif op == JUMP:
                pc = ins[1]
                continue
            elif op == CALL:
                callee = self.program.funcs[ins[2]]
                sub = [None] * callee.n_regs
                for dst, src in zip(callee.arg_regs, ins[3]):
                    sub[dst] = regs[src]
                rets = self.exec_tape(callee.code, sub, tally)
                for dst, v in zip(ins[1], rets or ()):
                    regs[dst] = v
            elif op in (RETURN, RETURN_GPU):
                return tuple(regs[r] for r in ins[1])
            else:
                raise E.UnknownOperation(f"opcode {op} at the top level of a tape")
            pc += 1
        return None

    @staticmethod
    def _offset(buf, idx, loc, E):
        off = 0
        for i, extent, stride in zip(idx, buf.shape, buf.strides):
            if i < 0 or i >= extent:
                raise E.OutOfBounds(
                    f"index {i} out of bounds for extent {extent} of {buf!r}{_where(loc)}")
            off += i * stride
        return off

    # -- regions ---------------------------------------------------------------
    def region(self, code, start, end, regs, tally):
        key = None
        cfg = self.cfg
        cacheable = cfg["plan_cache"] and self.shard is None and self.hook is None
        if cacheable:
            rkey = (plancache.region_key(self.program, code, start, end), self.ctx.mode,
                    cfg["precision"], cfg["fuse"], cfg["shadow"])
            key = plancache.lookup_key(rkey, regs)
            hit = plancache.get(key)
            if hit is not None:
                self.replay(hit, regs, tally)
                return
        E = _errors()
        try:
            r = lift_region(self.program, code, start, end, regs)
            evaluate(r)
        except Unsupported as exc:
            self.flush_pending()
            raise E.ModeUnsupported(f"b200 engine: {exc}") from None
        if r.has_launch and self.ctx.mode != "gpu_emulated":
            self.flush_pending()
            loc = _first_launch_loc(r.tree)
            raise E.ModeUnsupported(
                f"gpu.launch_func needs gpu_emulated mode, not {self.ctx.mode!r}{_where(loc)}")
        try:
            accesses = analysis.collect_accesses(r)
        except Unsupported as exc:
            self.flush_pending()
            raise E.ModeUnsupported(f"b200 engine: {exc}") from None
        if self.shard is not None:   # batch-sharded run (shard.py)
            try:
                self.shard.restrict(r, accesses, getattr(self.be, "stage", None))
            except E.ModeUnsupported:
                self.flush_pending()
                raise
        if self.hook is not None:   # races.check_races: static race proof
            self.hook(r, accesses)
        links, remainder = analysis.chain_of(r)
        safe = analysis.statically_in_bounds(r, accesses) and not analysis.invalid_steps(r)
        # a region with memref.alloc runs on one thread: its scratch buffer
        # is the reference's sequence of fresh buffers (lift._leaf ALLOC)
        band = analysis.choose_band(r, links, accesses) if safe and not r.has_alloc else []
        st = analysis.static_tally(r.tree)
        written = {a.slot for a in accesses if a.write}
        for slot in written:
            self.be.mark_dirty(r.buffers[slot])

        store = key is None and cacheable
        if safe and st is not None:
            g = templates.match_contraction(r, links, remainder, accesses)
            if g is not None:
                _add(tally, st)
                self.pending.append(fusion.ContractItem(g))
                if store:
                    plancache.put(rkey, regs, r, plancache.Plan("contract", st, written, g))
                return
            mm = templates.match_map(r, links, remainder, accesses, band)
            if mm is not None:
                _add(tally, st)
                self.pending.append(fusion.MapItem(mm))
                if store:
                    plancache.put(rkey, regs, r, plancache.Plan("map", st, written, mm))
                return

        # generic tier: the device tape VM (runs in order after queued plans)
        count = st is None
        try:
            prog = vmcode.encode(r, links, remainder, band, count, checked=not safe,
                                 max_regs=_vm_reg_limit())
        except Unsupported as exc:
            self.flush_pending()
            raise E.ModeUnsupported(f"b200 engine: {exc}") from None
        chain = analysis.chain_tally(links)[0] if count else None
        entry = ("vm", len(band), "checked" if not safe else "unchecked",
                 "count" if count else "static")
        plan = plancache.Plan("vm", st, written, prog, chain=chain, entry=entry,
                              checked=not safe)
        if store:
            plancache.put(rkey, regs, r, plan)
        self.run_vm(r, plan, tally)

    def run_vm(self, r, plan, tally):
        """Execute a VM plan after the queued plans; tally; raise its fault."""
        self.flush_pending({id(r.buffers[slot]) for slot in plan.written})
        prog = plan.item
        limit = _vm_reg_limit()
        if limit is not None and prog.n_regs > limit:
            # a cached plan encoded for the native tier, which is now off
            raise _errors().ModeUnsupported(
                f"b200 engine: region needs {prog.n_regs} VM registers (max {limit} without "
                f"the native tier)")
        dev_tally, fault = self.be.vm(r, prog, checked=plan.checked)
        if fault is not None:
            self.be.flush()
            self.raise_fault(r, prog, fault)
        if plan.chain is not None:
            _add(tally, plan.chain)
            _add(tally, dev_tally)
        else:
            _add(tally, plan.st)
        self.plan.append(plan.entry)

    def replay(self, hit, regs, tally):
        """A cached region plan (plancache) bound to this run's registers."""
        plan, shell = hit
        r = plancache.bind(shell, regs)
        for slot in plan.written:
            self.be.mark_dirty(r.buffers[slot])
        if plan.kind == "contract":
            _add(tally, plan.st)
            self.pending.append(fusion.ContractItem(
                plancache.rebind_contract(plan.item, r, plan.slots)))
        elif plan.kind == "map":
            _add(tally, plan.st)
            self.pending.append(fusion.MapItem(plancache.rebind_map(plan.item, r, plan.slots)))
        else:
            self.run_vm(r, plan, tally)

    def flush_pending(self, trigger_writes=()):
        """Execute the queued plans.  ``trigger_writes``: ids of the buffers
        the region that forced the flush will write (already marked dirty)."""
        if not self.pending:
            return
        items = fusion.fuse(self.pending) if self.cfg["fuse"] else self.pending
        if self.cfg["shadow"]:
            fusion.plan_shadows(items)
        self.pending = []
        # last_writer[i]: no later queued plan (nor the triggering region)
        # writes item i's output, so a write-back streamed by item i is final
        later = set(trigger_writes)
        last_writer = [False] * len(items)
        for i in range(len(items) - 1, -1, -1):
            it = items[i]
            if isinstance(it, fusion.ContractItem):
                last_writer[i] = id(it.g.C) not in later
                later.add(id(it.g.C))
            else:
                # conservatively every operand of a map counts as written
                last_writer[i] = not any(id(b) in later for b in it.m.buffers)
                later.update(id(b) for b in it.m.buffers)
        for it, last in zip(items, last_writer):
            if isinstance(it, fusion.ContractItem):
                kernels = self.be.contract(it.g, self.cfg["precision"], init=it.init,
                                           init_value=it.init_value, bias=it.bias,
                                           bias_base=it.bias_base,
                                           bias_stride=it.bias_stride,
                                           shadow_out=it.shadow_out, shadow_in=it.shadow_in,
                                           last_writer=last)
                g = it.g
                fused = list(it.fused)
                if it.shadow_in or it.shadow_out:
                    used_in, made_out = getattr(self.be, "last_shadow", (False, False))
                    fused += ["A<-shadow"] * used_in + ["C->shadow"] * made_out
                cta = getattr(self.be, "last_cta", None)
                if cta is not None:
                    tm, tn = g.tiles
                    fused.append(f"tile{tm or 1}x{tn or 1}->cta{cta[0]}x{cta[1]}")
                note = getattr(self.be, "last_note", None)
                if note:
                    fused.append(note)
                if "pack_conv_weight" in kernels:   # b200_conv2d_tc_fused
                    fused.append("input converted in-kernel")
                self.plan.append((kernels[-1], g.M, g.N, g.K) +
                                 ((tuple(fused),) if fused else ()))
            else:
                m = it.m
                self.be.map(m, last_writer=last)
                self.plan.append(("map_" + m.kind, tuple(m.trips),
                                  "vec4" if m.vector else "scalar"))

    def raise_fault(self, r, prog, fault):
        code, slot, index, extent, loc = fault
        E = _errors()
        if code == 1:
            loc = prog.locs[loc] if loc >= 0 else None
            raise E.OutOfBounds(
                f"index {index} out of bounds for extent {extent} of "
                f"{r.buffers[slot]!r}{_where(loc)}")
        if code == 2:
            raise E.InvalidBound("loop step must be positive at runtime")
        raise E.InvalidBound("scf.parallel steps must be positive at runtime")


def _first_launch_loc(nodes):
    from .analysis import _iter_nodes

    for n in _iter_nodes(nodes):
        if isinstance(n, Launch):
            return n.loc
    return None


def _add(tally, extra):
    for i, v in enumerate(extra):
        tally[i] += v


def _fdiv(a, b):
    if b == 0.0:
        if a != a or a == 0.0:
            return math.nan
        return math.copysign(math.inf, a) * math.copysign(1.0, b)
    return a / b


def _cmpf(p, a, b):
    if p == 0:
        return a == b
    if p == 1:
        return a == a and b == b and a != b
    return (a < b, a <= b, a > b, a >= b)[p - 2]


def _cmpi(p, a, b):
    return (a == b, a != b, a < b, a <= b, a > b, a >= b)[p]


def run_tape(program, code, regs, tally, ctx, backend=None, shard=None):
    """Engine-protocol entry point (machine.py:112).  ``shard``: a
    shard.Shard — execute only this rank's batch rows (shard.run)."""
    run = _Run(program, ctx, backend, shard)
    try:
        rets = run.exec_tape(code, regs, tally)
        run.flush_pending()
    except BaseException:
        try:
            run.flush_pending()
            run.be.flush()
        finally:
            _tls.last_plan = run.plan
        raise
    run.be.flush()
    _tls.last_plan = run.plan
    # the run's device copies (== the host Buffers after the flush): kept
    # until this thread's next run so a caller can post-process on the
    # device (the sweep's equivalence guard, sweep.py)
    _tls.last_staging = getattr(run.be, "stage", None)
    return rets


def release_last_staging():
    """Drop this thread's last run's device copies (kept for device_copy)."""
    _tls.last_staging = None


def device_copy(buf):
    """The last run's device tensor of ``buf`` (same contents), or None."""
    st = getattr(_tls, "last_staging", None)
    if st is None or not hasattr(st, "dev"):
        return None
    ent = st.dev.get(id(buf))
    return ent[1] if ent is not None and ent[0] is buf else None


class Session:
    """Device-resident execution of staircase modules on the B200.

    ``run()`` has the signature and results of ``machine.run`` but Buffers
    stay in HBM between runs (uploaded on first use, no write-back until
    ``sync()``), so chains of runs on the same data — or repeated timing
    runs — move no host data.  ``record()`` runs a module once and returns
    the exact launch sequence the engine chose (runtime.Recording), which
    ``replay()``s without re-planning; it can be captured in a CUDA graph.
    Host data changed after the first upload is not re-read (call
    ``forget(buf)``).
    """

    def __init__(self, shard=None):
        self.be = DeviceBackend()
        self.plan = []
        # (rank, world): every run executes only this rank's batch rows
        # (shard.py); the Session's device copies hold those rows
        self.shard = shard
        self.last_shard = None

    def _engine(self):
        sess = self

        class _Eng:
            ExecContext = globals()["ExecContext"]

            @staticmethod
            def run_tape(program, code, regs, tally, ctx):
                sh = None
                if sess.shard is not None:
                    from .shard import Shard

                    sh = sess.last_shard = Shard(*sess.shard)
                run = _Run(program, ctx, sess.be, sh)
                try:
                    rets = run.exec_tape(code, regs, tally)
                finally:
                    run.flush_pending()
                    sess.plan = run.plan
                return rets

        return _Eng

    def run(self, module, func, args, mode="sequential", workers=1):
        from staircase.interp import machine

        return machine.run(module, func, args, mode=mode, workers=workers,
                           engine=self._engine())

    def record(self, module, func, args, mode="sequential", workers=1):
        from .runtime import Recording

        self.be.recording = Recording()
        try:
            self.run(module, func, args, mode=mode, workers=workers)
        finally:
            rec, self.be.recording = self.be.recording, None
        return rec

    def tensor(self, buf):
        """The device tensor backing a Buffer in this session."""
        return self.be.stage.tensor(buf)

    def forget(self, buf):
        self.be.stage.dev.pop(id(buf), None)

    def sync(self):
        """Write every buffer the session's runs modified back to the host."""
        self.be.flush()


_previous_engine = None


def install():
    """Make this engine the default of staircase.interp.machine.run().

    machine.ENGINE_NAME (computed once at import, machine.py:34) is updated
    too, so the reference's reports name the engine that actually runs."""
    global _previous_engine
    from .host import ensure_staircase

    ensure_staircase()
    import sys

    from staircase.interp import machine

    me = sys.modules[__name__]
    if machine._engine is not me:
        _previous_engine = (machine._engine, machine.ENGINE_NAME)
    machine._engine = me
    machine.ENGINE_NAME = ENGINE_NAME
    return machine


def uninstall():
    """Restore the engine install() replaced."""
    global _previous_engine
    from staircase.interp import machine

    if _previous_engine is not None:
        machine._engine, machine.ENGINE_NAME = _previous_engine
        _previous_engine = None
    return machine


__all__ = ["ExecContext", "run_tape", "install", "uninstall", "configure", "using",
           "settings", "region_hook", "ENGINE_NAME"]
