"""The tile-size / unroll design-space sweep, sharded across GPUs.

Reference: ``staircase.tuner.search`` (reference pkg/src/staircase/tuner/
search.py:237-279) evaluates ``budget`` trials in sequence, trial 0 being the
identity point; each trial instantiates the pipeline template
(``default_pipeline``, search.py:38-53), runs it, interprets the result on
fixed seeded inputs, checks it against the baseline (rel 1e-6 / abs 1e-9,
search.py:109-138) and scores it with the tally cost model (or wall time).

``search`` here keeps those semantics by reusing the reference's own
``_Session`` for every trial (baseline, pass pipeline, guard, scoring) and
only changes *where* trials run: with ``torch.distributed`` initialised,
trial ``idx`` runs on rank ``idx % world``; every rank then exchanges its
trial records with one ``all_gather_object`` (NCCL or gloo) and all ranks
return the same ``(best, log)``.  For the ``random`` strategy the trial
parameters depend only on the seed (search.py:220-224), so every rank
regenerates the full sequence and the merged log equals the sequential log
(``objective="model"``: costs come from the exact tally).  ``grid`` (an
extension: trial 0 identity, then the Cartesian product in order) shards the
same way.  ``one_plus_one_es`` depends on earlier costs (search.py:226-234,
272-275) and runs as identical replicas on every rank; ``population_es``
(an extension) evaluates λ mutations of the parent per
generation, sharded over the ranks, and equals (1+1)-ES at λ = 1.

``objective="device"`` (an extension) scores a trial by the device time of
the launch sequence the engine chose for it (recorded, replayed between CUDA
events): on the B200 the reference's ``"wall"`` (``stats.wall_time``, the
whole host-side run()) is dominated by lifting and planning and barely sees
the tile choice, while the tile sizes select the CTA tile of the
contraction kernels (runtime.cta_tile), which the device time does see.

Trials run on the B200 engine: the session passes it to every run()
explicitly (no module-global patching).  With several ranks, an exception in
a trial is exchanged like a record and re-raised on every rank (the lowest
index first, as the sequential reference would raise it), so no rank is
left waiting in the all-gather.
"""
from __future__ import annotations

import itertools
import math
import os
import random

import numpy as np

from .host import ensure_staircase


def _dist():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist
    except ImportError:
        pass
    return None


_WANT_DEV = {}   # id(want Buffer) -> (Buffer, float64 device tensor): baseline copies


def _close_tensors(g, w):
    """math.isclose(g, w, rel_tol=1e-6, abs_tol=1e-9) elementwise, all():
    equal values (infinities included) are close; otherwise both must be
    finite and |g - w| <= max(1e-6 * max(|g|, |w|), 1e-9); NaN is never
    close (math.isclose semantics)."""
    xp_abs = abs
    diff = xp_abs(g - w)
    tol = (1e-6 * _maximum(xp_abs(g), xp_abs(w))).clip(min=1e-9)
    return (g == w) | (_isfinite(g) & _isfinite(w) & (diff <= tol))


def _maximum(a, b):
    import torch

    return torch.maximum(a, b) if isinstance(a, torch.Tensor) else np.maximum(a, b)


def _isfinite(a):
    import torch

    return torch.isfinite(a) if isinstance(a, torch.Tensor) else np.isfinite(a)


def _fast_buffers_close(got, want, dev_of=None, counter=None):
    """Vectorised twin of the reference guard's element test
    (math.isclose(g, w, rel_tol=1e-6, abs_tol=1e-9) over every element,
    tuner/search.py:128-138): the same predicate, evaluated on the GPU on
    the trial run's own device copy of ``got`` (engine.device_copy) against
    a cached device copy of the baseline, else with numpy."""
    from staircase.interp import Buffer

    if not isinstance(got, Buffer) or got.shape != want.shape:
        return False
    from . import engine

    tg = (dev_of or engine.device_copy)(got)
    ent = _WANT_DEV.get(id(want))
    if tg is None and ent is not None and ent[0] is want:
        # the baseline lives only on the device (a resident session's
        # baseline): compare the host result there
        import torch

        tg = torch.from_numpy(np.frombuffer(got.data, dtype=_NP_DT[got.dtype])).to("cuda")
    if tg is not None:
        import torch

        ent = _WANT_DEV.get(id(want))
        if ent is None or ent[0] is not want:
            dt = getattr(torch, {"f32": "float32", "f64": "float64", "i32": "int32",
                                 "i64": "int64"}[want.dtype])
            tw = torch.frombuffer(want.data, dtype=dt).to("cuda")
            ent = (want, tw.double() if want.dtype in ("f32", "f64") else tw)
            _WANT_DEV[id(want)] = ent
        tw = ent[1]
        if want.dtype not in ("f32", "f64"):
            return bool(torch.equal(tg, tw))
        if counter is not None:
            # one native kernel per buffer, counts summed on the device and
            # read once per trial (_state_matches): no temporaries
            import ctypes

            from .runtime import check, load_library

            P = ctypes.c_void_p
            check(load_library().b200_guard_close(
                0 if want.dtype == "f32" else 1, P(tg.data_ptr()), P(tw.data_ptr()), tg.numel(),
                1e-6, 1e-9, P(counter.data_ptr()),
                P(torch.cuda.current_stream().cuda_stream)), "b200_guard_close")
            return None
        return bool(_close_tensors(tg.double(), tw).all().item())
    if want.dtype not in ("f32", "f64"):
        return list(got.data) == list(want.data)
    dt = np.float32 if want.dtype == "f32" else np.float64
    g = np.frombuffer(got.data, dtype=dt).astype(np.float64)
    w = np.frombuffer(want.data, dtype=dt).astype(np.float64)
    with np.errstate(invalid="ignore", over="ignore"):
        close = _close_tensors(g, w)
    return bool(np.all(close))


def make_inputs(module, func, seed):
    """The reference's make_inputs (tuner/search.py:78-102), bit for bit, with
    the float memrefs drawn by numpy: ``random.Random(seed)``'s Mersenne
    Twister state is handed to a numpy RandomState, whose random_sample()
    is the same 53-bit draw as random.random(), so uniform(-2, 2) =
    -2 + 4 * random() gives the same doubles (and, stored into an f32
    Buffer, the same round-to-nearest floats); the state is handed back for
    the next argument.  Integer, i1 and scalar arguments use the Python
    generator itself.  ~30x faster on the sweep's 1024^2 operands, which
    dominated each rank's setup."""
    import importlib
    import math

    from staircase.interp import Buffer

    # the module (staircase.tuner re-exports the function under the same name)
    ref = importlib.import_module("staircase.tuner.search")

    func_op = ref._find_func(module, func)
    rng = random.Random(seed)
    out = []
    for arg in func_op.body().args:
        ty = arg.type
        if ty.kind == "memref" and ty.element.is_float:
            size = math.prod(ty.shape)
            dt = np.float32 if ty.element.kind == "f32" else np.float64
            out.append(_buffer_from(ty.shape, ty.element.kind, _uniform(rng, size, dt)))
        else:
            out.append(ref._fresh_argument(ty, rng))
    return out


def _uniform(rng, size, dt):
    """[rng.uniform(-2.0, 2.0) for _ in range(size)] as a numpy array of dt,
    leaving ``rng`` where that loop would: the native generator
    (b200_mt_uniform, host code) when the library loads, else a numpy
    RandomState seeded with the same Mersenne Twister state (random_sample()
    is the same 53-bit draw as random.random())."""
    st = rng.getstate()
    words = np.array(st[1][:-1], dtype=np.uint32)
    out = np.empty(size, dtype=dt)
    lib = _native()
    if lib is not None:
        import ctypes

        pos = ctypes.c_int32(st[1][-1])
        rc = lib.b200_mt_uniform(words.ctypes.data, ctypes.byref(pos), size, -2.0, 2.0,
                                 out.ctypes.data, 0 if dt == np.float32 else 1)
        if rc != 0:
            raise RuntimeError(f"b200_mt_uniform failed ({rc})")
        rng.setstate((3, tuple(words.tolist()) + (pos.value,), None))
        return out
    rs = np.random.RandomState()
    rs.set_state(("MT19937", words, st[1][-1]))
    vals = rs.random_sample(size)
    vals *= 2.0 - -2.0      # same rounding as -2 + (2 - -2) * random()
    vals += -2.0
    s2 = rs.get_state()
    rng.setstate((3, tuple(s2[1].tolist()) + (int(s2[2]),), None))
    out[...] = vals
    return out


def _native():
    try:
        from .runtime import load_library

        return load_library()
    except Exception:   # no library built: the numpy path draws the same values
        return None


def _buffer_from(shape, dtype, values):
    """A staircase Buffer holding ``values`` (a numpy array of the Buffer's
    element type), filled with one copy (Buffer(shape, dtype, bytes) makes
    three)."""
    from array import array

    from staircase.interp import Buffer
    from staircase.interp.buffer import _TYPECODES, row_major_strides

    b = Buffer.__new__(Buffer)
    b.shape = tuple(int(x) for x in shape)
    b.strides = row_major_strides(b.shape)
    b.dtype = dtype
    b.data = array(_TYPECODES[dtype])
    b.data.frombytes(memoryview(np.ascontiguousarray(values)).cast("B"))
    return b


def _session_class():
    """The reference trial session (tuner/search.py:151-201) bound to an
    engine and with a vectorised equivalence guard.

    ``__init__`` and ``trial`` restate the reference's (same baseline run,
    pass pipeline, skip rules, guard and scoring) with two differences: every
    run() goes to the session's engine explicitly — no patching of
    ``machine._engine`` — and the guard is ``_state_matches`` below, the
    reference predicate (search.py:115-127) evaluated on the device."""
    ensure_staircase()
    import importlib

    # the module (staircase.tuner re-exports the function under the same name)
    ref = importlib.import_module("staircase.tuner.search")
    from staircase.errors import PassFailure, StaircaseError, VerificationFailed
    from staircase.interp import machine
    from staircase.passes import run_pipeline
    from staircase.tuner.space import Trial

    def _state_matches(got_results, got_args, want_results, want_args, dev_of=None):
        from staircase.interp import Buffer

        if len(got_results) != len(want_results):
            return False
        counter = None
        if dev_of is not None:   # resident trial: device comparisons, one read-back
            import torch

            counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        for g, w in zip(got_results, want_results):
            if isinstance(w, Buffer):
                if _fast_buffers_close(g, w, dev_of, counter) is False:
                    return False
            elif not ref._values_close(g, w):
                return False
        for g, w in zip(got_args, want_args):
            if isinstance(w, Buffer) and _fast_buffers_close(g, w, dev_of, counter) is False:
                return False
        return counter is None or int(counter.item()) == 0

    class Session(ref._Session):
        """The reference trial session on a given engine."""

        def __init__(self, module, engine, func=None, seed=0, objective="model",
                     pipeline_template=None, mode="sequential", workers=1):
            if objective not in ("model", "wall", "device"):
                raise ValueError(f"unknown objective {objective!r}")
            if objective == "device" and engine is not _b200_engine():
                raise ValueError("objective 'device' times the B200 engine's kernels; "
                                 "it needs engine=paper_2307_16080_b200.engine")
            ref.verify_or_raise(module)
            self.engine = engine
            self.module = module
            self.func_op = ref._find_func(module, func)
            self.func = self.func_op.attributes["sym_name"].value
            self.seed = seed
            self.objective = objective
            self.template = pipeline_template or ref.default_pipeline
            self.mode = mode
            self.workers = workers
            self.inputs = make_inputs(module, self.func, seed)
            # resident trial inputs (B200 engine): every trial starts from
            # device clones of one upload instead of host copies + uploads
            self._masters = None
            stats = None
            if engine is _b200_engine() and RESIDENT:
                import torch

                from staircase.interp import Buffer

                self._masters = [
                    torch.from_numpy(np.frombuffer(a.data, dtype=_NP_DT[a.dtype])).to("cuda")
                    if isinstance(a, Buffer) else None for a in self.inputs]
                stats = self._device_baseline(module)
            if stats is None:
                args = ref._copy_args(self.inputs)
                results, stats = machine.run(module, self.func, args, mode="sequential",
                                             engine=engine)
                self.want_results = results
                self.want_args = args
            self.baseline_cost = (self._device_ms(module) if objective == "device"
                                  else self._score(stats))
            self.baseline_stats = stats

        def _device_baseline(self, module):
            """The baseline run on device clones of the inputs, its outputs
            kept on the device as the guard's reference (_WANT_DEV) — no host
            copies of the inputs, no write-back.  None (host baseline
            instead) when a baseline Buffer has no device copy to compare
            against."""
            from staircase.interp import Buffer

            sess, args = self._resident_args()
            results, stats = sess.run(module, self.func, args, mode="sequential")
            stage = sess.be.stage
            wants = [b for b in list(results) + list(args) if isinstance(b, Buffer)]
            devs = []
            for b in wants:
                ent = stage.dev.get(id(b))
                if ent is None or ent[0] is not b:
                    return None
                devs.append(ent[1])
            for b, t in zip(wants, devs):
                _WANT_DEV[id(b)] = (b, t.double() if b.dtype in ("f32", "f64") else t)
            self._want_session = sess      # keeps the device copies alive
            self.want_results = results
            self.want_args = args
            return stats

        def _resident_args(self):
            """(device Session, trial arguments) for a resident trial: Buffer
            shells share the input arrays (read only: a Session never writes
            back) and their device copies are clones of the resident inputs —
            the trial sees exactly the reference's fresh copies
            (search.py:105-106), without a host copy or an upload."""
            from staircase.interp import Buffer

            from .engine import Session as DeviceSession

            sess = DeviceSession()
            args = []
            for a, m in zip(self.inputs, self._masters):
                if isinstance(a, Buffer):
                    shell = Buffer.__new__(Buffer)
                    shell.shape, shell.strides, shell.dtype = a.shape, a.strides, a.dtype
                    shell.data = a.data
                    sess.be.stage.adopt(shell, m.clone())
                    args.append(shell)
                else:
                    args.append(a)
            return sess, args

        def _device_ms(self, module):
            """objective="device": the device time (ms) of the launch
            sequence the engine runs for ``module`` on this session's inputs
            — recorded once on resident copies, then replayed (1 warm-up,
            median of DEVICE_REPS) between CUDA events on the launch stream.
            Unlike the reference's "wall" (stats.wall_time: the whole run()
            on the host, dominated here by lifting and planning), this
            separates tile choices that select different kernels / CTA
            tiles.  Not log-equal to anything in the reference (timing)."""
            import torch

            from .engine import Session as DeviceSession

            if self._masters is not None:
                sess, args = self._resident_args()
            else:
                sess, args = DeviceSession(), ref._copy_args(self.inputs)
            rec = sess.record(module, self.func, args, mode=self.mode, workers=self.workers)
            if not rec.calls:
                return 0.0
            stream = torch.cuda.current_stream()
            rec.replay()
            times = []
            for _ in range(DEVICE_REPS):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rec.replay()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            times.sort()
            return times[len(times) // 2]

        def trial(self, idx, tiles, unroll):
            params = {"tiles": [int(t) for t in tiles], "unroll": int(unroll)}
            spec = self.template(params["tiles"], params["unroll"])
            try:
                work, _ = run_pipeline(self.module, spec)
            except (PassFailure, VerificationFailed):
                return Trial(idx, params, None, "skipped", self.seed)
            dev_of = None
            try:
                if self._masters is not None:
                    sess, args = self._resident_args()
                    results, stats = sess.run(work, self.func, args, mode=self.mode,
                                              workers=self.workers)
                    stage = sess.be.stage

                    def dev_of(buf):
                        ent = stage.dev.get(id(buf))
                        return ent[1] if ent is not None and ent[0] is buf else None
                else:
                    args = ref._copy_args(self.inputs)
                    results, stats = machine.run(work, self.func, args, mode=self.mode,
                                                 workers=self.workers, engine=self.engine)
                dev_ms = self._device_ms(work) if self.objective == "device" else None
            finally:
                if work in self.module.ctx.modules:
                    self.module.ctx.modules.remove(work)
            try:
                ok = _state_matches(results, args, self.want_results, self.want_args, dev_of)
            finally:
                # the guard was the last user of the trial's device copies
                release = getattr(self.engine, "release_last_staging", None)
                if release is not None:
                    release()
            if not ok:
                raise StaircaseError(
                    f"pipeline {spec!r} changed the results of @{self.func}; "
                    "transformed kernels must match the untransformed run")
            cost = dev_ms if dev_ms is not None else self._score(stats)
            return Trial(idx, params, cost, "evaluated", self.seed, stats=ref._digest(stats))

    return Session, ref


DEVICE_REPS = 5
# resident trial inputs on the B200 engine (B200_SWEEP_RESIDENT=0: every trial
# copies its inputs on the host and uploads them, as the reference copies)
RESIDENT = os.environ.get("B200_SWEEP_RESIDENT", "1") != "0"
_TORCH_DT = {"f32": "float32", "f64": "float64", "i32": "int32", "i64": "int64"}
_NP_DT = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}


def _b200_engine():
    from . import engine

    return engine


def _params(space, budget, seed, strategy):
    """Trial parameters for idx 1..budget-1 (random / grid only)."""
    out = {}
    if strategy == "random":
        from staircase.tuner.search import _sample_random

        rng = random.Random(seed)
        for idx in range(1, budget):
            out[idx] = _sample_random(space, rng)
    else:   # grid
        pts = itertools.product(*space.tile_sizes, space.unroll_factors)
        for idx, pt in zip(range(1, budget), pts):
            out[idx] = (list(pt[:-1]), pt[-1])
    return out


def search(kernel, pipeline_template=None, space=None, budget: int = 20, seed: int = 0,
           strategy: str = "random", *, func=None, objective="model", mode="sequential",
           workers=1, engine=None, rank=None, world=None, timing=None, lam=8, group=None):
    """``tuner.search`` with trials sharded over torch.distributed ranks.

    Returns ``(best, log)`` exactly like the reference; ``log`` is sorted by
    trial index and identical on every rank.  ``strategy="population_es"``
    (alias ``"1+lambda-es"``) is the (1+λ)-ES extension, ``lam`` children per
    generation (see ``_pop_es``).  ``timing`` (a dict), if given,
    receives this rank's ``setup_s`` (inputs + baseline run), ``trials_s``
    (its share of the trials), ``gather_s`` and ``trials`` (count).
    ``group``: a torch.distributed process group to shard over (with
    ``rank`` / ``world`` its own rank and size; search_many uses it).
    """
    import time

    t_start = time.perf_counter()
    _WANT_DEV.clear()   # baseline device copies belong to one search
    ensure_staircase()
    from staircase.errors import EmptySpace
    from staircase.tuner.space import Trial

    if space is None:
        raise EmptySpace("search needs a ParamSpace")
    if not isinstance(budget, int) or isinstance(budget, bool) or budget < 1:
        raise ValueError(f"budget must be a positive integer, got {budget!r}")
    strategy = {"es": "one_plus_one_es", "1+1-es": "one_plus_one_es",
                "1+lambda-es": "population_es", "pop-es": "population_es"}.get(strategy, strategy)
    if strategy not in ("random", "one_plus_one_es", "grid", "population_es"):
        raise ValueError(f"unknown strategy {strategy!r}")
    if not isinstance(lam, int) or isinstance(lam, bool) or lam < 1:
        raise ValueError(f"lam must be a positive integer, got {lam!r}")
    if strategy == "grid":
        budget = min(budget, 1 + math.prod(len(d) for d in space.tile_sizes) *
                     len(space.unroll_factors))
    dist = _dist()
    if rank is None:
        rank = dist.get_rank() if dist else 0
    if world is None:
        world = dist.get_world_size() if dist else 1

    if engine is None:
        from . import engine as b200_engine

        engine = b200_engine
    Session, ref = _session_class()
    module = ref._resolve_module(kernel)
    session = Session(module, engine, func=func, seed=seed, objective=objective,
                      pipeline_template=pipeline_template, mode=mode, workers=workers)
    if strategy == "one_plus_one_es":
        # cost-dependent mutations: sequential by definition; every rank
        # runs the same replica (no exchange needed)
        best, log = _es(session, space, budget, seed)
        return best, log
    if strategy == "population_es":
        t_trials = time.perf_counter()
        best, log = _pop_es(session, space, budget, seed, lam, rank, world, dist, group)
        if timing is not None:
            timing.update(setup_s=t_trials - t_start,
                          trials_s=time.perf_counter() - t_trials, gather_s=0.0,
                          trials=sum(1 for t in log if t.idx % world == rank))
        return best, log
    identity = space.identity()
    params = _params(space, budget, seed, strategy)
    mine = []
    t_trials = time.perf_counter()
    for idx in range(budget):
        if idx % world != rank:
            continue
        tiles, unroll = ((identity["tiles"], identity["unroll"]) if idx == 0 else
                         params[idx])
        rec = _guarded(session, idx, tiles, unroll, world)
        mine.append(rec)
        if rec[3] == _FAILED:
            break   # later trials of this rank cannot matter: idx order decides
    t_gather = time.perf_counter()
    records = _raise_first(sorted(_gather(dist, world, mine, group), key=lambda r: r[0]))
    if timing is not None:
        timing.update(setup_s=t_trials - t_start, trials_s=t_gather - t_trials,
                      gather_s=time.perf_counter() - t_gather, trials=len(mine))
    log = [Trial(i, p, c, s, sd, stats=st) for i, p, c, s, sd, st in records]
    evaluated = [t for t in log if t.status == "evaluated"]
    best = min(evaluated, key=lambda t: (t.cost, t.idx))
    return best, log


def rank_groups(weights, world):
    """Ranks for each of several sweeps (search_many): contiguous groups,
    sizes proportional to ``weights`` (largest remainders), at least one
    rank each.  With fewer ranks than sweeps, sweep k runs alone on rank
    k % world."""
    n = len(weights)
    if world < n:
        return [[k % world] for k in range(n)]
    total = float(sum(weights)) or 1.0
    raw = [world * w / total for w in weights]
    size = [max(1, int(r)) for r in raw]
    while sum(size) > world:   # the max(1, .) floors overshot: take from the largest
        size[max(range(n), key=lambda k: (size[k], -k))] -= 1
    order = sorted(range(n), key=lambda k: (-(raw[k] - int(raw[k])), k))
    i = 0
    while sum(size) < world:
        size[order[i % n]] += 1
        i += 1
    out, r0 = [], 0
    for k in range(n):
        out.append(list(range(r0, r0 + size[k])))
        r0 += size[k]
    return out


def search_many(kernels, pipeline_template=None, space=None, budget: int = 20, seed: int = 0,
                strategy: str = "random", *, weights=None, rank=None, world=None, timing=None,
                **kw):
    """Several sweeps at once (the paper's design space over more than one
    kernel), partitioned across the ranks: each kernel gets its own group of
    ranks (rank_groups, sizes proportional to ``weights``, default equal)
    whose members shard that kernel's trials ``idx % group size`` — so a
    rank builds one kernel's inputs and baseline instead of every kernel's
    (the per-kernel setup is replicated only inside a group).  Returns
    ``[(best, log), ...]`` in kernel order, identical on every rank and equal
    to ``search`` of each kernel alone.  ``timing`` receives this rank's
    kernel index and its search() phases."""
    import time

    dist = _dist()
    if rank is None:
        rank = dist.get_rank() if dist else 0
    if world is None:
        world = dist.get_world_size() if dist else 1
    n = len(kernels)
    groups = rank_groups(weights or [1] * n, world)
    pgs = [None] * n
    if dist is not None and world > 1:
        made = {}
        for k, g in enumerate(groups):   # every rank creates every group, same order
            key = tuple(g)
            if key not in made:
                made[key] = dist.new_group(list(g)) if len(g) > 1 else None
            pgs[k] = made[key]
    mine = {}
    for k, g in enumerate(groups):
        if rank not in g:
            continue
        t = {} if timing is not None else None
        t0 = time.perf_counter()
        mine[k] = search(kernels[k], pipeline_template, space, budget, seed, strategy,
                         rank=g.index(rank), world=len(g), group=pgs[k], timing=t, **kw)
        if timing is not None:
            timing.setdefault("kernels", []).append(k)
            for key, v in (t or {}).items():
                timing[key] = timing.get(key, 0) + v
            timing["wall_s"] = timing.get("wall_s", 0.0) + time.perf_counter() - t0
            timing.setdefault("per_kernel", {})[k] = dict(t or {}, wall_s=time.perf_counter() - t0)
    # every rank learns every kernel's result from the group leaders
    leaders = {k: v for k, v in mine.items() if groups[k][0] == rank}
    parts = _gather(dist, world, [leaders]) if dist is not None and world > 1 else [leaders]
    out = {}
    for part in parts:
        out.update(part)
    return [out[k] for k in range(n)]


_FAILED = "__failed__"


def _guarded(session, idx, tiles, unroll, world):
    """One trial as a record; with several ranks an exception (the guard's
    StaircaseError, an engine error) becomes a record too, so every rank
    still reaches the all-gather instead of leaving the others blocked in
    it.  _raise_first re-raises it on every rank."""
    if world == 1:
        return _record(session.trial(idx, tiles, unroll))
    try:
        return _record(session.trial(idx, tiles, unroll))
    except Exception as exc:   # noqa: BLE001 — re-raised after the exchange
        return (idx, None, None, _FAILED, None, exc)


def _raise_first(records):
    """Re-raise the exception of the lowest-index failed trial — the one the
    sequential reference would have raised first — on every rank."""
    for r in records:
        if r[3] == _FAILED:
            raise r[5]
    return records


def _gather(dist, world, mine, group=None):
    if dist is not None and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine, group=group)
        return [r for part in gathered for r in part]
    return list(mine)


def _pop_es(session, space, budget, seed, lam, rank, world, dist, group=None):
    """(1+λ)-ES (an extension of search.py:226-234,261-279).

    Each generation draws λ children of the current parent with the
    reference's ``_mutate`` from one ``random.Random(seed)`` stream, trial
    indices ``1 + g·λ + j``; children are evaluated on ranks ``idx % world``
    and exchanged with one all_gather per generation; the parent moves to
    the best evaluated child (lowest (cost, idx)) on strict improvement.
    Every rank holds the same parent, so the log does not depend on the
    world size, and λ = 1 is exactly the reference's (1+1)-ES.
    """
    from staircase.tuner.search import _mutate
    from staircase.tuner.space import Trial

    identity = space.identity()
    records = _raise_first(_gather(dist, world, [
        _guarded(session, 0, identity["tiles"], identity["unroll"], world)]
        if rank == 0 else [], group))
    log = [Trial(i, p, c, s, sd, stats=st) for i, p, c, s, sd, st in records]
    rng = random.Random(seed)
    parent, parent_cost = dict(log[0].params), log[0].cost
    idx = 1
    while idx < budget:
        kids = [(idx + j, _mutate(space, parent, rng)) for j in range(min(lam, budget - idx))]
        mine = [_guarded(session, i, tiles, unroll, world)
                for i, (tiles, unroll) in kids if i % world == rank]
        gen = _raise_first(sorted(_gather(dist, world, mine, group), key=lambda r: r[0]))
        gen = [Trial(i, p, c, s, sd, stats=st) for i, p, c, s, sd, st in gen]
        log.extend(gen)
        evaluated = [t for t in gen if t.status == "evaluated"]
        if evaluated:
            top = min(evaluated, key=lambda t: (t.cost, t.idx))
            if top.cost < parent_cost:
                parent, parent_cost = dict(top.params), top.cost
        idx += len(kids)
    evaluated = [t for t in log if t.status == "evaluated"]
    best = min(evaluated, key=lambda t: (t.cost, t.idx))
    return best, log


def _record(t):
    return (t.idx, t.params, t.cost, t.status, t.seed, t.stats)


def _es(session, space, budget, seed):
    """(1+1)-ES exactly as search.py:261-279."""
    from staircase.tuner.search import _mutate

    identity = space.identity()
    log = [session.trial(0, identity["tiles"], identity["unroll"])]
    rng = random.Random(seed)
    parent = dict(log[0].params)
    parent_cost = log[0].cost
    for idx in range(1, budget):
        tiles, unroll = _mutate(space, parent, rng)
        trial = session.trial(idx, tiles, unroll)
        log.append(trial)
        if trial.status == "evaluated" and trial.cost < parent_cost:
            parent = dict(trial.params)
            parent_cost = trial.cost
    evaluated = [t for t in log if t.status == "evaluated"]
    best = min(evaluated, key=lambda t: (t.cost, t.idx))
    return best, log


__all__ = ["search"]
