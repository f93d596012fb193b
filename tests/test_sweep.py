"""Sharded design-space sweep: logs equal the reference tuner's (CPU, gloo).

The reference ``staircase.tuner.search`` (tuner/search.py:237-279) is the
ground truth: for the same kernel, space, seed, budget and strategy the
sharded sweep must return an identical log (Trial equality: idx, params,
cost, status, seed) and the same best trial, for world sizes 1 and 2
(torch.distributed gloo on 127.0.0.1).  On CPU the trials run on the C
oracle engine; tests/test_gpu_sweep.py repeats this on the B200 engine.
"""
import os
import socket
import tempfile

import pytest

import conftest  # noqa: F401  (spawned workers re-import this module: shim first)
import corpus
import oracle

SPACE_ARGS = dict(tile_sizes=([1, 2, 4, 8, 16], [1, 2, 4, 8, 16]), unroll_factors=(1, 2, 4))


def _space():
    from staircase.tuner import ParamSpace

    return ParamSpace(**SPACE_ARGS)


def _ref(kernel, budget, seed, strategy):
    from staircase.interp import machine
    from staircase.tuner import search

    saved = machine._engine
    machine._engine = oracle
    try:
        return search(kernel, None, _space(), budget=budget, seed=seed, strategy=strategy)
    finally:
        machine._engine = saved


@pytest.mark.parametrize("strategy", ["random", "es"])
def test_world1_equals_reference(strategy):
    from paper_2307_16080_b200 import sweep

    oracle.build()
    kernel = corpus.conv_small.module
    best_r, log_r = _ref(kernel, 10, 7, strategy)
    best, log = sweep.search(kernel, None, _space(), budget=10, seed=7, strategy=strategy,
                             engine=oracle, rank=0, world=1)
    assert log == log_r
    assert best == best_r


def test_grid_strategy_enumerates_the_space_in_order():
    from paper_2307_16080_b200 import sweep

    oracle.build()
    best, log = sweep.search(corpus.conv_small.module, None, _space(), budget=6, seed=0,
                             strategy="grid", engine=oracle, rank=0, world=1)
    assert [t.params["tiles"] for t in log] == [[1, 1], [1, 1], [1, 1], [1, 1], [1, 2], [1, 2]]
    assert [t.params["unroll"] for t in log] == [1, 1, 2, 4, 1, 2]
    assert best.cost <= log[0].cost


def _worker(rank, world, port, out_dir, budget, seed, strategy="random", lam=8):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import conftest  # noqa: F401  (path + staircase shim)
    import torch.distributed as dist

    import corpus as c
    import oracle as o
    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace
    from staircase.tuner.log import persist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        best, log = sweep.search(c.conv_small.module, None, ParamSpace(**SPACE_ARGS),
                                 budget=budget, seed=seed, strategy=strategy, engine=o, lam=lam)
        persist(log, os.path.join(out_dir, f"log{rank}.jsonl"))
        with open(os.path.join(out_dir, f"best{rank}.txt"), "w") as fh:
            fh.write(f"{best.idx} {best.cost}")
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_world2_gloo_log_equals_reference():
    import torch.multiprocessing as mp
    from staircase.tuner.log import load

    oracle.build()
    budget, seed = 12, 3
    best_r, log_r = _ref(corpus.conv_small.module, budget, seed, "random")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, budget, seed), nprocs=2, join=True)
        for rank in range(2):
            log = load(os.path.join(d, f"log{rank}.jsonl"))
            assert log == log_r
            idx, cost = open(os.path.join(d, f"best{rank}.txt")).read().split()
            assert int(idx) == best_r.idx and float(cost) == best_r.cost


def test_guard_predicate_is_math_isclose():
    """The vectorised guard (numpy and torch forms) agrees with the reference's
    math.isclose(g, w, rel_tol=1e-6, abs_tol=1e-9) on edge values."""
    import math

    import numpy as np
    import torch

    from paper_2307_16080_b200.sweep import _close_tensors

    inf, nan = float("inf"), float("nan")
    vals = [0.0, -0.0, 1e-10, -1e-10, 5e-10, 1.0, 1.0 + 1e-7, 1.0 + 3e-6, -1.0, 3.4e38,
            1e-300, inf, -inf, nan]
    g = [a for a in vals for _ in vals]
    w = [b for _ in vals for b in vals]
    want = [math.isclose(a, b, rel_tol=1e-6, abs_tol=1e-9) for a, b in zip(g, w)]
    with np.errstate(invalid="ignore", over="ignore"):
        got_np = _close_tensors(np.array(g), np.array(w)).tolist()
    got_t = _close_tensors(torch.tensor(g, dtype=torch.float64),
                           torch.tensor(w, dtype=torch.float64)).tolist()
    assert got_np == want
    assert got_t == want


def _pop_es_spec(kernel, budget, seed, lam):
    """(1+λ)-ES written directly on the reference's _Session (sequential)."""
    import random
    import sys

    from staircase.interp import machine

    ref = sys.modules["staircase.tuner.search"]

    saved = machine._engine
    machine._engine = oracle
    try:
        session = ref._Session(kernel, func=None, seed=seed, objective="model",
                               pipeline_template=None)
        space = _space()
        ident = space.identity()
        log = [session.trial(0, ident["tiles"], ident["unroll"])]
        rng = random.Random(seed)
        parent, pcost = dict(log[0].params), log[0].cost
        while len(log) < budget:
            n = min(lam, budget - len(log))
            pts = [ref._mutate(space, parent, rng) for _ in range(n)]
            gen = [session.trial(len(log) + j, t, u) for j, (t, u) in enumerate(pts)]
            log += gen
            ok = [t for t in gen if t.status == "evaluated"]
            if ok:
                top = min(ok, key=lambda t: (t.cost, t.idx))
                if top.cost < pcost:
                    parent, pcost = dict(top.params), top.cost
        return log
    finally:
        machine._engine = saved


def test_population_es_lambda1_is_the_reference_one_plus_one_es():
    from paper_2307_16080_b200 import sweep

    oracle.build()
    kernel = corpus.conv_small.module
    best_r, log_r = _ref(kernel, 10, 5, "es")
    best, log = sweep.search(kernel, None, _space(), budget=10, seed=5,
                             strategy="population_es", lam=1, engine=oracle, rank=0, world=1)
    assert log == log_r
    assert best == best_r


def test_population_es_follows_its_definition():
    from paper_2307_16080_b200 import sweep

    oracle.build()
    kernel = corpus.conv_small.module
    best, log = sweep.search(kernel, None, _space(), budget=11, seed=2,
                             strategy="1+lambda-es", lam=4, engine=oracle, rank=0, world=1)
    assert [t.idx for t in log] == list(range(11))
    assert log == _pop_es_spec(kernel, 11, 2, 4)
    assert best.cost <= log[0].cost
    with pytest.raises(ValueError):
        sweep.search(kernel, None, _space(), budget=3, strategy="population_es", lam=0,
                     engine=oracle, rank=0, world=1)


def test_population_es_world2_gloo_equals_world1():
    import torch.multiprocessing as mp
    from staircase.tuner.log import load

    from paper_2307_16080_b200 import sweep

    oracle.build()
    budget, seed = 13, 4
    best1, log1 = sweep.search(corpus.conv_small.module, None, _space(), budget=budget,
                               seed=seed, strategy="population_es", lam=4, engine=oracle,
                               rank=0, world=1)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, budget, seed, "population_es", 4),
                 nprocs=2, join=True)
        for rank in range(2):
            assert load(os.path.join(d, f"log{rank}.jsonl")) == log1
            idx, cost = open(os.path.join(d, f"best{rank}.txt")).read().split()
            assert int(idx) == best1.idx and float(cost) == best1.cost


def _failing_template(tiles, unroll):
    """A pipeline template that fails on two grid points (idx 3 and 6 of the
    grid over SPACE_ARGS) — the sharded search must raise the idx-3 error on
    every rank instead of leaving a rank blocked in the all-gather."""
    from staircase.tuner.search import default_pipeline

    if (list(tiles), unroll) in (([1, 1], 4), ([1, 2], 4)):
        raise RuntimeError(f"template failure at tiles={list(tiles)} unroll={unroll}")
    return default_pipeline(tiles, unroll)


def _fail_worker(rank, world, port, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import conftest  # noqa: F401
    import torch.distributed as dist

    import corpus as c
    import oracle as o
    import test_sweep as ts
    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        try:
            sweep.search(c.conv_small.module, ts._failing_template, ParamSpace(**SPACE_ARGS),
                         budget=10, seed=0, strategy="grid", engine=o)
            msg = "no error"
        except RuntimeError as exc:
            msg = str(exc)
        with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()


def test_world2_trial_error_raises_on_every_rank():
    import torch.multiprocessing as mp

    oracle.build()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_fail_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        msgs = [open(os.path.join(d, f"err{r}.txt")).read() for r in range(2)]
    first = "template failure at tiles=[1, 1] unroll=4"
    assert msgs == [first, first]
    # the sequential search raises the same error
    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace

    with pytest.raises(RuntimeError, match=r"tiles=\[1, 1\] unroll=4"):
        sweep.search(corpus.conv_small.module, _failing_template, ParamSpace(**SPACE_ARGS),
                     budget=10, seed=0, strategy="grid", engine=oracle)


@pytest.mark.parametrize("fn", [corpus.conv_small, corpus.matmul_par, corpus.int_ops,
                                corpus.scalar_args, corpus.linear32])
@pytest.mark.parametrize("seed", [0, 3, 12345])
def test_fast_make_inputs_is_the_reference_stream(fn, seed):
    """sweep.make_inputs draws the float memrefs with numpy from the same
    Mersenne Twister state: every argument bit-identical to the reference's
    make_inputs (tuner/search.py:78-102), including what follows them."""
    from paper_2307_16080_b200 import sweep
    from staircase.interp import Buffer
    from staircase.tuner.search import make_inputs

    want = make_inputs(fn.module, fn.__name__, seed)
    got = sweep.make_inputs(fn.module, fn.__name__, seed)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        if isinstance(w, Buffer):
            assert (g.shape, g.dtype) == (w.shape, w.dtype)
            assert g.data.tobytes() == w.data.tobytes()
        else:
            assert type(g) is type(w) and g == w


def test_device_objective_needs_the_b200_engine():
    """objective="device" times the B200 engine's recorded kernels; any other
    engine is refused up front (like the reference's unknown-objective check)."""
    from vm_sim import SimEngine

    from paper_2307_16080_b200 import sweep

    with pytest.raises(ValueError, match="device"):
        sweep.search(corpus.conv_small.module, None, _space(), budget=2, seed=0,
                     objective="device", engine=SimEngine(), rank=0, world=1)
    with pytest.raises(ValueError, match="objective"):
        sweep.search(corpus.conv_small.module, None, _space(), budget=2, seed=0,
                     objective="cycles", engine=SimEngine(), rank=0, world=1)


def test_rank_groups():
    from paper_2307_16080_b200.sweep import rank_groups

    assert rank_groups([1, 1], 1) == [[0], [0]]
    assert rank_groups([1, 1], 2) == [[0], [1]]
    assert rank_groups([1, 1], 3) == [[0, 1], [2]]
    assert rank_groups([1, 1], 8) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert rank_groups([5, 3], 8) == [[0, 1, 2, 3, 4], [5, 6, 7]]
    assert rank_groups([1, 100], 4) == [[0], [1, 2, 3]]
    assert rank_groups([1, 1, 1], 2) == [[0], [1], [0]]
    for w in range(1, 12):
        for wts in ([1, 1], [3, 1], [1, 2, 3]):
            g = rank_groups(wts, w)
            assert all(g) and all(0 <= r < w for grp in g for r in grp)
            if w >= len(wts):
                assert sorted(r for grp in g for r in grp) == list(range(w))


def _many_worker(rank, world, port, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import conftest  # noqa: F401  (path + staircase shim)
    import torch.distributed as dist

    import corpus as c
    import oracle as o
    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace
    from staircase.tuner.log import persist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        res = sweep.search_many([c.conv_small.module, c.conv_rows.module], None,
                                ParamSpace(**SPACE_ARGS), budget=10, seed=4, strategy="grid",
                                engine=o)
        for k, (best, log) in enumerate(res):
            persist(log, os.path.join(out_dir, f"log{rank}_{k}.jsonl"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_search_many_gloo_equals_single_searches(world):
    """Two kernels swept at once over 2 and 3 gloo ranks (one group per
    kernel; at 3 the first group shards its trials over two ranks): every
    rank returns each kernel's log exactly as a world-1 search of it."""
    import torch.multiprocessing as mp
    from staircase.tuner import ParamSpace
    from staircase.tuner.log import load

    from paper_2307_16080_b200 import sweep

    oracle.build()
    want = [sweep.search(m, None, ParamSpace(**SPACE_ARGS), budget=10, seed=4,
                         strategy="grid", engine=oracle, rank=0, world=1)[1]
            for m in (corpus.conv_small.module, corpus.conv_rows.module)]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_many_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for rank in range(world):
            for k in range(2):
                assert load(os.path.join(d, f"log{rank}_{k}.jsonl")) == want[k]


@pytest.mark.parametrize("native", [True, False])
def test_uniform_stream_is_pythons(native, monkeypatch):
    """make_inputs' float draws (native b200_mt_uniform, or the numpy
    fallback) equal [rng.uniform(-2, 2) ...] bit for bit across many twists,
    from odd start positions, and leave the generator in the same state."""
    import random

    import numpy as np

    from paper_2307_16080_b200 import sweep

    if not native:
        monkeypatch.setattr(sweep, "_native", lambda: None)
    r1, r2 = random.Random(7), random.Random(7)
    for n in (1, 311, 624, 1249, 20011):
        r1.random()
        r2.random()
        for dt in (np.float64, np.float32):
            got = sweep._uniform(r1, n, dt)
            want = np.array([r2.uniform(-2.0, 2.0) for _ in range(n)]).astype(dt)
            assert got.tobytes() == want.tobytes()
            assert r1.getstate() == r2.getstate()


def test_make_inputs_equals_reference():
    import importlib

    from paper_2307_16080_b200 import sweep

    ref = importlib.import_module("staircase.tuner.search")
    for fn in (corpus.conv_small, corpus.matmul_par, corpus.int_ops, corpus.scalar_args,
               corpus.linear32):
        for seed in (0, 9):
            got, want = sweep.make_inputs(fn.module, None, seed), ref.make_inputs(
                fn.module, None, seed)
            for g, w in zip(got, want):
                if hasattr(w, "data"):
                    assert (g.shape, g.strides, g.dtype) == (w.shape, w.strides, w.dtype)
                    assert g.data.tobytes() == w.data.tobytes()
                else:
                    assert g == w
