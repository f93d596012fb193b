"""The sharded sweep on the B200 engine reproduces the reference tuner's log.

Trial costs come from the exact tally and the guard compares every output
(rel 1e-6), so the log (idx, params, cost, status, seed) must equal the
reference's own ``tuner.search`` run on the C oracle engine.
"""
import pytest

import corpus
import oracle
from test_sweep import _ref, _space

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fn,strategy", [(corpus.conv_small, "random"),
                                         (corpus.conv_rows, "random"),
                                         (corpus.matmul_par, "es")])
def test_sweep_on_b200_equals_reference(fn, strategy):
    from paper_2307_16080_b200 import sweep

    oracle.build()
    best_r, log_r = _ref(fn.module, 12, 11, strategy)
    best, log = sweep.search(fn.module, None, _space(), budget=12, seed=11, strategy=strategy,
                             rank=0, world=1)
    assert log == log_r
    assert best == best_r


def test_population_es_on_b200_equals_its_definition():
    from paper_2307_16080_b200 import sweep
    from test_sweep import _pop_es_spec

    oracle.build()
    best, log = sweep.search(corpus.conv_small.module, None, _space(), budget=17, seed=6,
                             strategy="population_es", lam=8, rank=0, world=1)
    assert log == _pop_es_spec(corpus.conv_small.module, 17, 6, 8)
    assert best.cost <= log[0].cost


def test_device_objective_sees_the_tile_choice():
    """objective="device": costs are device milliseconds of each trial's
    launch sequence; the log's statuses and params equal the model run's
    (same guard, same skips), and the tile sizes, which select the CTA tile
    of the exact GEMM, show up as different costs."""
    import bench_kernels as bk
    from staircase.tuner import ParamSpace

    from paper_2307_16080_b200 import sweep

    space = ParamSpace(tile_sizes=([1, 8, 32], [1, 8, 32]), unroll_factors=[1])
    kw = dict(budget=10, seed=0, strategy="grid", rank=0, world=1)
    _, log_m = sweep.search(bk.mm_par1024.module, None, space, **kw)
    best, log_d = sweep.search(bk.mm_par1024.module, None, space, objective="device", **kw)
    assert [(t.idx, t.params, t.status) for t in log_d] == \
        [(t.idx, t.params, t.status) for t in log_m]
    costs = [t.cost for t in log_d if t.status == "evaluated"]
    assert all(0 < c < 1e3 for c in costs)
    # 2 * 1024^3 flops at >= 5 TFLOP/s: well under a millisecond each
    assert min(costs) < 0.5
    assert best.cost == min(costs)
    assert len({round(c, 2) for c in costs}) > 1


@pytest.mark.parametrize("fn", [corpus.conv_rows, corpus.matmul_par, corpus.linear32])
def test_resident_trials_equal_host_copied_trials(fn, monkeypatch):
    """Trials that start from device clones of the resident inputs produce the
    log of trials that copy and upload their inputs (the reference's
    _copy_args), including the baseline and the guard's verdicts."""
    from staircase.tuner import ParamSpace

    from paper_2307_16080_b200 import sweep

    space = ParamSpace(tile_sizes=([1, 2, 4, 8],) * 2, unroll_factors=[1, 2])
    kw = dict(budget=12, seed=3, strategy="grid", rank=0, world=1)
    monkeypatch.setattr(sweep, "RESIDENT", False)
    _, host_log = sweep.search(fn.module, None, space, **kw)
    monkeypatch.setattr(sweep, "RESIDENT", True)
    _, dev_log = sweep.search(fn.module, None, space, **kw)
    assert dev_log == host_log


def test_guard_failure_raises_the_reference_error(monkeypatch):
    """Resident trials (device clones, guard on the device): a baseline that
    no trial can match must raise the reference's StaircaseError."""
    from staircase.errors import StaircaseError
    from staircase.tuner import ParamSpace

    from paper_2307_16080_b200 import sweep

    orig = sweep._session_class

    def patched():
        S, ref = orig()

        class Perturbed(S):
            def __init__(self, *a, **k):
                super().__init__(*a, **k)
                w = self.want_args[-1]               # the baseline output, one element
                ent = sweep._WANT_DEV.get(id(w))
                if ent is not None:                  # kept on the device (resident)
                    ent[1].view(-1)[0] += 1.0
                else:
                    w.data[0] += 1.0

        return Perturbed, ref

    monkeypatch.setattr(sweep, "_session_class", patched)
    space = ParamSpace(tile_sizes=([1, 2, 4],) * 2, unroll_factors=[1, 2])
    with pytest.raises(StaircaseError, match="changed the results"):
        sweep.search(corpus.matmul_par.module, None, space, budget=6, seed=0,
                     strategy="grid", rank=0, world=1)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_native_guard_is_math_isclose(dtype):
    """b200_guard_close counts exactly the elements math.isclose(g, w,
    rel_tol=1e-6, abs_tol=1e-9) rejects (reference tuner/search.py:128-138),
    special values included."""
    import ctypes
    import math

    import numpy as np
    import torch

    from paper_2307_16080_b200 import runtime

    inf, nan = float("inf"), float("nan")
    pairs = [(1.0, 1.0), (1.0, 1.0 + 1e-7), (1.0, 1.0 + 1e-5), (0.0, 5e-10), (0.0, 2e-9),
             (-0.0, 0.0), (inf, inf), (-inf, inf), (inf, 1e308), (nan, nan), (nan, 1.0),
             (1e30, 1e30 * (1 + 5e-7)), (1e30, 1e30 * (1 + 2e-6)), (-3.5, -3.5), (2.0, -2.0)]
    rng = np.random.default_rng(1)
    extra = rng.uniform(-2, 2, 2000)
    pairs += [(float(v), float(v) * (1 + d)) for v, d in zip(extra, rng.uniform(-3e-6, 3e-6,
                                                                          2000))]
    npdt = np.float32 if dtype == "f32" else np.float64
    g = np.array([p[0] for p in pairs], dtype=npdt)
    w = np.array([p[1] for p in pairs], dtype=npdt).astype(np.float64)
    want_bad = sum(not math.isclose(float(a), float(b), rel_tol=1e-6, abs_tol=1e-9)
                   for a, b in zip(g.astype(np.float64), w))
    tg, tw = torch.from_numpy(g).cuda(), torch.from_numpy(w).cuda()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    P = ctypes.c_void_p
    rc = runtime.load_library().b200_guard_close(
        0 if dtype == "f32" else 1, P(tg.data_ptr()), P(tw.data_ptr()), tg.numel(), 1e-6, 1e-9,
        P(bad.data_ptr()), P(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    assert int(bad.item()) == want_bad > 0
