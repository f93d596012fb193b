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
