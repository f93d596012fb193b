"""The device race recorder (races.record_region) on the B200 (-m gpu).

For parallels the static proof cannot clear — genuine races (a shared
accumulator, a shifted copy) and non-affine but data-independent indices
(y[i*i]) — check_races must return the reference recorder's exact conflict
list (interp/races.py:20-97: same triples, same order) WITHOUT running the
reference's simulation; indices computed from loaded data still fall back
to it.  The reference answer is computed here with the reference's own
check_races (baseline/_ref).
"""
import pytest

import harness
from test_races import _kernels, scatter_args, scatter_module

pytestmark = pytest.mark.gpu


def _reference(module, name, args):
    from staircase.interp.races import check_races

    return check_races(module, name, args)


@pytest.mark.parametrize("name", ["racy", "gather", "shift", "stencil"])
@pytest.mark.parametrize("seed", [3, 4])
def test_recorder_matches_reference(name, seed, monkeypatch):
    import staircase.interp.races as ref_races

    from paper_2307_16080_b200 import races

    fn = _kernels()[name]
    args = harness.make_args(fn, seed)
    want = _reference(fn.module, fn.__name__, args)
    monkeypatch.setattr(ref_races, "check_races",
                        lambda *a, **k: pytest.fail("fell back to the reference simulation"))
    got = races.check_races(fn.module, fn.__name__, args)
    assert got == want
    if name in ("racy", "shift"):
        assert got, "a racy kernel must report conflicts"


def test_recorder_large_racy_accumulate(monkeypatch):
    """A 2-D parallel accumulating into a handful of addresses: thousands of
    conflicts, emitted on the device and put back in the recorder's order."""
    import bench_kernels as bk
    import staircase.interp.races as ref_races

    from paper_2307_16080_b200 import races

    src = """
@staged
def acc2d(x: MemRef[(128, 48), F32], acc: MemRef[(6,), F32]):
    for i, j in parallel((0, 0), (128, 6)):
        acc[j] = acc[j] + x[i, j * 8]
"""
    fn = bk._capture_from_source(src, "acc2d", {}, "races_big")
    args = harness.make_args(fn, 2)
    want = _reference(fn.module, fn.__name__, args)
    assert len(want) > 1000
    monkeypatch.setattr(ref_races, "check_races",
                        lambda *a, **k: pytest.fail("fell back to the reference simulation"))
    assert races.check_races(fn.module, fn.__name__, args) == want


def test_data_dependent_scatter_falls_back():
    from paper_2307_16080_b200 import races

    got = races.check_races(scatter_module(), "scatter", scatter_args())
    assert got == _reference(scatter_module(), "scatter", scatter_args()) and got
