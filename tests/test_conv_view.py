"""templates.conv_view recognises tiled / unrolled conv nests (CPU).

The sweep's configurations tile the conv's parallel loops (passes/tiling.py:
index = origin + offset) and unroll its innermost reduction loop
(passes/unroll.py); each such nest is still conv_2d_nchw_fchw, so it must map
to the same ConvView (and run on the direct conv kernels) — with the
reduction roles in nest order, the order the kernels round in.  Nests that
are not a conv must not.
"""
import pytest

import harness
from vm_sim import SimEngine


def _capture_matches(fn, pipe, monkeypatch):
    from paper_2307_16080_b200 import engine, templates

    got = []
    orig = templates.match_contraction

    def wrap(*a, **k):
        g = orig(*a, **k)
        got.append(g)
        return g

    monkeypatch.setattr(engine.templates, "match_contraction", wrap)
    harness.run_engine(SimEngine(), fn, pipe, "sequential", 4)
    return [g for g in got if g is not None]


@pytest.mark.parametrize("sizes,unroll", [([1, 2, 8, 7], 3), ([1, 1, 2, 2], 3), ([2, 4], 1),
                                          ([1, 1, 4, 4], 2), ([1, 1, 1, 1], 1)])
def test_tiled_conv_is_a_conv(sizes, unroll, monkeypatch):
    from staircase.tuner.search import default_pipeline

    import test_gpu_conv as tg
    from paper_2307_16080_b200 import templates

    fn = tg._conv_kernel(2, 16, 8, 16, 28, 3, 3)
    (g,) = _capture_matches(fn, default_pipeline(sizes, unroll), monkeypatch)
    cv = templates.conv_view(None, g, ("f32",))
    assert cv is not None
    assert (cv.nb, cv.c, cv.f, cv.ho, cv.wo, cv.kh, cv.kw) == (2, 16, 8, 16, 28, 3, 3)
    assert cv.k_order == ("ci", "ki", "kj")


def test_matmul_is_not_a_conv(monkeypatch):
    import corpus
    from paper_2307_16080_b200 import templates

    for g in _capture_matches(corpus.matmul_par, None, monkeypatch):
        assert templates.conv_view(None, g, ("f32",)) is None


def test_single_channel_conv_is_a_conv(monkeypatch):
    """The paper's conv (1,1,1282,1282)*(1,1,3,3): N = C = F = 1, so those
    loops have trip 1 and carry no variable."""
    import bench_kernels as bk
    from paper_2307_16080_b200 import templates

    (g,) = _capture_matches(bk.conv_paper, None, monkeypatch)
    cv = templates.conv_view(None, g, ("f32",))
    assert cv is not None
    assert (cv.nb, cv.c, cv.f, cv.ho, cv.wo, cv.kh, cv.kw) == (1, 1, 1, 1280, 1280, 3, 3)


@pytest.mark.parametrize("rank,world,rows", [(0, 2, (0, 2)), (1, 2, (2, 4)), (3, 4, (3, 4)),
                                             (1, 3, (1, 2))])
def test_batch_shard_conv_is_a_conv(rank, world, rows, monkeypatch):
    """A batch shard (shard.py) restricts the conv's batch loop to rows
    [r0, r1): still conv_2d_nchw_fchw, over nb = r1 - r0 images from n0 = r0
    (a one-image shard has no batch variable left: n0 comes from the
    operands' base offsets)."""
    import corpus
    from paper_2307_16080_b200 import engine, shard, templates
    from vm_sim import SimBackend

    got = []
    orig = templates.match_contraction

    def wrap(*a, **k):
        g = orig(*a, **k)
        got.append(g)
        return g

    monkeypatch.setattr(engine.templates, "match_contraction", wrap)
    fn = corpus.conv_mid          # (4, 16, 34, 34) * (8, 16, 3, 3)
    shard.run(fn.module, fn.__name__, harness.make_args(fn, 0), rank=rank, world=world,
              backend=SimBackend())
    (g,) = [x for x in got if x is not None]
    cv = templates.conv_view(None, g, ("f32",))
    assert cv is not None
    assert (cv.n0, cv.nb, cv.c, cv.f, cv.ho, cv.wo) == (rows[0], rows[1] - rows[0], 16, 8, 32, 32)


@pytest.mark.parametrize("shape", [(16, 1, 5, 1, 1), (70, 1, 34, 1, 1), (16, 3, 1, 1, 1),
                                   (8, 1, 1, 1, 1), (16, 1, 1, 3, 3)])
def test_size_one_dimensions_are_still_a_conv(shape, monkeypatch):
    """One output row and a 1x1 filter make the input's channel and row
    strides equal (both W), so two roles share a coefficient signature; the
    variable still takes the role its index range fits (found by the
    extended random-shape run: these nests had fallen back to the exact
    contraction at bf16)."""
    import test_gpu_conv as tg
    from paper_2307_16080_b200 import templates

    c, ho, wo, kh, kw = shape
    fn = tg._conv_kernel(3, c, 64, ho, wo, kh, kw)
    (g,) = _capture_matches(fn, None, monkeypatch)
    cv = templates.conv_view(None, g, ("f32",))
    assert cv is not None
    assert (cv.nb, cv.c, cv.f, cv.ho, cv.wo, cv.kh, cv.kw) == (3, c, 64, ho, wo, kh, kw)
    assert cv.k_order[0] == "ci"
