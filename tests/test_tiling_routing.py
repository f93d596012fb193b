"""Tiled matmul / Linear nests are strided GEMMs, and their tile sizes pick the CTA tile (CPU).

The reference's tiling pass rewrites every tiled index as origin + offset
(reference passes/tiling.py:56-80), so a tiled matmul's output loops are two
variables each.  templates.match_contraction must merge each pair back into
one strided dimension (so the nest runs on the strided GEMM kernels — the
tensor cores at bf16 / tf32), report the tile sizes, and runtime.cta_tile
must turn those into a CTA tile shape.  Reference tile sizes: (8, 8) and
(4, 16) (reference SPEC.md:778).
"""
import pytest

import corpus
import harness
from vm_sim import SimEngine


def _matches(fn, pipe, monkeypatch):
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


@pytest.mark.parametrize("pipe,tiles", [(None, (None, None)), (harness.TILE88, (8, 8)),
                                        (harness.TILE416, (4, 16)),
                                        (harness.TILE88_U3, (8, 8))])
def test_tiled_matmul_is_strided(pipe, tiles, monkeypatch):
    # corpus.matmul_par: C(32 x 64) += A(32 x 48) . B(48 x 64), parallel (i, k), j reduction
    (g,) = _matches(corpus.matmul_par, pipe, monkeypatch)
    assert g.strided, g
    assert (g.M, g.N, g.K) == (32, 64, 48)
    assert tuple(g.sA) == (48, 1) and tuple(g.sB) == (64, 1) and tuple(g.sC) == (64, 1)
    assert (g.offA, g.offB, g.offC) == (0, 0, 0)
    assert g.tiles == tiles


def test_tiled_parallel_linear_is_strided(monkeypatch):
    import bench_kernels as bk

    fn = bk.make_linear_stack(64)
    pipe = harness._spec("scf-parallel-loop-tiling{sizes=[4, 16]}")
    gs = _matches(fn, pipe, monkeypatch)
    assert len(gs) == 2
    for g in gs:
        assert g.strided and g.tiles == (4, 16)
    assert [(g.M, g.N, g.K) for g in gs] == [(64, 4096, 1024), (64, 1024, 4096)]


def test_cta_tile_mapping():
    from paper_2307_16080_b200.runtime import cta_tile

    assert cta_tile("exact", (None, None)) is None
    assert cta_tile("bf16", None) is None
    assert cta_tile("exact", (8, 8)) == (128, 128)
    assert cta_tile("exact", (4, 16)) == (64, 256)
    assert cta_tile("exact", (16, 4)) == (256, 64)
    assert cta_tile("exact", (2, 2)) == (64, 64)
    assert cta_tile("exact", (None, 8)) == (64, 64)      # (1, 8): area 8
    assert cta_tile("exact", (None, 32)) == (64, 256)
    assert cta_tile("bf16", (8, 8)) == (256, 256)
    assert cta_tile("tf32", (4, 16)) == (128, 256)
    assert cta_tile("bf16", (16, 4)) == (256, 256)


def test_irregular_tiles_stay_table_addressed(monkeypatch):
    """A conv's output groups are not one progression in A (input rows are
    wider than output rows), so they keep the tables / conv path."""
    (g,) = _matches(corpus.conv_f32, harness.TILE88, monkeypatch)
    assert not g.strided


@pytest.mark.parametrize("sizes", ["[8, 8]", "[4, 16]"])
def test_tiled_linear_stack_fuses_fill_and_bias(sizes):
    """Tiled fill / bias nests still fuse into the contractions (fusion._bias
    sees the origin + offset map dims as one progression per GEMM dim), and
    the result stays bit-identical to the oracle (pinned to the reference)."""
    import bench_kernels as bk
    from paper_2307_16080_b200 import engine

    fn = bk.make_linear_stack(8)
    pipe = harness._spec(f"scf-parallel-loop-tiling{{sizes={sizes}}}")
    sim = SimEngine()
    _, got, tally, _ = harness.run_engine(sim, fn, pipe, "sequential", 2)
    plan = engine.last_plan
    kinds = [p[0] for p in plan]
    assert kinds.count("contract_exact") == 2 and len(kinds) == 2, plan
    assert all(set(p[4]) >= {"fill", "bias"} for p in plan), plan
    import oracle

    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, pipe, "sequential", 2)
    assert tally == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()
