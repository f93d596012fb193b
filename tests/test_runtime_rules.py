"""Host-side routing rules of the runtime (CPU only): the tile -> CTA tile
map of tiled nests, row panels, and which convs the fused tensor-core kernel
takes."""
import types

import pytest


def test_cta_tile_map():
    from paper_2307_16080_b200.runtime import cta_tile

    assert cta_tile("exact", None) is None and cta_tile("bf16", (None, None)) is None
    # the reference tile sizes
    assert cta_tile("exact", (8, 8)) == (128, 128)
    assert cta_tile("exact", (4, 16)) == (64, 256)
    assert cta_tile("bf16", (8, 8)) == (256, 256)
    assert cta_tile("bf16", (4, 16)) == (128, 256)
    assert cta_tile("tf32", (16, 4)) == (256, 256)
    assert cta_tile("exact", (2, 2)) == (64, 64)
    assert cta_tile("exact", (32, 4)) == (256, 64)


def test_row_panels():
    from paper_2307_16080_b200.runtime import STREAM_MIN_BYTES, row_panels

    assert row_panels(4096, 16, 256) is None                      # too little traffic
    rows = 4096
    per_row = STREAM_MIN_BYTES // rows * 4
    p = row_panels(rows, per_row, 256)
    assert p[0][0] == 0 and p[-1][1] == rows and all(b - a > 0 for a, b in p)
    p8 = row_panels(rows, per_row, 256, count=8)
    assert len(p8) == 8 and all((b - a) % 256 == 0 for a, b in p8)
    assert len(row_panels(512, per_row * 8, 256, count=8)) == 2   # capped by rows / align


def _cv(**kw):
    d = dict(kw=3, kh=3, f=64, c=64, nb=8, hp=58, wp=58, ho=56, wo=56)
    d.update(kw)
    st = (d["c"] * d["hp"] * d["wp"], d["hp"] * d["wp"], d["wp"], 1)
    d.setdefault("inp", types.SimpleNamespace(strides=st))
    return types.SimpleNamespace(**d)


@pytest.mark.parametrize("kw,ok", [
    ({}, True), (dict(nb=9), False), (dict(f=128), False), (dict(kw=5, kh=5), False),
    (dict(c=100), False), (dict(hp=57, ho=55), False), (dict(wp=90, wo=88), False),
    (dict(c=48), True), (dict(f=32, nb=4), True),
])
def test_fused_conv_routing(kw, ok, monkeypatch):
    from paper_2307_16080_b200 import runtime

    monkeypatch.delenv("B200_CONV_UNFUSED", raising=False)
    assert runtime.conv_tc_fused_ok(_cv(**kw)) is ok
    monkeypatch.setenv("B200_CONV_UNFUSED", "1")
    assert runtime.conv_tc_fused_ok(_cv(**kw)) is False


def test_fused_conv_needs_dense_planes():
    import types as t

    from paper_2307_16080_b200 import runtime

    cv = _cv()
    cv.inp = t.SimpleNamespace(strides=(64 * 58 * 60, 58 * 60, 60, 1))   # padded rows
    assert runtime.conv_tc_fused_ok(cv) is False
