"""Pipelined host copies (runtime.Staging.stream_rows) leave results unchanged.

Large first-use contractions and convs are split into row / image panels
whose uploads, kernels and write-backs overlap (engine.STREAM_IO).  With the
size thresholds lowered, test-size plans run as several panels; every buffer
and the tally must equal the unstreamed run's bit for bit (and the C
oracle's on the exact path), including a GEMM whose output a later,
unfused region modifies (the streamed write-back must not be final there).
"""
import pytest

import bench_kernels as bk
import harness
import oracle

pytestmark = pytest.mark.gpu

GEMM_THEN_VM = '''
@staged
def gemm_then_vm(A: MemRef[(512, 64), F32], B: MemRef[(64, 96), F32],
                 C: MemRef[(512, 96), F32]):
    for i in range(512):
        for k in range(64):
            for j in range(96):
                C[i, j] = C[i, j] + A[i, k] * B[k, j]
    for i in range(96):
        for j in range(i):
            C[i, j] = C[j, i] + C[i, j]
'''


# a streamed GEMM whose output is rewritten by later regions: a map over all
# of C and a second contraction into C (neither waits for the first one's
# streamed write-back; flush() copies C again after it)
GEMM_THEN_REWRITE = '''
@staged
def gemm_then_rewrite(A: MemRef[(512, 64), F32], B: MemRef[(64, 128), F32],
                      C: MemRef[(512, 128), F32]):
    for i in range(512):
        for k in range(64):
            for j in range(128):
                C[i, j] = C[i, j] + A[i, k] * B[k, j]
    for i, j in parallel((0, 0), (512, 128)):
        C[i, j] = C[i, j] * constant(0.5, F32)
    for i in range(512):
        for k in range(64):
            for j in range(128):
                C[i, j] = C[i, j] + A[i, k] * B[k, j]
'''


def _gemm_then_vm():
    return bk._capture_from_source(GEMM_THEN_VM, "gemm_then_vm", {}, "stream")


def _run(fn, precision, stream, monkeypatch, pipeline=None):
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import engine, runtime

    monkeypatch.setattr(runtime, "STREAM_MIN_BYTES", 1)
    monkeypatch.setattr(runtime, "STREAM_PANEL_BYTES", 1 << 12)
    with engine.using(precision=precision, stream_io=stream):
        _, bufs, tally, _ = harness.run_engine(b2.engine, fn, pipeline, "sequential", 5)
    return bufs, tally, list(engine.last_plan), engine.last_staging.panels


CASES = [("mm1024", "exact"), ("mm1024", "bf16"), ("ls512", "exact"), ("ls512", "bf16"),
         ("conv4", "exact"), ("conv4", "bf16"), ("gemm_then_vm", "exact"), ("saxpy", "exact"),
         ("fill_then_scale", "exact"), ("gemm_then_rewrite", "exact"),
         ("gemm_then_rewrite", "bf16")]

FILL_THEN_SCALE = '''
@staged
def fill_then_scale(x: MemRef[(256, 512), F32], y: MemRef[(256, 512), F32]):
    for i, j in parallel((0, 0), (256, 512)):
        y[i, j] = constant(1.5, F32)
    for i, j in parallel((0, 0), (256, 512)):
        y[i, j] = y[i, j] * x[i, j]
'''

SAXPY = '''
@staged
def saxpy_s(x: MemRef[(512, 1024), F32], y: MemRef[(512, 1024), F32]):
    for i, j in parallel((0, 0), (512, 1024)):
        y[i, j] = y[i, j] + x[i, j] * constant(2.0, F32)
'''



def _fn(name):
    return {"mm1024": lambda: bk.mm_par1024, "ls512": lambda: bk.make_linear_stack(512),
            "conv4": lambda: bk.make_conv(4), "gemm_then_vm": _gemm_then_vm,
            "saxpy": lambda: bk._capture_from_source(SAXPY, "saxpy_s", {}, "stream"),
            "gemm_then_rewrite": lambda: bk._capture_from_source(
                GEMM_THEN_REWRITE, "gemm_then_rewrite", {}, "stream"),
            "fill_then_scale": lambda: bk._capture_from_source(FILL_THEN_SCALE,
                                                               "fill_then_scale", {},
                                                               "stream")}[name]()


@pytest.mark.parametrize("name,precision", CASES)
def test_streamed_equals_unstreamed(name, precision, monkeypatch):
    fn = _fn(name)
    want, t_want, plan_want, panels0 = _run(fn, precision, False, monkeypatch)
    got, t_got, plan_got, panels = _run(fn, precision, True, monkeypatch)
    assert panels0 == 0 and panels >= 2, (panels0, panels)
    assert plan_got == plan_want
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()


@pytest.mark.parametrize("name", ["gemm_then_vm", "gemm_then_rewrite"])
def test_streamed_write_back_before_a_later_writer_matches_the_oracle(name, monkeypatch):
    fn = _fn(name)
    got, t_got, plan, panels = _run(fn, "exact", True, monkeypatch)
    assert panels >= 2 and plan[0][0] == "gemm_f32_exact", plan
    if name == "gemm_then_vm":
        assert plan[-1][0] == "vm", plan
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", 5)
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()


@pytest.mark.parametrize("shape", [None, "4,2,3,1", "2,2,2,3", "4,2,3,5"])
@pytest.mark.parametrize("name", ["mm1024", "ls512"])
def test_block_streamed_exact_gemm_equals_row_panels(name, shape, monkeypatch):
    """The exact GEMM streamed in (row, column) blocks and K slices (B by
    column panels, runtime._gemm_streamed_2d; shape = row panels, column
    panels, streams, K slices) equals the row-panel pipeline and the
    unstreamed run bit for bit, tally included — init, fill and bias only on
    a block's first / last K slice."""
    from paper_2307_16080_b200 import runtime

    if shape:
        monkeypatch.setenv("B200_STREAM_2D_SHAPE", shape)
    fn = _fn(name)
    want, t_want, plan_want, _ = _run(fn, "exact", False, monkeypatch)
    monkeypatch.setattr(runtime, "STREAM_2D", False)
    rows, t_rows, _, p_rows = _run(fn, "exact", True, monkeypatch)
    monkeypatch.setattr(runtime, "STREAM_2D", True)
    blocks, t_blocks, plan, p_blocks = _run(fn, "exact", True, monkeypatch)
    assert p_rows >= 2 and p_blocks >= 2
    assert plan == plan_want and t_blocks == t_rows == t_want
    for g, r, w in zip(blocks, rows, want):
        assert g.data.tobytes() == r.data.tobytes() == w.data.tobytes()


@pytest.mark.parametrize("tiles", ["tile88", "tile416"])
def test_block_streamed_tiled_gemm_uses_its_cta_tile(tiles, monkeypatch):
    """A reference-tiled matmul streamed in blocks runs each block on the CTA
    tile its tile sizes select (plan label), bit-identical to the unstreamed
    run, tally included."""
    fn = _fn("mm1024")
    pipe = {"tile88": harness.TILE88, "tile416": harness.TILE416}[tiles]
    want, t_want, plan_want, _ = _run(fn, "exact", False, monkeypatch, pipe)
    got, t_got, plan, panels = _run(fn, "exact", True, monkeypatch, pipe)
    assert panels >= 2 and plan == plan_want and t_got == t_want, (plan, plan_want)
    assert ("cta64x256" if tiles == "tile416" else "cta128x128") in str(plan), plan
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()
