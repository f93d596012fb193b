"""The reference command line on the B200 engine (python -m paper_2307_16080_b200).

`staircase run` (reference staircase/cli.py:204-231) is executed twice on the
same .sir file and JSON argument files: once with the reference's own engine
(_evalcy) and once through ``paper_2307_16080_b200.__main__`` (the same CLI
with the B200 engine installed as machine._engine).  The written buffers
and results must be byte-identical, the stats JSON equal except wall_time,
and errors must give the same exit code and message.
"""
import contextlib
import io
import json
import os

import pytest

import corpus
import harness

pytestmark = pytest.mark.gpu


def _write_inputs(tmp, fn, seed):
    from staircase.interp import buffer_to_json
    from staircase.textio import print_module

    sir = os.path.join(tmp, "k.sir")
    with open(sir, "w") as fh:
        fh.write(print_module(fn.module))
    paths = []
    for i, a in enumerate(harness.make_args(fn, seed)):
        p = os.path.join(tmp, f"a{i}.json")
        with open(p, "w") as fh:
            fh.write(buffer_to_json(a) if hasattr(a, "data") else json.dumps(a))
        paths.append(p)
    return sir, paths


def _run(main, argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("fn,mode", [
    (corpus.matmul_96, "sequential"),
    (corpus.conv_f32, "worksharing:2"),
    (corpus.ewise_gpu, "gpu"),
    (corpus.oob_kernel, "sequential"),
], ids=["matmul", "conv-worksharing", "gpu-module", "out-of-bounds"])
def test_cli_run_matches_reference(tmp_path, fn, mode):
    import paper_2307_16080_b200.__main__ as ours
    from staircase import cli
    from staircase.interp import machine

    sir, args = _write_inputs(str(tmp_path), fn, seed=5)
    name = fn.__name__
    saved = machine._engine
    results = {}
    for tag, main in (("ref", cli.main), ("b200", ours.main)):
        outdir = os.path.join(str(tmp_path), tag)
        argv = ["run", "--input", sir, "--func", name, "--mode", mode, "--out", outdir,
                "--args", *args]
        try:
            results[tag] = _run(main, argv) + (outdir,)
        finally:
            machine._engine = saved
    (rc_r, out_r, err_r, dir_r), (rc_b, out_b, err_b, dir_b) = results["ref"], results["b200"]
    assert rc_b == rc_r
    assert err_b == err_r
    if rc_r != 0:
        return
    s_r, s_b = json.loads(out_r), json.loads(out_b)
    for s in (s_r, s_b):
        s.pop("wall_time")
        s["outputs"] = [os.path.basename(p) for p in s["outputs"]]
    assert s_b == s_r
    for f in sorted(os.listdir(dir_r)):
        assert open(os.path.join(dir_b, f)).read() == open(os.path.join(dir_r, f)).read(), f


def test_cli_run_device_mode_matches_reference(tmp_path):
    """`run --mode b200` writes what the reference's `run --mode sequential`
    writes (buffers byte-identical, stats equal but wall time)."""
    import paper_2307_16080_b200.__main__ as ours
    from staircase import cli
    from staircase.interp import machine

    fn = corpus.matmul_96
    sir, args = _write_inputs(str(tmp_path), fn, seed=7)
    saved = machine._engine
    results = {}
    for tag, main, mode in (("ref", cli.main, "sequential"), ("b200", ours.main, "b200")):
        outdir = os.path.join(str(tmp_path), tag)
        argv = ["run", "--input", sir, "--func", fn.__name__, "--mode", mode, "--out", outdir,
                "--args", *args]
        try:
            results[tag] = _run(main, argv) + (outdir,)
        finally:
            machine._engine = saved
    (rc_r, out_r, _, dir_r), (rc_b, out_b, _, dir_b) = results["ref"], results["b200"]
    assert rc_r == rc_b == 0
    s_r, s_b = json.loads(out_r), json.loads(out_b)
    for s in (s_r, s_b):
        s.pop("wall_time")
        s["outputs"] = [os.path.basename(p) for p in s["outputs"]]
    assert s_b == s_r
    for f in sorted(os.listdir(dir_r)):
        assert open(os.path.join(dir_b, f)).read() == open(os.path.join(dir_r, f)).read(), f
