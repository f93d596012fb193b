"""CPU checks of the CLI wrapper (python -m paper_2307_16080_b200).

Non-executing subcommands (verify, opt) must behave exactly like the
reference CLI, and the wrapper must install the B200 engine as
machine._engine and honour --precision.  Execution itself is covered on the
B200 by tests/test_gpu_cli.py.
"""
import contextlib
import io
import os

import corpus


def _run(main, argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_verify_and_opt_match_reference(tmp_path):
    import paper_2307_16080_b200 as b2
    import paper_2307_16080_b200.__main__ as ours
    from staircase import cli
    from staircase.interp import machine
    from staircase.textio import print_module

    sir = os.path.join(str(tmp_path), "k.sir")
    with open(sir, "w") as fh:
        fh.write(print_module(corpus.conv_f32.module))
    saved = machine._engine
    try:
        for argv in (["verify", "--input", sir],
                     ["opt", "--input", sir, "--pipeline",
                      "scf-parallel-loop-tiling{sizes=4,4}"],
                     ["run", "--input", sir]):   # argparse error: exit code 2
            assert _run(ours.main, list(argv)) == _run(cli.main, list(argv))
        rc, _, _ = _run(ours.main, ["--precision", "bf16", "verify", "--input", sir])
        assert rc == 0
        assert machine._engine is b2.engine
        assert b2.engine.PRECISION == "bf16"
    finally:
        machine._engine = saved
        b2.configure(precision="exact")


def test_device_mode_argument_rewrite():
    """`run --mode b200[:precision]` maps to the reference's
    sequential mode with the engine's precision set; other modes untouched."""
    from paper_2307_16080_b200.__main__ import _device_mode

    assert _device_mode(["run", "--mode", "b200", "--func", "f"], "exact") == (
        ["run", "--mode", "sequential", "--func", "f"], "exact")
    assert _device_mode(["run", "--mode=b200:bf16"], "exact") == (
        ["run", "--mode", "sequential"], "bf16")
    assert _device_mode(["run", "--mode", "worksharing:2"], "tf32") == (
        ["run", "--mode", "worksharing:2"], "tf32")
