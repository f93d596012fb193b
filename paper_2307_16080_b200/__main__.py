"""The reference's command line, executed on the B200 backend.

    python -m paper_2307_16080_b200 [--precision exact|f32x3|tf32|bf16] <staircase CLI arguments>

e.g. ``python -m paper_2307_16080_b200 run --input k.sir --func matmul --args a.json
b.json c.json --out outdir`` or ``python -m paper_2307_16080_b200 tune --input
kernels.py --func conv --tiles '8,16;8,16' --unroll 1,2 --log log.jsonl``.

The reference CLI (staircase/cli.py) is used unchanged: its ``run`` and
``tune`` commands call ``staircase.interp.machine.run()`` without an engine
argument (cli.py:211, tuner/search.py:170,190), so installing this package
as ``machine._engine`` routes every tape they execute through the B200
engine — same outputs, stats JSON, exit codes and error messages
(cli.py:385-387).  ``--precision`` selects the contraction precision
(default exact: bit-identical to the reference).  ``run --mode b200`` (or
``b200:bf16`` / ``b200:tf32``) is accepted as the device mode:
it runs the program's sequential semantics on the B200 at that precision.
"""
from __future__ import annotations

import sys


def _device_mode(argv, precision):
    """Rewrite ``--mode b200[:precision]`` to the reference's sequential mode
    (the engine is installed for every mode); returns (argv, precision)."""
    out, i = [], 0
    while i < len(argv):
        a = argv[i]
        if a == "--mode" and i + 1 < len(argv) and argv[i + 1].split(":")[0] == "b200":
            val, i = argv[i + 1], i + 2
        elif a.startswith("--mode=") and a[7:].split(":")[0] == "b200":
            val, i = a[7:], i + 1
        else:
            out.append(a)
            i += 1
            continue
        if ":" in val:
            precision = val.split(":", 1)[1]
        out += ["--mode", "sequential"]
    return out, precision


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    precision = "exact"
    if argv[:1] == ["--precision"] and len(argv) >= 2:
        precision, argv = argv[1], argv[2:]
    elif argv and argv[0].startswith("--precision="):
        precision, argv = argv[0].split("=", 1)[1], argv[1:]
    argv, precision = _device_mode(argv, precision)
    from . import configure, install

    install()
    configure(precision=precision)
    from staircase import cli

    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
