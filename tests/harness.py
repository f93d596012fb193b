"""Shared helpers: seeded inputs, pipeline variants, run-and-compare.

Input recipe (used identically by tests/golden/make_golden.py): for every
parameter of the staged function, in order, ``random.Random(seed)`` draws
U(-2, 2) floats for float memrefs and float scalars, integers in [-50, 50)
for integer memrefs, and index scalars take ``INDEX_ARGS`` (the tuner's
make_inputs recipe, staircase/tuner/search.py:78-95, with a pinned index
value so loop bounds stay in range).
"""
import random

import corpus
from staircase.interp import Buffer, machine
from staircase.passes import run_pipeline

INDEX_ARGS = 20


def make_args(fn, seed):
    rng = random.Random(seed)
    out = []
    for a in fn.func_op.body().args:
        t = a.type
        if t.kind == "memref":
            n = 1
            for s in t.shape:
                n *= s
            if t.element.kind in ("f32", "f64"):
                data = [rng.uniform(-2.0, 2.0) for _ in range(n)]
            else:
                data = [rng.randrange(-50, 50) for _ in range(n)]
            out.append(Buffer(t.shape, t.element.kind, data))
        elif t.kind in ("f32", "f64"):
            out.append(rng.uniform(-2.0, 2.0))
        elif t.kind == "index":
            out.append(INDEX_ARGS)
        else:
            out.append(rng.randrange(-50, 50))
    return out


def transformed(fn, pipeline):
    if not pipeline:
        return fn.module
    work, _ = run_pipeline(fn.module, pipeline)
    return work


def _spec(*items):
    return "builtin.module(func.func(" + ", ".join(items) + "))"


def _mspec(func_items, module_items=()):
    inner = "func.func(" + ", ".join(func_items) + ")"
    return "builtin.module(" + ", ".join([inner, *module_items]) + ")"


UNROLL2 = _spec("lower-affine", "loop-unroll{factor=2}")
UNROLL4 = _spec("lower-affine", "loop-unroll{factor=4}")
TILE88 = _spec("scf-parallel-loop-tiling{sizes=[8, 8]}")
TILE416 = _spec("scf-parallel-loop-tiling{sizes=[4, 16]}")
TILE88_U3 = _spec("scf-parallel-loop-tiling{sizes=[8, 8]}", "loop-unroll{factor=3}")
OUTLINE = _mspec(["gpu-map-parallel-loops"], ["gpu-kernel-outlining"])
TILE_OUTLINE = _mspec(["scf-parallel-loop-tiling{sizes=[8, 8]}", "gpu-map-parallel-loops"],
                      ["gpu-kernel-outlining"])

# (kernel, variant name, pipeline spec or None, mode)
CASES = [
    (corpus.matmul_affine, "base", None, "sequential"),
    (corpus.matmul_affine, "unroll2", UNROLL2, "sequential"),
    (corpus.matmul_affine, "unroll4", UNROLL4, "sequential"),
    (corpus.matmul_96, "base", None, "sequential"),
    (corpus.matmul_par, "base", None, "sequential"),
    (corpus.matmul_par, "tile416", TILE416, "sequential"),
    (corpus.matmul_par, "tile88_u3", TILE88_U3, "sequential"),
    (corpus.matmul_par, "outline", TILE_OUTLINE, "gpu_emulated"),
    (corpus.linear32, "base", None, "sequential"),
    (corpus.linear32, "unroll4", UNROLL4, "sequential"),
    (corpus.conv2d_desk, "base", None, "sequential"),
    (corpus.conv2d_desk, "outline", OUTLINE, "gpu_emulated"),
    (corpus.conv_small, "base", None, "sequential"),
    (corpus.conv_small, "tile88", TILE88, "sequential"),
    (corpus.conv_small, "tile416", TILE416, "sequential"),
    (corpus.conv_small, "tile_outline", TILE_OUTLINE, "gpu_emulated"),
    (corpus.conv_rows, "base", None, "sequential"),
    (corpus.conv_rows, "unroll2", UNROLL2, "sequential"),
    (corpus.conv_f32, "base", None, "sequential"),
    (corpus.conv_f32, "tile88", TILE88, "worksharing"),
    (corpus.saxpy, "base", None, "sequential"),
    (corpus.saxpy_f32, "base", None, "sequential"),
    (corpus.saxpy_f32, "unroll4", UNROLL4, "sequential"),
    (corpus.strided, "base", None, "sequential"),
    (corpus.ewise_ops, "base", None, "sequential"),
    (corpus.int_ops, "base", None, "sequential"),
    (corpus.cond_body, "base", None, "sequential"),
    (corpus.triangle, "base", None, "sequential"),
    (corpus.prefix, "base", None, "sequential"),
    (corpus.scalar_args, "base", None, "sequential"),
    (corpus.ewise_gpu, "base", None, "gpu_emulated"),
    (corpus.ewise_gpu, "seq_mode", None, "sequential"),
    (corpus.oob_kernel, "base", None, "sequential"),
]


def run_engine(engine, fn, pipeline, mode, seed, args=None):
    """Run through the reference's own run() with the given engine.

    Returns (results, args, tally, stats) or raises what run() raises.
    """
    module = transformed(fn, pipeline)
    if args is None:
        args = make_args(fn, seed)
    box = {}

    class Tap:
        ExecContext = engine.ExecContext

        @staticmethod
        def run_tape(program, code, regs, tally, ctx):
            out = engine.run_tape(program, code, regs, tally, ctx)
            box["t"] = list(tally)
            return out

    results, stats = machine.run(module, fn.__name__, args, mode=mode, engine=Tap)
    return results, args, box["t"], stats
