"""DSL nests for the BASELINE.json configs, captured with the reference frontend.

Full-size kernels (run on the B200 through the engine) and the thin slices
the reference CPU executor is timed on (same loop structure and reduction
length).  Capture reads source from disk, so
they live in a module.

  mm4096      linalg.matmul 4096^3 (reference tests/kernels.py:24-38 nest)
  conv_cv     conv_2d_nchw_fchw ResNet-50 layer: (256,64,58,58) pre-padded
              input x (64,64,3,3) -> (256,64,56,56)
  linear32    torch.nn.Linear(32,32) lowering
  ls_*        batched Linear stack 65536 x 1024 -> 4096 -> 1024 with fill and
              bias nests (two Linear lowerings chained, fill into the output)
  saxpy8k     elementwise y = y + x * 2 over 8192 x 8192 f32 (512 MB working set > L2)
"""
from staircase import F32, F64, MemRef, constant, parallel, staged

# -- matmul -------------------------------------------------------------------


@staged(range_ctor="affine_for")
def mm4096(A: MemRef[(4096, 4096), F32], B: MemRef[(4096, 4096), F32],
           C: MemRef[(4096, 4096), F32]):
    for i in range(4096):
        for j in range(4096):
            for k in range(4096):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


@staged(range_ctor="affine_for")
def mm_slice(A: MemRef[(1, 4096), F32], B: MemRef[(4096, 256), F32],
             C: MemRef[(1, 256), F32]):
    for i in range(1):
        for j in range(4096):
            for k in range(256):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


# -- convolution (per-rank batch shards are separate captures) -------------------


def make_conv(nb):
    """conv_2d_nchw_fchw over a batch shard of nb images (C=F=64, 56x56, 3x3)."""
    ns = {"F32": F32, "MemRef": MemRef, "parallel": parallel, "staged": staged}
    src = f'''
@staged
def conv_cv(inp: MemRef[({nb}, 64, 58, 58), F32], ker: MemRef[(64, 64, 3, 3), F32],
            out: MemRef[({nb}, 64, 56, 56), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), ({nb}, 64, 56, 56)):
        for ci in range(0, 64):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]
'''
    return _capture_from_source(src, "conv_cv", ns, nb)


@staged
def conv_slice(inp: MemRef[(1, 64, 58, 58), F32], ker: MemRef[(2, 64, 3, 3), F32],
               out: MemRef[(1, 2, 8, 56), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 2, 8, 56)):
        for ci in range(0, 64):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


# -- Linear(32, 32) -----------------------------------------------------------------


@staged(range_ctor="scf_for")
def linear32(x: MemRef[(32, 32), F32], wt: MemRef[(32, 32), F32],
             bias: MemRef[(32,), F32], tmp: MemRef[(32, 32), F32],
             out: MemRef[(32, 32), F32]):
    for i in range(32):
        for j in range(32):
            tmp[i, j] = constant(0.0, F32)
    for i in range(32):
        for j in range(32):
            out[i, j] = tmp[i, j]
    for i in range(32):
        for j in range(32):
            for k in range(32):
                a = x[i, k]
                b = wt[k, j]
                c = out[i, j]
                d = a * b
                e = c + d
                out[i, j] = e
    for i in range(32):
        for j in range(32):
            out[i, j] = out[i, j] + bias[j]


# -- Linear stack -----------------------------------------------------------------


def make_linear_stack(rows):
    """Two chained Linear lowerings (fill, contraction, bias) over `rows` rows."""
    ns = {"F32": F32, "MemRef": MemRef, "parallel": parallel, "staged": staged,
          "constant": constant}
    src = f'''
@staged
def linear_stack(x: MemRef[({rows}, 1024), F32], w1t: MemRef[(1024, 4096), F32],
                 b1: MemRef[(4096,), F32], h: MemRef[({rows}, 4096), F32],
                 w2t: MemRef[(4096, 1024), F32], b2: MemRef[(1024,), F32],
                 y: MemRef[({rows}, 1024), F32]):
    for i, j in parallel((0, 0), ({rows}, 4096)):
        h[i, j] = constant(0.0, F32)
    for i, j in parallel((0, 0), ({rows}, 4096)):
        for k in range(1024):
            h[i, j] += x[i, k] * w1t[k, j]
    for i, j in parallel((0, 0), ({rows}, 4096)):
        h[i, j] = h[i, j] + b1[j]
    for i, j in parallel((0, 0), ({rows}, 1024)):
        y[i, j] = constant(0.0, F32)
    for i, j in parallel((0, 0), ({rows}, 1024)):
        for k in range(4096):
            y[i, j] += h[i, k] * w2t[k, j]
    for i, j in parallel((0, 0), ({rows}, 1024)):
        y[i, j] = y[i, j] + b2[j]
'''
    return _capture_from_source(src, "linear_stack", ns, rows)


# -- elementwise ------------------------------------------------------------------


@staged
def saxpy8k(x: MemRef[(8192, 8192), F32], y: MemRef[(8192, 8192), F32]):
    for i, j in parallel((0, 0), (8192, 8192)):
        y[i, j] = y[i, j] + x[i, j] * constant(2.0, F32)


# -- design-space sweep targets (tiled / unrolled by the tuner's pipeline) ----------


@staged
def mm_par1024(A: MemRef[(1024, 1024), F32], B: MemRef[(1024, 1024), F32],
               C: MemRef[(1024, 1024), F32]):
    for i, k in parallel((0, 0), (1024, 1024)):
        for j in range(1024):
            C[i, k] += A[i, j] * B[j, k]


@staged
def conv_paper(inp: MemRef[(1, 1, 1282, 1282), F32], ker: MemRef[(1, 1, 3, 3), F32],
               out: MemRef[(1, 1, 1280, 1280), F32]):
    # the paper's tuning target: (1,1,1280,1280) * (1,3,3)
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 1, 1280, 1280)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


@staged
def mm_slice1024(A: MemRef[(1, 1024), F32], B: MemRef[(1024, 1024), F32],
                 C: MemRef[(1, 1024), F32]):
    # one output row of mm_par1024: same loop structure and reduction length
    for i, k in parallel((0, 0), (1, 1024)):
        for j in range(1024):
            C[i, k] += A[i, j] * B[j, k]


@staged
def conv_paper_slice(inp: MemRef[(1, 1, 10, 1282), F32], ker: MemRef[(1, 1, 3, 3), F32],
                     out: MemRef[(1, 1, 8, 1280), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 1, 8, 1280)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


@staged
def conv_desk_small(input: MemRef[(1, 1, 18, 18), F64], kernel: MemRef[(2, 1, 3, 3), F64],
                    output: MemRef[(1, 2, 16, 16), F64]):
    # desk-scale tuning target (reference tests/kernels.py:67-88 shapes)
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 2, 16, 16)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    output[n, co, ho, wo] += input[n, ci, ho + ki, wo + kj] * kernel[co, ci, ki, kj]


@staged
def saxpy_slice(x: MemRef[(16, 4096), F32], y: MemRef[(16, 4096), F32]):
    for i, j in parallel((0, 0), (16, 4096)):
        y[i, j] = y[i, j] + x[i, j] * constant(2.0, F32)


# capture needs real source files: write each generated kernel once
_GEN = {}


def _capture_from_source(src, name, ns, size):
    import importlib.util
    import os
    import tempfile

    key = (name, size)
    if key in _GEN:
        return _GEN[key]
    import hashlib

    d = os.path.join(tempfile.gettempdir(), "b200_bench_kernels")
    os.makedirs(d, exist_ok=True)
    header = ("from staircase import F32, F64, MemRef, constant, parallel, staged\n")
    text = header + src
    # content-addressed, written atomically: several ranks (or test workers)
    # capture the same kernel concurrently and must never read a partial file
    path = os.path.join(d, f"{name}_{size}_{hashlib.sha1(text.encode()).hexdigest()[:12]}.py")
    if not os.path.exists(path):
        tmp = f"{path}.{os.getpid()}.tmp"
        with open(tmp, "w") as fh:
            fh.write(text)
        os.replace(tmp, path)
    spec = importlib.util.spec_from_file_location(f"_b200_{name}_{size}", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    fn = getattr(mod, name)
    _GEN[key] = fn
    return fn


# -- matmul, parallel form (tile-size knob applies: scf-parallel-loop-tiling) ----------


@staged
def mm_par4096(A: MemRef[(4096, 4096), F32], B: MemRef[(4096, 4096), F32],
               C: MemRef[(4096, 4096), F32]):
    # BASELINE configs[1] "with reference tile sizes": the parallel form of the
    # matmul nest, tiled (8, 8) or (4, 16) by the reference's pass
    for i, k in parallel((0, 0), (4096, 4096)):
        for j in range(4096):
            C[i, k] += A[i, j] * B[j, k]
