"""DSL kernel corpus for the parity tests.

Captured with the reference's unchanged frontend (staircase ``@staged`` /
``GPUModule``).  Capture reads function source from disk, so these live in
a real module.  The nests restate the paper's loop nests:

- ``matmul_affine``  — the affine matmul of PAPER.md:143-191
  (same nest as reference tests/kernels.py:24-38, M,N,K = 4,16,8);
- ``linear32``       — the torch.nn.Linear(32,32) loop-level lowering of
  PAPER.md:427-468 (fill, copy, contraction, bias), SURVEY.md Appendix A.1;
- ``conv2d_desk``    — the NCHW/FCHW conv parallel over outputs
  (reference tests/kernels.py:50-64 shapes);
- ``conv_small``, ``conv_rows`` — the tiling/unrolling targets
  (reference tests/kernels.py:67-107 shapes);
- ``saxpy``, ``strided`` — elementwise nests (benchmarks/bench_interp.py:46-49,
  tests/kernels.py:110-113);
- ``ewise_gpu``      — the GPUModule elementwise kernel of PAPER.md:749-785.
"""
from staircase import (F32, F64, I32, I64, Index, GPUModule, MemRef, block_id_x,
                       block_id_y, constant, parallel, staged)


@staged(range_ctor="affine_for")
def matmul_affine(A: MemRef[(4, 16), F32], B: MemRef[(16, 8), F32],
                  C: MemRef[(4, 8), F32]):
    for i in range(4):
        for j in range(16):
            for k in range(8):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


@staged(range_ctor="affine_for")
def matmul_96(A: MemRef[(64, 96), F32], B: MemRef[(96, 80), F32],
              C: MemRef[(64, 80), F32]):
    for i in range(64):
        for j in range(96):
            for k in range(80):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


@staged
def matmul_par(A: MemRef[(32, 48), F32], B: MemRef[(48, 64), F32],
               C: MemRef[(32, 64), F32]):
    for i, k in parallel((0, 0), (32, 64)):
        for j in range(48):
            C[i, k] += A[i, j] * B[j, k]


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


@staged
def conv2d_desk(input: MemRef[(1, 1, 64, 64), F64],
                kernel: MemRef[(3, 1, 3, 3), F64],
                output: MemRef[(1, 3, 62, 62), F64]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 3, 62, 62)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    ii = ho + ki
                    jj = wo + kj
                    inp = input[n, ci, ii, jj]
                    ker = kernel[co, ci, ki, kj]
                    output[n, co, ho, wo] += inp * ker


@staged
def conv_small(input: MemRef[(1, 1, 18, 18), F64],
               kernel: MemRef[(2, 1, 3, 3), F64],
               output: MemRef[(1, 2, 16, 16), F64]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 2, 16, 16)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    inp = input[n, ci, ho + ki, wo + kj]
                    ker = kernel[co, ci, ki, kj]
                    output[n, co, ho, wo] += inp * ker


@staged
def conv_rows(input: MemRef[(1, 1, 64, 64), F64],
              kernel: MemRef[(3, 1, 3, 3), F64],
              output: MemRef[(1, 3, 62, 62), F64]):
    for co, ho in parallel((0, 0), (3, 62)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    for wo in range(0, 62):
                        inp = input[0, ci, ho + ki, wo + kj]
                        ker = kernel[co, ci, ki, kj]
                        output[0, co, ho, wo] += inp * ker


@staged
def conv_f32(inp: MemRef[(2, 8, 18, 18), F32], ker: MemRef[(4, 8, 3, 3), F32],
             out: MemRef[(2, 4, 16, 16), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (2, 4, 16, 16)):
        for ci in range(0, 8):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


@staged
def saxpy(x: MemRef[(256, 256), F64], y: MemRef[(256, 256), F64]):
    for i, j in parallel((0, 0), (256, 256)):
        y[i, j] = y[i, j] + x[i, j] * 2.0


@staged
def saxpy_f32(x: MemRef[(64, 128), F32], y: MemRef[(64, 128), F32]):
    for i in range(64):
        for j in range(128):
            y[i, j] = y[i, j] + x[i, j] * constant(2.0, F32)


@staged
def strided(buf: MemRef[(64,), F64]):
    for i in range(0, 42, 2):
        buf[i] = buf[i] * 3.0 + 1.0


@staged
def ewise_ops(a: MemRef[(16, 24), F32], b: MemRef[(16, 24), F32],
              c: MemRef[(16, 24), F32]):
    for i in range(16):
        for j in range(24):
            x = a[i, j]
            y = b[i, j]
            c[i, j] = (x - y) / (x * y + constant(0.5, F32))


@staged
def int_ops(a: MemRef[(8, 8), I32], b: MemRef[(8, 8), I64], c: MemRef[(8, 8), I32]):
    for i in range(8):
        for j in range(8):
            c[i, j] = a[i, j] * a[j, i] + a[i, j]
            b[i, j] = b[i, j] * b[i, j] - b[j, i]


@staged
def cond_body(a: MemRef[(16, 16), F32], out: MemRef[(16, 16), F32]):
    for i in range(16):
        for j in range(16):
            v = a[i, j]
            if v > constant(0.0, F32):
                out[i, j] = v
            else:
                out[i, j] = v * constant(-2.0, F32)


@staged
def triangle(a: MemRef[(16, 16), F32]):
    for i in range(16):
        for j in range(i):
            a[i, j] = a[j, i] + a[i, j]


@staged
def prefix(a: MemRef[(64,), F64]):
    for i in range(1, 64):
        a[i] = a[i] + a[i - 1]


@staged
def oob_kernel(a: MemRef[(8, 8), F32], b: MemRef[(8, 8), F32]):
    for i in range(8):
        for j in range(8):
            b[i, j] = a[i, j + 1]


@staged
def scalar_args(a: MemRef[(32,), F32], s: F32, n: Index):
    for i in range(n):
        a[i] = a[i] * s


class EwiseGPU(GPUModule):
    def kernel(self, A: MemRef[(4, 4), F32], B: MemRef[(4, 4), F32],
               C: MemRef[(4, 4), F32]):
        x = block_id_x()
        y = block_id_y()
        a = A[x, y]
        b = B[x, y]
        C[x, y] = a * b
        return


_ewise_mod = EwiseGPU()


@staged
def ewise_gpu(A: MemRef[(4, 4), F32], B: MemRef[(4, 4), F32],
              C: MemRef[(4, 4), F32]):
    _ewise_mod.kernel(A, B, C, grid_size=[4, 4, 1], block_size=[1, 1, 1])


ALL = [oob_kernel, matmul_affine, matmul_96, matmul_par, linear32, conv2d_desk, conv_small,
       conv_rows, conv_f32, saxpy, saxpy_f32, strided, ewise_ops, int_ops,
       cond_body, triangle, prefix, scalar_args, ewise_gpu]


# -- larger shapes for the GPU parity tests (edges not multiples of the tiles)


@staged(range_ctor="affine_for")
def matmul_odd(A: MemRef[(130, 150), F32], B: MemRef[(150, 70), F32],
               C: MemRef[(130, 70), F32]):
    for i in range(130):
        for j in range(150):
            for k in range(70):
                C[i, k] = C[i, k] + A[i, j] * B[j, k]


@staged
def matmul_t(A: MemRef[(96, 160), F32], Bt: MemRef[(200, 160), F32],
             C: MemRef[(96, 200), F32]):
    for i, n in parallel((0, 0), (96, 200)):
        for k in range(160):
            C[i, n] = C[i, n] + A[i, k] * Bt[n, k]


@staged
def conv_mid(inp: MemRef[(4, 16, 34, 34), F32], ker: MemRef[(8, 16, 3, 3), F32],
             out: MemRef[(4, 8, 32, 32), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (4, 8, 32, 32)):
        for ci in range(0, 16):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


BIG = [matmul_odd, matmul_t, conv_mid]


# -- tensor-core smoke shapes (__graft_entry__.smoke) ----------------------------


@staged
def mm_tc_smoke(A: MemRef[(256, 192), F32], B: MemRef[(192, 256), F32],
                C: MemRef[(256, 256), F32]):
    for i, k in parallel((0, 0), (256, 256)):
        for j in range(192):
            C[i, k] += A[i, j] * B[j, k]


@staged
def conv_tc_smoke(inp: MemRef[(2, 64, 18, 30), F32], ker: MemRef[(64, 64, 3, 3), F32],
                  out: MemRef[(2, 64, 16, 28), F32]):
    for n, co, ho, wo in parallel((0, 0, 0, 0), (2, 64, 16, 28)):
        for ci in range(0, 64):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]


@staged
def store_then_load(x: MemRef[(64, 128), F32], y: MemRef[(64, 128), F32],
                    z: MemRef[(64, 128), F32]):
    # a store followed by a load of the same element inside one point: the
    # JIT map kernel must not treat the two y operands as non-aliasing
    for i, j in parallel((0, 0), (64, 128)):
        y[i, j] = constant(3.0, F32)
        z[i, j] = y[i, j] * x[i, j]


@staged
def conv_ones8(input: MemRef[(1, 1, 8, 8), F64], kernel: MemRef[(1, 1, 3, 3), F64],
               output: MemRef[(1, 1, 6, 6), F64]):
    # SPEC.md:568 "conv2d on input 1x1x8x8 ones, kernel 1x3x3 ones -> interior
    # outputs 9.0" (valid conv: every output is interior)
    for n, co, ho, wo in parallel((0, 0, 0, 0), (1, 1, 6, 6)):
        for ci in range(0, 1):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    output[n, co, ho, wo] += input[n, ci, ho + ki, wo + kj] * kernel[co, ci, ki, kj]


@staged
def conv_ones64(inp: MemRef[(2, 64, 10, 30), F32], ker: MemRef[(64, 64, 3, 3), F32],
                out: MemRef[(2, 64, 8, 28), F32]):
    # the same known answer through the tcgen05 conv (C = F = 64): 9 * 64
    for n, co, ho, wo in parallel((0, 0, 0, 0), (2, 64, 8, 28)):
        for ci in range(0, 64):
            for ki in range(0, 3):
                for kj in range(0, 3):
                    out[n, co, ho, wo] += inp[n, ci, ho + ki, wo + kj] * ker[co, ci, ki, kj]
