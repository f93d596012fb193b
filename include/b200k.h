/*
 * b200k.h — C ABI of the B200 execution backend for staircase tapes.
 *
 * The reference executes loop nests on the CPU through its engine protocol:
 * staircase.interp.machine.run() calls  eng.run_tape(program, code, regs,
 * tally, ctx)  (reference pkg/src/staircase/interp/machine.py:105-112), whose
 * implementations are the pure and compiled evaluators
 * (interp/_evalpy.py:81-331, interp/_evalcy.pyx:74-344).  The Python engine
 * module paper_2307_16080_b200.engine keeps that protocol and lowers every
 * loop-nest region of the tape onto the entry points below.  Each entry point
 * replaces the part of run_tape named in its comment.
 *
 * Conventions: all data pointers are DEVICE pointers (the host side owns the
 * allocations); `stream` is a cudaStream_t passed as void*; every call only
 * enqueues work on `stream` (no host synchronisation) and returns 0 on
 * success or a negative b200_status on a launch/configuration error.
 * Runtime faults of the executed program (OutOfBounds, InvalidBound) are
 * reported through the device-side b200_vm_error record.
 */
#ifndef B200K_H
#define B200K_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum b200_status {
  B200_OK = 0,
  B200_EINVAL = -1,     /* bad shape / argument */
  B200_ELAUNCH = -2,    /* CUDA launch or attribute error */
  B200_EUNSUPPORTED = -3
};

/* dtype codes shared by all entry points (reference interp/buffer.py:16) */
enum b200_dtype { B200_F32 = 0, B200_F64 = 1, B200_I32 = 2, B200_I64 = 3 };

/* A memref argument: dense row-major storage (reference interp/buffer.py:34-131). */
typedef struct {
  void *ptr;            /* device pointer */
  int32_t dtype;        /* b200_dtype */
  int32_t rank;
  int64_t shape[8];
  int64_t strides[8];   /* in elements */
} b200_buffer;

/* First fault of a checked VM run (reference interp/_evalpy.py:74-78,149-153). */
typedef struct {
  int32_t code;         /* 0 none, 1 OutOfBounds, 2 InvalidBound (loop), 3 InvalidBound (parallel) */
  int32_t slot;         /* buffer slot of the faulting access */
  int64_t index;        /* offending index value */
  int64_t extent;       /* extent of the faulting dimension */
  int64_t loc;          /* location id of the faulting op */
} b200_vm_error;

/*
 * Tape VM: executes a region of a tape, one band point per GPU thread.
 * Replaces run_tape's interpretation of loops, parallel loops, launches,
 * branches, loads/stores and arithmetic (interp/_evalpy.py:81-232,
 * _run_parallel :244-273, _run_launch :303-331) for the region.
 *
 *   prog/n_words     encoded per-thread program (paper_2307_16080_b200/vmcode.py)
 *   init_regs/vals   registers preloaded before the program runs
 *   n_regs           register file size (<= 256)
 *   bufs/n_bufs      DEVICE array of b200_buffer
 *   band_*           HOST arrays, nd band dimensions: register, lower bound, step,
 *                    trip count (copied into the kernel parameters)
 *   count            1: accumulate tally counters into `tally` (25 x uint64, device)
 *   err              DEVICE b200_vm_error, must be zeroed by the caller
 */
int b200_vm_run(const int32_t *prog, int32_t n_words, const int32_t *init_regs,
                const int64_t *init_vals, int32_t n_init, int32_t n_regs,
                const b200_buffer *bufs, int32_t n_bufs, int32_t nd,
                const int32_t *band_regs, const int64_t *band_lb,
                const int64_t *band_step, const int64_t *band_trip, int32_t count,
                unsigned long long *tally, b200_vm_error *err, void *stream);

/*
 * Exact fp32 contraction C[m,n] = C[m,n] (+) sum_k A[m,k]*B[k,n], every
 * product and sum individually rounded (__fmul_rn/__fadd_rn), k ascending:
 * bit-identical to the reference's matmul nests (reference
 * tests/kernels.py:24-38; interp/_evalpy.py:115-127 rounding).
 * Replaces run_tape on a recognised matmul/Linear nest.  Strides in elements,
 * any sign.  init: 0 = accumulate into C, 1 = start from `init_value`.
 * bias (nullable): out[m,n] = out + bias[n*bias_stride] after the chain
 * (the Linear lowering's bias nest).
 */
int b200_gemm_f32_exact(const float *A, int64_t sAm, int64_t sAk,
                        const float *B, int64_t sBk, int64_t sBn,
                        float *C, int64_t sCm, int64_t sCn,
                        int64_t M, int64_t N, int64_t K,
                        int32_t init, float init_value,
                        const float *bias, int64_t bias_stride, void *stream);

/*
 * b200_gemm_f32_exact with an explicit CTA tile (cta_m x cta_n outputs per
 * CTA; <= 0 = the kernel's own choice).  The engine derives it from the tile
 * sizes of a tiled matmul nest (reference passes/tiling.py:56-80, whose
 * outer loop gpu-map sends to blocks: passes/gpumap.py:22-34); supported
 * shapes 128x128, 64x256, 256x64, 64x64, 32x32 (B200_EUNSUPPORTED
 * otherwise); operands that tile whole (unit-stride, 16-byte aligned rows,
 * M / N multiples of the tile, K of 32) run the TMA-fed kernel with that
 * CTA tile, anything else the general tiled kernel.  Results are identical
 * for every tile: each output's k-chain is the same.
 */
int b200_gemm_f32_exact_tiled(const float *A, int64_t sAm, int64_t sAk,
                              const float *B, int64_t sBk, int64_t sBn,
                              float *C, int64_t sCm, int64_t sCn,
                              int64_t M, int64_t N, int64_t K,
                              int32_t init, float init_value,
                              const float *bias, int64_t bias_stride,
                              int32_t cta_m, int32_t cta_n, void *stream);

/*
 * Exact separable contraction (f32 or f64, per-op rounding, K in nest order):
 *   C[c_m[m] + c_n[n]] = (init ? init_value : C[..]) +
 *                        sum_k A[a_m[m] + a_k[k]] * B[b_k[k] + b_n[n]]  (+ bias)
 * with int64 element-offset tables (DEVICE arrays).  Replaces run_tape on any
 * contraction nest whose index maps split into output-row (M), output-column
 * (N) and reduction (K) variable groups — e.g. the NCHW/FCHW conv nest
 * (reference tests/kernels.py:50-64) as an implicit GEMM
 * M = (n, ho, wo), N = co, K = (ci, ki, kj).  a_k_fast / b_n_fast pick the
 * coalesced loader orientation.  Bit-identical to the reference.
 */
int b200_contract_exact(int32_t dtype, const void *A, const int64_t *a_m, const int64_t *a_k,
                        const void *B, const int64_t *b_k, const int64_t *b_n, void *C,
                        const int64_t *c_m, const int64_t *c_n, int64_t M, int64_t N, int64_t K,
                        int32_t a_k_fast, int32_t b_n_fast, int32_t init, double init_value,
                        const void *bias, int64_t bias_stride, void *stream);

/*
 * Pointwise f32 nest (fill / copy / elementwise / broadcast bias): every point
 * of the nd-dim box runs the straight-line program `prog` (map.cu encoding:
 * LD/CF/BF/ST over 8 registers) on n_ops operands addressed
 * ptrs[k] + sum_d coefs[k*nd + d] * i_d.  Replaces run_tape on race-free
 * straight-line nests (reference interp/_evalpy.py:90-127; PAPER.md:431-441,
 * 455-462 fill/copy/bias nests).  Per-op IEEE f32 rounding (bit-exact).
 * ptrs/coefs/trips/prog/consts are HOST arrays (copied into the kernel
 * parameters).  vector: 128-bit path (innermost trip % 4 == 0, operands
 * contiguous or broadcast along it); nload: number of leading LD words
 * whose loads may be issued together (0..4).
 */
int b200_map_f32(const int32_t *prog, int32_t n_words, const float *consts, int32_t n_consts,
                 float *const *ptrs, const int64_t *coefs, int32_t n_ops, const int64_t *trips,
                 int32_t nd, int32_t vector, int32_t nload, void *stream);

/*
 * Operand packing for the tensor-core contraction: dst[r][c] (dense
 * row-major, i.e. K-major for the GEMM) = round(src[r*s_row + c*s_col]),
 * kind 0 -> bf16 (RN), kind 1 -> tf32 held in f32 (RN, low 13 bits zero).
 * kinds 2 / 3: the split pack of the fp32-accurate "f32x3" path (3xTF32):
 * with hi = tf32(x), lo = tf32(x - hi), each dst row holds 3 * cols
 * values, [hi | hi | lo] (kind 2, the A operand) or [hi | lo | hi]
 * (kind 3, B^T), so a kind-1 b200_gemm_tc over K' = 3K sums
 * hiA.hiB + hiA.loB + loA.hiB.
 * Used to stage A (rows = M) and B^T (rows = N) of a recognised matmul nest,
 * whatever the nest's index maps (reference tests/kernels.py:24-38).
 */
int b200_pack_operand(int32_t kind, const float *src, int64_t s_row, int64_t s_col,
                      void *dst, int64_t rows, int64_t cols, void *stream);

/*
 * Tensor-core contraction (tcgen05.mma, TMEM accumulators, TMA operand
 * loads): C[m*sCm + n*sCn] = (init ? init_value : C[...]) + sum_k A[m,k]*Bt[n,k]
 * (+ bias[n*bias_stride]), fp32 accumulate.  kind 0: bf16 operands
 * (kind::f16), kind 1: tf32 operands (kind::tf32).  A is M x K and Bt is
 * N x K, dense K-major (b200_pack_operand output).  Replaces run_tape on a
 * recognised matmul / Linear contraction when the engine precision is bf16
 * or tf32 (accumulation-order tolerance).  max_ctas <= 0 uses
 * one persistent CTA per SM.  variant: 0 auto, 1 single-CTA 128x256 tiles,
 * 2 CTA-pair 256x256 tiles (tcgen05 cta_group::2), 3 128x256 tiles as
 * cta_group::1 MMAs in 2-CTA clusters sharing the B tile by TMA multicast
 * (the engine's choice for the reference's (4, 16) tiling).
 */
int b200_gemm_tc(int32_t kind, const void *A, const void *Bt, float *C, int64_t sCm,
                 int64_t sCn, int64_t M, int64_t N, int64_t K, int32_t init,
                 float init_value, const float *bias, int64_t bias_stride,
                 int32_t max_ctas, int32_t variant, void *stream);

/*
 * b200_gemm_tc that also writes the final C (after init / bias) rounded to
 * bf16 into c16 (row-major, leading dimension ld16 >= N): the K-major packed
 * A operand of a following contraction that reads C — e.g. the second
 * Linear of a chained Linear stack, whose activations the reference keeps in
 * an f32 Buffer (the f32 C is still written in full).  Saves the separate
 * b200_pack_operand pass over C.
 */
/*
 * b200_gemm_tc with B given as a K x N row-major bf16 tensor — the matmul
 * nest's own B layout, converted to bf16 but not transposed — read MN-major
 * by the tensor cores (no transposing pack).  kind must be 0 (bf16); c16 /
 * ld16 as in b200_gemm_tc_shadow, c16 may be NULL.  N must be a multiple of
 * 64 (B200_EUNSUPPORTED otherwise).
 */
int b200_gemm_tc_kn(int32_t kind, const void *A, const void *B, float *C, int64_t sCm,
                    int64_t sCn, int64_t M, int64_t N, int64_t K, int32_t init,
                    float init_value, const float *bias, int64_t bias_stride, void *c16,
                    int64_t ld16, void *stream);

int b200_gemm_tc_shadow(int32_t kind, const void *A, const void *Bt, float *C, int64_t sCm,
                        int64_t sCn, int64_t M, int64_t N, int64_t K, int32_t init,
                        float init_value, const float *bias, int64_t bias_stride,
                        void *c16, int64_t ld16, void *stream);

/*
 * Convolution on the tensor cores (conv_2d_nchw_fchw, valid, stride 1;
 * reference tests/kernels.py:50-64), engine precision
 * bf16.  b200_pack_conv_input: NCHW f32 (element strides sstr[4], HOST array)
 * -> NHWC bf16 with channels zero-padded to cp (multiple of 64).
 * b200_pack_conv_weight: FCHW f32 -> [F][KH][KW][cp] bf16.
 * b200_conv2d_tc: out[n,f,h,w] = (init ? init_value : out[..]) + sum over
 * (ki, kj, c) of in*w, fp32 accumulation in TMEM (tcgen05.mma, TMA operand
 * boxes, weights resident in shared memory).  out_strides: HOST array of the
 * NCHW element strides (w stride must be 1).  F in {32, 64, 128}.
 */
int b200_pack_conv_input(const float *src, const int64_t *sstr, void *dst, int64_t nb,
                         int64_t c, int64_t h, int64_t w, int64_t cp, void *stream);
int b200_pack_conv_weight(const float *src, const int64_t *sstr, void *dst, int64_t f,
                          int64_t c, int64_t kh, int64_t kw, int64_t cp, void *stream);
/*
 * b200_pack_conv_input and b200_pack_conv_weight in one launch when the
 * input takes the all-bulk pack (dense planes, 16-byte channel / image
 * strides), else the two packs back to back.  Same arguments as the two.
 */
int b200_pack_conv(const float *src, const int64_t *sstr, void *dst, int64_t nb, int64_t c,
                   int64_t h, int64_t w, int64_t cp, const float *ker, const int64_t *wstr,
                   void *wdst, int64_t f, int64_t kh, int64_t kw, void *stream);

int b200_conv2d_tc(const void *in_nhwc, const void *wt, float *out, const int64_t *out_strides,
                   int64_t nb, int64_t cp, int64_t hp, int64_t wp, int64_t f, int64_t ho,
                   int64_t wo, int64_t kh, int64_t kw, int32_t init, float init_value,
                   void *stream);
/*
 * b200_conv2d_tc without the input repack: `in` is the NCHW f32 input
 * (element strides in_strides[4], HOST array; dense planes: w stride 1,
 * h stride = wp, 16-byte channel and image strides), read by TMA in raw
 * f32 row spans and converted to the bf16 NHWC patch inside the kernel by a
 * converter warpgroup.  `wt` as for b200_conv2d_tc (b200_pack_conv_weight,
 * cp = c rounded up to 64).  3x3 merged-tap tiling only (F in {32, 64});
 * B200_EUNSUPPORTED otherwise, and the caller packs instead.
 */
int b200_conv2d_tc_fused(const float *in, const int64_t *in_strides, const void *wt, float *out,
                         const int64_t *out_strides, int64_t nb, int64_t c, int64_t hp,
                         int64_t wp, int64_t f, int64_t ho, int64_t wo, int64_t kh, int64_t kw,
                         int32_t init, float init_value, void *stream);

/*
 * Bit-exact direct convolution (conv_2d_nchw_fchw, valid, stride 1;
 * reference tests/kernels.py:50-64) at the exact precision: out[n,f,h,w] =
 * (init ? init_value : out[..]) + the ci -> ki -> kj chain of individually
 * rounded products and sums (interp/_evalpy.py:115-127), f32 (dtype 0) or
 * f64 (dtype 1).  in / w / out strides are HOST arrays of 4 element strides
 * (NCHW, FCHW, NCHW).  w_work: DEVICE scratch of f*c*kh*kw elements (the
 * weights transposed to [C][KH*KW][F]).  Same results as
 * b200_contract_exact on the conv nest, with operands staged in shared
 * memory instead of gathered through offset tables.
 */
int b200_conv2d_exact(int32_t dtype, const void *in, const int64_t *in_strides, const void *w,
                      const int64_t *w_strides, void *w_work, void *out,
                      const int64_t *out_strides, int64_t nb, int64_t c, int64_t hp, int64_t wp,
                      int64_t f, int64_t ho, int64_t wo, int64_t kh, int64_t kw, int32_t init,
                      double init_value, void *stream);

/*
 * The tuner's seeded inputs (replaces the per-element
 * [rng.uniform(-2.0, 2.0) for _ in range(size)] of _fresh_argument,
 * reference pkg/src/staircase/tuner/search.py:78-90).  HOST code: `state` is
 * the 624-word MT19937 state of a Python random.Random (getstate()[1][:624]),
 * `*pos` its index (getstate()[1][624]); writes n values lo + (hi - lo) *
 * random() as f32 (round to nearest) or f64 into host memory `out` and
 * advances state / pos exactly as n Python draws would.
 */
int b200_mt_uniform(uint32_t *state, int32_t *pos, int64_t n, double lo, double hi, void *out,
                    int32_t dtype);

/*
 * A strided host <-> device block copy (cudaMemcpy2DAsync): `rows` rows of
 * `width` bytes, row pitches `dpitch` / `spitch` bytes; kind 1 = host to
 * device, 2 = device to host; enqueued on `stream`.  Used to stream column
 * panels of B and (row, column) blocks of C around the exact GEMM (replaces
 * the per-run Buffer upload / write-back of interp/buffer.py for those).
 */
int b200_copy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
                int64_t rows, int32_t kind, void *stream);

/*
 * The tuner's equivalence guard (replaces the per-element
 * math.isclose(got, want, rel_tol=1e-6, abs_tol=1e-9) loop of
 * reference tuner/search.py:128-138): adds to *bad (device counter) the
 * number of the n elements of `got` (B200_F32 / B200_F64, device) that are not
 * close to `want` (device, f64).
 */
int b200_guard_close(int32_t dtype, const void *got, const double *want, int64_t n,
                     double rel_tol, double abs_tol, unsigned long long *bad, void *stream);

/*
 * Runtime specialisation (NVRTC, sm_100a): compile generated CUDA C `src`
 * and return the kernel `kernel` as an opaque handle in *fn.  The engine
 * generates straight-line kernels for region shapes whose generic execution
 * would be interpretive (pointwise nests: reference interp/_evalpy.py:90-127
 * per point).  b200_jit_log() returns the last compiler log.
 */
int b200_jit_compile(const char *src, const char *kernel, void **fn);
const char *b200_jit_log(void);

/*
 * The same compilation split in two for the on-disk kernel cache (jit.py):
 * b200_jit_cubin compiles to an sm_100a cubin image (no device needed;
 * *size = image bytes, B200_EINVAL if cap is too small), b200_jit_load turns
 * an image into the kernel's CUfunction.
 */
int b200_jit_cubin(const char *src, void *out, size_t cap, size_t *size);
int b200_jit_load(const void *image, const char *kernel, void **fn);

/* Launch a b200_jit_compile kernel; args = array of pointers to argument values. */
int b200_jit_launch(void *fn, uint32_t gx, uint32_t gy, uint32_t gz, uint32_t bx, uint32_t by,
                    uint32_t bz, uint32_t smem, void **args, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* B200K_H */
