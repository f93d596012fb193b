// Pointwise nests on the B200: fill / copy / elementwise / broadcast-bias.
//
// Replaces run_tape on a region whose every loop variable is distributed
// (the whole iteration box is race-free, analysis.choose_band) and whose body
// is straight-line f32 code: loads, constants, add/sub/mul/div, stores
// (reference interp/_evalpy.py:90-127; nests such as PAPER.md:431-441 fill /
// copy, PAPER.md:455-462 bias, benchmarks/bench_interp.py:46-49 saxpy).
//
// Each operand is addressed affinely over the box: off = base + sum_d coef_d*i_d.
// Vector path: the innermost box dimension is split into groups of 4 and every
// operand is either contiguous (coef 1, 16-byte aligned) or broadcast (coef 0)
// along it, so each thread moves 128-bit vectors; otherwise one element per
// thread.  The per-element program runs in reference order with each f32 op
// individually rounded (__f*_rn), so results are bit-identical to the
// reference.  Grid: persistent, 148 SMs x 8 CTAs x 256 threads, grid-stride.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"

namespace {

constexpr int kMaxDims = 8;
constexpr int kMaxOps = 16;
constexpr int kMaxRegs = 32;
constexpr int kMaxProg = 256;  // words
constexpr int kMaxConst = 32;

enum { M_LD = 0, M_CF = 1, M_BF = 2, M_ST = 3 };

struct MapParams {
  float *ptr[kMaxOps];
  int64_t coef[kMaxOps][kMaxDims];
  int64_t trip[kMaxDims];
  int32_t prog[kMaxProg];
  float consts[kMaxConst];
  int32_t nd, nops, nwords;
  int64_t total;   // work items (vectors or elements)
};

__device__ __forceinline__ float fop(int f, float a, float b) {
  return f == 0 ? __fadd_rn(a, b) : f == 1 ? __fsub_rn(a, b) : f == 2 ? __fmul_rn(a, b)
                                                                   : __fdiv_rn(a, b);
}

template <bool VEC, bool ONE_D, int NL>
__global__ void __launch_bounds__(256) map_kernel(const __grid_constant__ MapParams p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < p.total; w += stride) {
    // decompose the work index over the box (innermost dim in vectors of 4)
    int64_t off[kMaxOps];
    if (ONE_D) {
      // dims merged on the host: a dense 1-D walk, no division
      const int64_t i = VEC ? w * 4 : w;
#pragma unroll
      for (int k = 0; k < kMaxOps; ++k) off[k] = k < p.nops ? p.coef[k][0] * i : 0;
    } else {
      int64_t rem = w;
#pragma unroll
      for (int k = 0; k < kMaxOps; ++k) off[k] = 0;
      for (int d = p.nd - 1; d >= 0; --d) {
        const int64_t trip = (VEC && d == p.nd - 1) ? p.trip[d] / 4 : p.trip[d];
        int64_t i = rem % trip;
        rem /= trip;
        if (VEC && d == p.nd - 1) i *= 4;
#pragma unroll
        for (int k = 0; k < kMaxOps; ++k)
          if (k < p.nops) off[k] += p.coef[k][d] * i;
      }
    }
    float4 r[kMaxRegs];
    // hoisted loads: operand q feeds the q-th leading LD word; compile-time q
    // keeps them in registers, all NL loads in flight together
    float4 L[NL > 0 ? NL : 1];
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      const float *src = p.ptr[q] + off[q];
      if (VEC) {
        if (p.coef[q][p.nd - 1] == 1) L[q] = *reinterpret_cast<const float4 *>(src);
        else { const float v = *src; L[q] = make_float4(v, v, v, v); }
      } else {
        L[q].x = *src;
      }
    }
#pragma unroll
    for (int q = 0; q < NL; ++q) r[(p.prog[q] >> 8) & 0xff] = L[q];
    for (int pc = NL; pc < p.nwords;) {
      const int32_t w0 = p.prog[pc];
      const int op = w0 & 0xff, dst = (w0 >> 8) & 0xff, a = (w0 >> 16) & 0xff,
                b = (w0 >> 24) & 0xff;
      switch (op) {
        case M_LD: {
          const float *src = p.ptr[a] + off[a];
          if (VEC) {
            if (p.coef[a][p.nd - 1] == 1) r[dst] = *reinterpret_cast<const float4 *>(src);
            else { const float v = *src; r[dst] = make_float4(v, v, v, v); }
          } else {
            r[dst].x = *src;
          }
          pc += 1;
          break;
        }
        case M_CF: {
          const float c = p.consts[a];
          r[dst] = make_float4(c, c, c, c);
          pc += 1;
          break;
        }
        case M_BF: {
          const int f = p.prog[pc + 1];
          const float4 x = r[a], y = r[b];
          if (VEC) r[dst] = make_float4(fop(f, x.x, y.x), fop(f, x.y, y.y), fop(f, x.z, y.z),
                                        fop(f, x.w, y.w));
          else r[dst].x = fop(f, x.x, y.x);
          pc += 2;
          break;
        }
        default: {  // M_ST: operand a <- register dst
          float *d = p.ptr[a] + off[a];
          if (VEC) *reinterpret_cast<float4 *>(d) = r[dst];
          else *d = r[dst].x;
          pc += 1;
          break;
        }
      }
    }
  }
}

template <bool VEC, bool ONE_D>
void dispatch_vec(const MapParams &p, int nload, unsigned blocks, cudaStream_t s) {
  switch (nload) {
    case 1: map_kernel<VEC, ONE_D, 1><<<blocks, 256, 0, s>>>(p); break;
    case 2: map_kernel<VEC, ONE_D, 2><<<blocks, 256, 0, s>>>(p); break;
    case 3: map_kernel<VEC, ONE_D, 3><<<blocks, 256, 0, s>>>(p); break;
    case 4: map_kernel<VEC, ONE_D, 4><<<blocks, 256, 0, s>>>(p); break;
    default: map_kernel<VEC, ONE_D, 0><<<blocks, 256, 0, s>>>(p); break;
  }
}

void dispatch_nl(const MapParams &p, bool vec, bool one_d, int nload, unsigned blocks,
                 cudaStream_t s) {
  if (vec && one_d) dispatch_vec<true, true>(p, nload, blocks, s);
  else if (vec) dispatch_vec<true, false>(p, nload, blocks, s);
  else if (one_d) dispatch_vec<false, true>(p, nload, blocks, s);
  else dispatch_vec<false, false>(p, nload, blocks, s);
}

}  // namespace

extern "C" int b200_map_f32(const int32_t *prog, int32_t n_words, const float *consts,
                            int32_t n_consts, float *const *ptrs, const int64_t *coefs,
                            int32_t n_ops, const int64_t *trips, int32_t nd, int32_t vector,
                            int32_t nload, void *stream) {
  if (nd < 1 || nd > kMaxDims || n_ops < 1 || n_ops > kMaxOps || n_words > kMaxProg ||
      n_consts > kMaxConst)
    return B200_EINVAL;
  MapParams p{};
  int64_t total = 1;
  for (int d = 0; d < nd; ++d) {
    p.trip[d] = trips[d];
    total *= trips[d];
  }
  if (total == 0) return B200_OK;
  for (int k = 0; k < n_ops; ++k) {
    p.ptr[k] = ptrs[k];
    for (int d = 0; d < nd; ++d) p.coef[k][d] = coefs[k * nd + d];
  }
  for (int i = 0; i < n_words; ++i) p.prog[i] = prog[i];
  for (int i = 0; i < n_consts; ++i) p.consts[i] = consts[i];
  p.nd = nd;
  p.nops = n_ops;
  p.nwords = n_words;
  if (vector) {
    if (trips[nd - 1] % 4) return B200_EINVAL;
    total /= 4;
  }
  p.total = total;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dispatch_nl(p, vector != 0, nd == 1, nload, (unsigned)blocks, s);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

// ---------------------------------------------------------------------------
// The tuner's equivalence guard on the device (sweep.py): counts the
// elements of a trial's buffer that are NOT math.isclose(got, want,
// rel_tol, abs_tol) (reference tuner/search.py:128-138): equal values
// (infinities included) are close; otherwise both must be finite and
// |got - want| <= max(rel_tol * max(|got|, |want|), abs_tol); NaN is never
// close.  got: f32 or f64 (the trial's device copy), want: f64 (the
// baseline, cached on the device); the count is atomically added to *bad.
namespace {

template <typename T>
__global__ void guard_close_kernel(const T *__restrict__ got, const double *__restrict__ want,
                                   int64_t n, double rel, double abs_tol,
                                   unsigned long long *bad) {
  unsigned long long mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double g = (double)got[i], w = want[i];
    bool ok = g == w;
    if (!ok && isfinite(g) && isfinite(w)) {
      const double tol = fmax(rel * fmax(fabs(g), fabs(w)), abs_tol);
      ok = fabs(g - w) <= tol;
    }
    mine += ok ? 0 : 1;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(bad, mine);
}

}  // namespace

extern "C" int b200_guard_close(int32_t dtype, const void *got, const double *want, int64_t n,
                                double rel_tol, double abs_tol, unsigned long long *bad,
                                void *stream) {
  if (n < 0 || (n > 0 && (!got || !want || !bad))) return B200_EINVAL;
  if (n == 0) return B200_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == B200_F32)
    guard_close_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<const float *>(got), want, n, rel_tol, abs_tol, bad);
  else if (dtype == B200_F64)
    guard_close_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<const double *>(got), want, n, rel_tol, abs_tol, bad);
  else
    return B200_EINVAL;
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}
