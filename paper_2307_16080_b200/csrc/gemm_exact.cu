// Bit-exact fp32 contraction on the FP32 pipes of sm_100a.
//
// The reference computes every f32 product and sum in double and rounds it
// back to f32 (reference pkg/src/staircase/interp/_evalpy.py:115-127 and
// interp/_evalcy.pyx:122-136).  Double rounding is innocuous for + - * /
// (53 >= 2*24+2), so each op equals one IEEE f32 op; there is no FMA and the
// reduction runs k-ascending.  This kernel performs exactly that chain per
// output — __fmul_rn/__fadd_rn cannot be contracted — so results are
// bit-identical to the reference for every shape, stride and tile config.
//
// Tiling: 128x128 CTA tile, BK = 16, 256 threads each owning an 8x8 register
// micro-tile (split as 2x2 blocks of 4x4 so shared-memory reads are
// conflict-free float4 broadcasts); global->shared staging is register
// double-buffered so the next k-tile's loads overlap the current tile's math.
// Operands are arbitrary-strided (the recogniser hands over the affine index
// maps of the nest), loads are coalesced along whichever dimension has unit
// stride.  Epilogue: optional init value (the fill/copy nests of the Linear
// lowering) and optional bias add,
// each a separately rounded f32 op in reference order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"

namespace {

constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8;
constexpr int kThreads = 256;
constexpr int APAD = 4;   // As row padding: conflict-light transposed stores

struct GemmArgs {
  const float *A, *B;
  float *C;
  const float *bias;
  int64_t sAm, sAk, sBk, sBn, sCm, sCn, bias_stride;
  int64_t M, N, K;
  int init;
  float init_value;
};

// Each thread stages 8 A elements and 8 B elements per k-tile.
__device__ __forceinline__ void load_tile(const GemmArgs &g, int64_t m0, int64_t n0, int64_t k0,
                                          float (&ra)[8], float (&rb)[8]) {
  const int t = threadIdx.x;
  // A tile: BM x BK = 2048 elements.  If A is k-contiguous walk k fastest.
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int e = t + i * kThreads;
    int mm, kk;
    if (g.sAk == 1) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
    int64_t m = m0 + mm, k = k0 + kk;
    ra[i] = (m < g.M && k < g.K) ? __ldg(g.A + m * g.sAm + k * g.sAk) : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int e = t + i * kThreads;
    int nn, kk;
    if (g.sBn == 1) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
    int64_t n = n0 + nn, k = k0 + kk;
    rb[i] = (n < g.N && k < g.K) ? __ldg(g.B + k * g.sBk + n * g.sBn) : 0.0f;
  }
}

__device__ __forceinline__ void store_tile(const GemmArgs &g, float (*As)[BM + APAD], float (*Bs)[BN],
                                           const float (&ra)[8], const float (&rb)[8]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int e = t + i * kThreads;
    int mm, kk;
    if (g.sAk == 1) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
    As[kk][mm] = ra[i];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int e = t + i * kThreads;
    int nn, kk;
    if (g.sBn == 1) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
    Bs[kk][nn] = rb[i];
  }
}

__global__ void __launch_bounds__(kThreads) gemm_exact_kernel(GemmArgs g) {
  __shared__ __align__(16) float As[2][BK][BM + APAD];
  __shared__ __align__(16) float Bs[2][BK][BN];

  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int tx = threadIdx.x % 16;   // n direction
  const int ty = threadIdx.x / 16;   // m direction
  // micro-tile rows: ty*4 + {0..3} and 64 + ty*4 + {0..3}; cols likewise.
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      float v = g.init_value;
      if (!g.init && m < g.M && n < g.N) v = g.C[m * g.sCm + n * g.sCn];
      acc[i][j] = v;
    }
  }

  float ra[8], rb[8];
  const int64_t ktiles = (g.K + BK - 1) / BK;
  load_tile(g, m0, n0, 0, ra, rb);
  store_tile(g, As[0], Bs[0], ra, rb);
  __syncthreads();

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < ktiles) load_tile(g, m0, n0, (kt + 1) * BK, ra, rb);
    const int64_t krem = g.K - kt * BK;
    if (krem >= BK) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float4 a0 = *reinterpret_cast<const float4 *>(&As[cur][kk][ty * 4]);
        float4 a1 = *reinterpret_cast<const float4 *>(&As[cur][kk][64 + ty * 4]);
        float4 b0 = *reinterpret_cast<const float4 *>(&Bs[cur][kk][tx * 4]);
        float4 b1 = *reinterpret_cast<const float4 *>(&Bs[cur][kk][64 + tx * 4]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
      }
    } else {
      for (int kk = 0; kk < krem; ++kk) {
        float av[8], bv[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          av[i] = As[cur][kk][ty * 4 + i];
          av[4 + i] = As[cur][kk][64 + ty * 4 + i];
          bv[i] = Bs[cur][kk][tx * 4 + i];
          bv[4 + i] = Bs[cur][kk][64 + tx * 4 + i];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
      }
    }
    if (kt + 1 < ktiles) {
      store_tile(g, As[cur ^ 1], Bs[cur ^ 1], ra, rb);
      __syncthreads();
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.bias) v = __fadd_rn(v, __ldg(g.bias + n * g.bias_stride));
      g.C[m * g.sCm + n * g.sCn] = v;
    }
  }
}

}  // namespace

extern "C" int b200_gemm_f32_exact(const float *A, int64_t sAm, int64_t sAk, const float *B,
                                   int64_t sBk, int64_t sBn, float *C, int64_t sCm, int64_t sCn,
                                   int64_t M, int64_t N, int64_t K, int32_t init,
                                   float init_value, const float *bias, int64_t bias_stride,
                                   void *stream) {
  if (M < 0 || N < 0 || K < 0) return B200_EINVAL;
  if (M == 0 || N == 0) return B200_OK;
  GemmArgs g{A, B, C, bias, sAm, sAk, sBk, sBn, sCm, sCn, bias_stride, M, N, K, init, init_value};
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  if (grid.y > 65535) return B200_EINVAL;
  gemm_exact_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}
