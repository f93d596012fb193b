// Bit-exact contraction on the FP32/FP64 pipes of sm_100a.
//
// The reference computes every f32 product and sum in double and rounds it
// back to f32 (reference pkg/src/staircase/interp/_evalpy.py:115-127 and
// interp/_evalcy.pyx:122-136).  Double rounding is innocuous for + - * /
// (53 >= 2*24+2), so each op equals one IEEE f32 op; there is no FMA and the
// reduction runs in nest order.  These kernels perform exactly that chain per
// output — __fmul_rn/__fadd_rn (__dmul_rn/__dadd_rn for f64) cannot be
// contracted — so results are bit-identical to the reference for every shape,
// stride and tile config.
//
// Two operand addressings share one tiled core, both separable
// (offset = row part + column part):
//   * strided (b200_gemm_f32_exact): A[m*sAm + k*sAk] etc. — matmul nests;
//   * tables (b200_contract_exact): A[a_m[m] + a_k[k]], B[b_k[k] + b_n[n]],
//     C[c_m[m] + c_n[n]] — any contraction whose index maps split into
//     output-row / output-column / reduction variable groups, e.g. the
//     NCHW/FCHW convolution (reference tests/kernels.py:50-64) as an implicit
//     GEMM with M = (n, ho, wo), N = co, K = (ci, ki, kj) in nest order.
// Tiles (256 threads, register micro-tiles as 2x2 blocks of TM/2 x TN/2 so
// shared-memory reads are vector broadcasts): f32 128x128 (8x8) or, for
// narrow N (conv's F = 64), 256x64 (8x8); f64 64x64 (4x4).  BK = 16 with
// register double-buffered global->shared staging; loads are coalesced along
// whichever operand dimension has unit stride, and each thread's fixed row
// offset (the separable half) is looked up once per CTA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "../../include/b200k.h"
#include "tc_common.cuh"

namespace {

constexpr int BK = 16;
constexpr int kThreads = 256;

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Separable operand addressing: a(m,k) = am(m) + ak(k), etc.
struct Strided {
  int64_t sAm, sAk, sBk, sBn, sCm, sCn;
  bool a_k_fast, b_n_fast;
  __device__ __forceinline__ int64_t am(int64_t m) const { return m * sAm; }
  __device__ __forceinline__ int64_t ak(int64_t k) const { return k * sAk; }
  __device__ __forceinline__ int64_t bk(int64_t k) const { return k * sBk; }
  __device__ __forceinline__ int64_t bn(int64_t n) const { return n * sBn; }
  __device__ __forceinline__ int64_t c(int64_t m, int64_t n) const { return m * sCm + n * sCn; }
};
struct Tables {
  const int64_t *a_m, *a_k, *b_k, *b_n, *c_m, *c_n;
  bool a_k_fast, b_n_fast;
  int64_t sAm = 0, sBk = 0;   // unused: only the strided form takes the VEC path
  __device__ __forceinline__ int64_t am(int64_t m) const { return __ldg(a_m + m); }
  __device__ __forceinline__ int64_t ak(int64_t k) const { return __ldg(a_k + k); }
  __device__ __forceinline__ int64_t bk(int64_t k) const { return __ldg(b_k + k); }
  __device__ __forceinline__ int64_t bn(int64_t n) const { return __ldg(b_n + n); }
  __device__ __forceinline__ int64_t c(int64_t m, int64_t n) const {
    return __ldg(c_m + m) + __ldg(c_n + n);
  }
};

template <typename T, typename Addr>
struct Args {
  const T *A, *B;
  T *C;
  const T *bias;
  int64_t bias_stride;
  int64_t M, N, K;
  int init;
  T init_value;
  Addr ad;
  // linear tile order (ntn > 0): block b computes tile tile_base + b / sub of
  // the grid of (BM x sub BN) tiles, ntn of them per row, columns
  // (b % sub) BN .. +BN of it; otherwise the 2-D grid (blockIdx.y, .x)
  int64_t tile_base = 0, ntn = 0;
  int sub = 1;
};

// f32 8x8 micro-tiles are held to 128 registers so two CTAs share an SM:
// with one CTA (8 warps) the FP pipe starved on shared-memory latency (ncu:
// 12.5 % occupancy, 52 % issue-slot use).
template <typename T, int TM, int TN>
struct MinBlocks {
  static constexpr int value = (sizeof(T) == 4 && TM * TN >= 32) ? 2 : 1;
};

// VEC (strided f32 only): A k-contiguous and B n-contiguous with 16-byte
// aligned rows and K, N multiples of 4 — the tiles are staged with 16-byte
// global loads (A transposed into As by four scalar stores, B stored as is).
// Shared staging of one CTA: A (k-major, padded) and B double buffers.
template <typename T, int BM, int BN>
constexpr size_t smem_bytes() {
  return (size_t)2 * BK * ((BM + 16 / sizeof(T)) + BN) * sizeof(T);
}

template <typename T, typename Addr, int BM, int BN, int TM, int TN, bool VEC = false,
          int MINB = MinBlocks<T, TM, TN>::value>
__global__ void __launch_bounds__(kThreads, MINB)
    contract_exact_kernel(Args<T, Addr> g) {
  constexpr int PAD = 16 / sizeof(T);
  constexpr int LA = BM * BK / kThreads;  // A elements staged per thread
  constexpr int LB = BN * BK / kThreads;
  constexpr int HM = TM / 2, HN = TN / 2;  // micro-tile halves
  constexpr int TX = BN / TN;              // threads along n
  static_assert((BM / TM) * (BN / TN) == kThreads, "tile / thread mismatch");
  static_assert(kThreads % BM == 0 && kThreads % BN == 0, "fixed-row staging");
  static_assert(BM % 64 == 0 || !VEC, "VEC staging: rows t / 4 + 64 i");
  // dynamic shared memory (tiles above 48 KB of staging need the opt-in)
  extern __shared__ __align__(16) unsigned char smem_dyn[];
  auto As = reinterpret_cast<T (*)[BK][BM + PAD]>(smem_dyn);
  auto Bs = reinterpret_cast<T (*)[BK][BN]>(smem_dyn + (size_t)2 * BK * (BM + PAD) * sizeof(T));

  int64_t m0, n0;
  if (g.ntn > 0) {
    const int64_t tl = g.tile_base + blockIdx.x / g.sub;
    m0 = (tl / g.ntn) * BM;
    n0 = (tl % g.ntn) * ((int64_t)BN * g.sub) + (int64_t)(blockIdx.x % g.sub) * BN;
  } else {
    m0 = (int64_t)blockIdx.y * BM;
    n0 = (int64_t)blockIdx.x * BN;
  }
  const int t = threadIdx.x;
  const int tx = t % TX;
  const int ty = t / TX;
  auto row_of = [&](int i) { return i < HM ? ty * HM + i : BM / 2 + ty * HM + (i - HM); };
  auto col_of = [&](int j) { return j < HN ? tx * HN + j : BN / 2 + tx * HN + (j - HN); };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + row_of(i);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + col_of(j);
      T v = g.init_value;
      if (!g.init && m < g.M && n < g.N) v = g.C[g.ad.c(m, n)];
      acc[i][j] = v;
    }
  }

  // staging geometry.  m-fast A: this thread always stages row mm_fix and
  // k rows kk0 + i * (kThreads / BM); k-fast A: column kk_fix, rows vary.
  const bool afast = g.ad.a_k_fast, bfast = g.ad.b_n_fast;
  const int mm_fix = t % BM;
  const int kk_fix_a = t % BK;
  const int nn_fix = t % BN;
  const int kk_fix_b = t % BK;
  const int64_t m_fix = m0 + mm_fix;
  const int64_t n_fix = n0 + nn_fix;
  const int64_t arow_fix = (!afast && m_fix < g.M) ? g.ad.am(m_fix) : 0;
  const int64_t bcol_fix = (bfast && n_fix < g.N) ? g.ad.bn(n_fix) : 0;

  T ra[LA], rb[LB];
  // VEC: per-thread operand pointers (rows / columns fixed for the CTA)
  const float *vp_a[VEC ? LA / 4 : 1];
  bool vm_a[VEC ? LA / 4 : 1];
  const float *vp_b = nullptr;
  bool vm_b = false;
  if constexpr (VEC) {
#pragma unroll
    for (int i = 0; i < LA / 4; ++i) {
      const int64_t m = m0 + t / 4 + i * (kThreads / 4);
      vm_a[i] = m < g.M;
      vp_a[i] = reinterpret_cast<const float *>(g.A) + (vm_a[i] ? m : 0) * g.ad.sAm +
                4 * (t % 4);
    }
    const int64_t n = n0 + 4 * (t % (BN / 4));
    vm_b = n < g.N;
    vp_b = reinterpret_cast<const float *>(g.B) + (vm_b ? n : 0);
  }
  auto load = [&](int64_t k0) {
    if constexpr (VEC) {
      // A: LA / 4 vectors per thread (rows t / 4 + 64 i, k quad t % 4),
      // from per-thread row pointers set up once (vp_a below)
#pragma unroll
      for (int i = 0; i < LA / 4; ++i) {
        const float4 v = (vm_a[i] && k0 + 4 * (t % 4) < g.K)
                             ? __ldg(reinterpret_cast<const float4 *>(vp_a[i] + k0))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        ra[4 * i] = v.x, ra[4 * i + 1] = v.y, ra[4 * i + 2] = v.z, ra[4 * i + 3] = v.w;
      }
      // B goes straight to shared memory (cp.async, zero-filled past the
      // edges): no staging registers, so the 8x8 tile fits 128 registers
      const int buf = (int)((k0 / BK) & 1);
#pragma unroll
      for (int i = 0; i < LB / 4; ++i) {
        const int kr = t / (BN / 4) + i * (kThreads / (BN / 4)), nq = 4 * (t % (BN / 4));
        const bool ok = vm_b && k0 + kr < g.K;
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(&Bs[buf][kr][nq]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d),
                     "l"(ok ? vp_b + (k0 + kr) * g.ad.sBk : g.B), "r"(ok ? 16 : 0)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = t + i * kThreads;
      if (afast) {
        const int64_t m = m0 + e / BK, k = k0 + kk_fix_a;
        ra[i] = (m < g.M && k < g.K) ? __ldg(g.A + g.ad.am(m) + g.ad.ak(k)) : T(0);
      } else {
        const int64_t k = k0 + e / BM;
        ra[i] = (m_fix < g.M && k < g.K) ? __ldg(g.A + arow_fix + g.ad.ak(k)) : T(0);
      }
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = t + i * kThreads;
      if (bfast) {
        const int64_t k = k0 + e / BN;
        rb[i] = (n_fix < g.N && k < g.K) ? __ldg(g.B + g.ad.bk(k) + bcol_fix) : T(0);
      } else {
        const int64_t n = n0 + e / BK, k = k0 + kk_fix_b;
        rb[i] = (n < g.N && k < g.K) ? __ldg(g.B + g.ad.bk(k) + g.ad.bn(n)) : T(0);
      }
    }
  };
  auto store = [&](int buf) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < LA / 4; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          As[buf][4 * (t % 4) + u][t / 4 + i * (kThreads / 4)] = ra[4 * i + u];
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");   // this thread's B copies
      return;
    }
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = t + i * kThreads;
      if (afast) As[buf][kk_fix_a][e / BK] = ra[i];
      else As[buf][e / BM][mm_fix] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = t + i * kThreads;
      if (bfast) Bs[buf][e / BN][nn_fix] = rb[i];
      else Bs[buf][kk_fix_b][e / BK] = rb[i];
    }
  };

  const int64_t ktiles = (g.K + BK - 1) / BK;
  if (ktiles > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < ktiles) load((kt + 1) * BK);
    const int64_t krem = g.K - kt * BK;
    const int kn = krem >= BK ? BK : (int)krem;
    auto step = [&](int kk) {
      T av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < HM; ++i) {
        av[i] = As[cur][kk][ty * HM + i];
        av[HM + i] = As[cur][kk][BM / 2 + ty * HM + i];
      }
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        bv[j] = Bs[cur][kk][tx * HN + j];
        bv[HN + j] = Bs[cur][kk][BN / 2 + tx * HN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = add_rn(acc[i][j], mul_rn(av[i], bv[j]));
    };
    if (kn == BK) {
      // full k-tile: constant trip count, no remainder test (a full unroll
      // hoists too many operand loads: spills at 128 registers)
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) step(kk);
    } else {
#pragma unroll 1
      for (int kk = 0; kk < kn; ++kk) step(kk);
    }
    if (kt + 1 < ktiles) {
      store(cur ^ 1);   // cur^1 was last read before the previous barrier
      __syncthreads();
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + row_of(i);
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + col_of(j);
      if (n >= g.N) continue;
      T v = acc[i][j];
      if (g.bias) v = add_rn(v, __ldg(g.bias + n * g.bias_stride));
      g.C[g.ad.c(m, n)] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Whole-tile strided f32 kernel (the 4096^3 / Linear-stack shapes): M, N
// multiples of 128, K a multiple of 32, A k-contiguous and B n-contiguous
// with 16-byte aligned rows.  Same arithmetic as contract_exact_kernel (one
// __fmul_rn and one __fadd_rn per MAC, k ascending), different staging:
//   * both operands arrive by cp.async (16-byte, L2-only) in a 3-stage ring
//     of BK = 32 slices — no staging registers, one barrier per 32 k;
//   * A stays row-major in shared memory ([m][k], rows padded to 36 floats so
//     the two rows a warp reads sit 16 banks apart) and is read AK k at a
//     time per row (LDS.64 / LDS.128), B is read as two LDS.128 per k;
//   * no bounds tests and 32-bit shared addressing in the main loop.
// The generic kernel spent ~190 issue slots per 16-k slice on 64-bit index
// and bounds arithmetic (SASS; ~11 % of all issued instructions at 4096^3).
constexpr int FBM = 128, FBN = 128, FBK = 32, FSTAGES = 3, FAPAD = 36;
constexpr size_t kFullStageA = (size_t)FBM * FAPAD * 4;
constexpr size_t kFullStageB = (size_t)FBK * FBN * 4;
constexpr size_t kFullSmem = FSTAGES * (kFullStageA + kFullStageB);

__device__ __forceinline__ void cp_async16(uint32_t dst, const float *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int AK>
__global__ void __launch_bounds__(kThreads, 2) gemm_exact_full_kernel(Args<float, Strided> g) {
  extern __shared__ __align__(16) unsigned char smem_dyn[];
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dyn));
  const float *As = reinterpret_cast<const float *>(smem_dyn);
  const float *Bs = reinterpret_cast<const float *>(smem_dyn + FSTAGES * kFullStageA);
  const uint32_t sA0 = sbase, sB0 = sbase + (uint32_t)(FSTAGES * kFullStageA);

  int64_t m0, n0;
  if (g.ntn > 0) {
    const int64_t tl = g.tile_base + blockIdx.x;
    m0 = (tl / g.ntn) * FBM;
    n0 = (tl % g.ntn) * FBN;
  } else {
    m0 = (int64_t)blockIdx.y * FBM;
    n0 = (int64_t)blockIdx.x * FBN;
  }
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;

  // copy assignments: A chunk c = t + 256 i -> row c / 8, k quad c % 8;
  // B chunk c -> k row c / 32, n quad c % 32
  const float *ga = g.A + (m0 + t / 8) * g.ad.sAm + 4 * (t % 8);
  const int64_t ga_step = 32 * g.ad.sAm;   // rows t/8 + 32 i
  const float *gb = g.B + (int64_t)(t / 32) * g.ad.sBk + n0 + 4 * (t % 32);
  const int64_t gb_step = 8 * g.ad.sBk;    // k rows t/32 + 8 i
  const uint32_t da = (uint32_t)(((t / 8) * FAPAD + 4 * (t % 8)) * 4);
  const uint32_t db = (uint32_t)(((t / 32) * FBN + 4 * (t % 32)) * 4);
  auto load = [&](int64_t k0, int st) {
    const uint32_t a = sA0 + (uint32_t)(st * kFullStageA) + da;
    const uint32_t b = sB0 + (uint32_t)(st * kFullStageB) + db;
#pragma unroll
    for (int i = 0; i < 4; ++i) cp_async16(a + i * 32 * FAPAD * 4, ga + i * ga_step + k0);
    const float *pb = gb + k0 * g.ad.sBk;
#pragma unroll
    for (int i = 0; i < 4; ++i) cp_async16(b + i * 8 * FBN * 4, pb + i * gb_step);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      acc[i][j] = g.init ? g.init_value : g.C[g.ad.c(m, n)];
    }
  }

  const int64_t ktiles = g.K / FBK;
#pragma unroll
  for (int s = 0; s < FSTAGES - 1; ++s) {
    if (s < ktiles) load(s * FBK, s);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // this thread's first A row / B column inside a stage
  const int arow = ty * 4, bcol = tx * 4;
  int st = 0;
#pragma unroll 1
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(FSTAGES - 2) : "memory");
    __syncthreads();   // stage st complete for every thread; stage st-1 drained
    {
      const int64_t kn = kt + FSTAGES - 1;
      const int ls = st == 0 ? FSTAGES - 1 : st - 1;
      if (kn < ktiles) load(kn * FBK, ls);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const float *as = As + st * (kFullStageA / 4);
    const float *bs = Bs + st * (kFullStageB / 4);
#pragma unroll 2
    for (int kq = 0; kq < FBK; kq += AK) {
      float a[8][AK];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float *p = as + (i < 4 ? arow + i : 64 + arow + i - 4) * FAPAD + kq;
        if constexpr (AK == 4) {
          const float4 v = *reinterpret_cast<const float4 *>(p);
          a[i][0] = v.x, a[i][1] = v.y, a[i][2] = v.z, a[i][3] = v.w;
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(p);
          a[i][0] = v.x, a[i][1] = v.y;
        }
      }
#pragma unroll
      for (int u = 0; u < AK; ++u) {
        const float4 b0 = *reinterpret_cast<const float4 *>(bs + (kq + u) * FBN + bcol);
        const float4 b1 = *reinterpret_cast<const float4 *>(bs + (kq + u) * FBN + 64 + bcol);
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i][u], b[j]));
      }
    }
    st = st + 1 == FSTAGES ? 0 : st + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      float v = acc[i][j];
      if (g.bias) v = __fadd_rn(v, __ldg(g.bias + n * g.bias_stride));
      g.C[g.ad.c(m, n)] = v;
    }
  }
}

// TMA-fed whole-tile kernel (the default; B200_GEMM_EXACT_TMA=0 selects the
// cp.async kernel above): the same tile, micro-tile
// and arithmetic, but each stage is two TMA boxes (A 128 x 32, B 32 x 128)
// issued by thread 0 and tracked by mbarriers — no per-thread copy
// addressing and no CTA-wide barrier: a warp waits only for the stage it
// reads (full) and thread 0 refills a stage once all eight warps released it
// (empty), so the other warps run up to two stages ahead.  A rows are 128 B
// unpadded (a warp's two rows share banks: 2-way, the LSU absorbs it).
constexpr int TSTAGES = 3;
constexpr size_t kTmaStageA = (size_t)FBM * FBK * 4;   // 16 KB
constexpr size_t kTmaStageB = (size_t)FBK * FBN * 4;   // 16 KB

// Shared memory of the TMA kernel with an MI x NJ micro-tile per thread (a
// 16 MI x 16 NJ CTA tile) and STG stages.
constexpr size_t tma_smem(int mi, int nj, int stg) {
  return 1024 + (size_t)stg * ((size_t)16 * mi * FBK * 4 + (size_t)FBK * 16 * nj * 4) + 64;
}
constexpr size_t kTmaSmem = tma_smem(8, 8, TSTAGES);

// MI x NJ = 8 x 8 is the 128 x 128 CTA tile of untiled and (8, 8)-tiled
// nests; 4 x 16 (64 x 256) and 16 x 4 (256 x 64) are the tiles runtime.cta_tile
// gives (4, 16)- and (16, 4)-tiled ones.  Thread (tx, ty) owns rows
// 64 (i / 4) + 4 ty + i % 4 and columns 64 (j / 4) + 4 tx + j % 4: 16-byte
// shared loads, conflict-free across a warp.  The 40 KB stages of the
// non-square tiles come two per CTA (two CTAs per SM).
template <int AK, int UNR = 2, bool EAGER = false, int MI = 8, int NJ = 8, int STG = TSTAGES>
__global__ void __launch_bounds__(kThreads, MI * NJ >= 64 ? 2 : 4)
    gemm_exact_tma_kernel(const __grid_constant__ CUtensorMap tma_a,
                          const __grid_constant__ CUtensorMap tma_b, Args<float, Strided> g) {
  using namespace b200tc;
  constexpr int BM = 16 * MI, BN = 16 * NJ;
  constexpr size_t SA = (size_t)BM * FBK * 4, SB = (size_t)FBK * BN * 4;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  const uint32_t base = (smem_u32(smem_dyn) + 1023u) & ~1023u;
  unsigned char *gbase = smem_dyn + (base - smem_u32(smem_dyn));
  const float *As = reinterpret_cast<const float *>(gbase);
  const float *Bs = reinterpret_cast<const float *>(gbase + STG * SA);
  const uint32_t sA0 = base, sB0 = base + (uint32_t)(STG * SA);
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + STG * (SA + SB));
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int st) { return bar0 + 8u * st; };
  auto empty = [&](int st) { return bar0 + 8u * (STG + st); };

  // grouped raster: consecutive CTAs walk GROUP_M tile rows across all tile
  // columns, so a wave touches a few A panels and reuses B panels from L2.
  // DRAM bytes read at 4096^3 (ncu, one launch): row-major order 510 MB,
  // GROUP_M 8: 433, 16: 364, 32: 530 (A, B and C once: 192); compute-bound
  // either way (31.4 TFLOP/s for all of them)
  constexpr int64_t GROUP_M = 16;
  const int64_t mt = g.M / BM, nt = g.N / BN;
  const int64_t tl = blockIdx.x;
  const int64_t first_m = (tl / (GROUP_M * nt)) * GROUP_M;
  const int64_t gm = mt - first_m < GROUP_M ? mt - first_m : GROUP_M;
  const int64_t tin = tl % (GROUP_M * nt);
  const int64_t m0 = (first_m + tin % gm) * BM, n0 = (tin / gm) * BN;
  const int t = threadIdx.x, lane = t % 32;
  const int tx = t % 16, ty = t / 16;
  const int64_t ktiles = g.K / FBK;
  auto issue = [&](int64_t kt) {
    const int st = (int)(kt % STG);
    mbar_expect_tx(full(st), (uint32_t)(SA + SB));
    tma_load_2d(&tma_a, full(st), sA0 + st * (uint32_t)SA, (int32_t)(kt * FBK), (int32_t)m0);
    tma_load_2d(&tma_b, full(st), sB0 + st * (uint32_t)SB, (int32_t)n0, (int32_t)(kt * FBK));
  };
  if (t == 0) {
    for (int st = 0; st < STG; ++st) {
      mbar_init(full(st), 1);
      mbar_init(empty(st), kThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int64_t kt = 0; kt < STG && kt < ktiles; ++kt) issue(kt);

  auto row = [&](int i) { return (i >> 2) * 64 + ty * 4 + (i & 3); };
  auto col = [&](int j) { return (j >> 2) * 64 + tx * 4 + (j & 3); };
  float acc[MI][NJ];
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t m = m0 + row(i);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t n = n0 + col(j);
      acc[i][j] = g.init ? g.init_value : g.C[g.ad.c(m, n)];
    }
  }
  // stage / phase counters instead of kt % STG (a 64-bit division on the
  // integer pipe the FMULs / FADDs share)
  int st = 0, pst = STG - 1;
  uint32_t ph = 0, pph = 1;
  const int nk = (int)ktiles;
#pragma unroll 1
  for (int kt = 0; kt < nk; ++kt) {
    // thread 0 refills the stage every warp released one chunk ago (chunk
    // kt - 1 -> kt + STG - 1): waiting one chunk late lets warp 0 run a
    // chunk ahead of the slowest warp instead of stalling on it
    if (EAGER) {
    } else if (t == 0 && kt > 0 && kt - 1 + STG < nk) {
      mbar_wait(empty(pst), pph);
      issue(kt - 1 + STG);
    }
    mbar_wait(full(st), ph);
    const float *as = As + st * (SA / 4);
    const float *bs = Bs + st * (SB / 4);
#pragma unroll UNR
    for (int kq = 0; kq < FBK; kq += AK) {
      float a[MI][AK];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const float *p = as + row(i) * FBK + kq;
        if constexpr (AK == 4) {
          const float4 v = *reinterpret_cast<const float4 *>(p);
          a[i][0] = v.x, a[i][1] = v.y, a[i][2] = v.z, a[i][3] = v.w;
        } else {
          const float2 v = *reinterpret_cast<const float2 *>(p);
          a[i][0] = v.x, a[i][1] = v.y;
        }
      }
#pragma unroll
      for (int u = 0; u < AK; ++u) {
        float b[NJ];
#pragma unroll
        for (int q = 0; q < NJ / 4; ++q) {
          const float4 v = *reinterpret_cast<const float4 *>(bs + (kq + u) * BN + 64 * q + tx * 4);
          b[4 * q] = v.x, b[4 * q + 1] = v.y, b[4 * q + 2] = v.z, b[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i][u], b[j]));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty(st));
    if (EAGER && t == 0 && kt + STG < nk) {
      mbar_wait(empty(st), ph);   // every warp is done with this stage
      issue(kt + STG);
    }
    pst = st;
    pph = ph;
    if (++st == STG) { st = 0; ph ^= 1; }
  }

#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t m = m0 + row(i);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t n = n0 + col(j);
      float v = acc[i][j];
      if (g.bias) v = __fadd_rn(v, __ldg(g.bias + n * g.bias_stride));
      g.C[g.ad.c(m, n)] = v;
    }
  }
}

bool make_exact_maps(CUtensorMap *ma, CUtensorMap *mb, const Args<float, Strided> &g,
                     int bm = FBM, int bn = FBN) {
  using namespace b200tc;
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint32_t estr[2] = {1, 1};
  cuuint64_t da[2] = {(cuuint64_t)g.K, (cuuint64_t)g.M};
  cuuint64_t sa[1] = {(cuuint64_t)(g.ad.sAm * 4)};
  cuuint32_t ba[2] = {(cuuint32_t)FBK, (cuuint32_t)bm};
  cuuint64_t db[2] = {(cuuint64_t)g.N, (cuuint64_t)g.K};
  cuuint64_t sb[1] = {(cuuint64_t)(g.ad.sBk * 4)};
  cuuint32_t bb[2] = {(cuuint32_t)bn, (cuuint32_t)FBK};
  return enc(ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(g.A), da, sa, ba, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS &&
         enc(mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(g.B), db, sb, bb, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS;
}

// One whole-tile TMA launch of the MI x NJ kernel (grid = the tiles), or 1
// when its tensor maps do not apply (the caller falls back).
template <int AK, int MI, int NJ, int STG, bool EAGER = false, int UNR = 2>
int launch_tma_shape(const Args<float, Strided> &g, void *stream) {
  constexpr int BM = 16 * MI, BN = 16 * NJ;
  CUtensorMap ma, mb;
  if (!make_exact_maps(&ma, &mb, g, BM, BN)) return 1;
  auto k = gemm_exact_tma_kernel<AK, UNR, EAGER, MI, NJ, STG>;
  constexpr size_t smem = tma_smem(MI, NJ, STG);
  static_assert((MI * NJ >= 64 ? 2 : 4) * smem <= 232448, "CTAs per SM");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t tiles = (g.M / BM) * (g.N / BN);
  if (tiles >= (int64_t(1) << 31)) return 1;
  k<<<(unsigned)tiles, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(ma, mb, g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

int launch_tma(const Args<float, Strided> &g, void *stream) {
  // (measured at 4096^3: <AK 4, unroll 2> 31.4 TFLOP/s, <2, 2> 31.3, <4, 4>
  // 29.9 — it spills)
  const char *ev = getenv("B200_GEMM_EXACT_EAGER");   // dev A/B: refill right after release
  if (ev && ev[0] == '1') return launch_tma_shape<4, 8, 8, TSTAGES, true>(g, stream);
  return launch_tma_shape<4, 8, 8, TSTAGES>(g, stream);
}

inline bool full_ok(const Args<float, Strided> &g, int bm = FBM, int bn = FBN) {
  const auto &a = g.ad;
  return a.sAk == 1 && a.sBn == 1 && g.M % bm == 0 && g.N % bn == 0 && g.K % FBK == 0 &&
         g.K > 0 && a.sAm % 4 == 0 && a.sBk % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(g.B) & 15) == 0 && g.M / bm <= 65535;
}

int launch_full(const Args<float, Strided> &g, void *stream) {
  const char *tv = getenv("B200_GEMM_EXACT_TMA");   // dev A/B: "0" = cp.async kernel
  const bool tma = !(tv && tv[0] == '0');
  if (tma && g.ntn == 0) {
    const int rc = launch_tma(g, stream);
    if (rc != 1) return rc;   // 1: a tensor map the driver refused -> the cp.async kernel
  }
  static int ak = -1;
  if (ak < 0) {
    const char *e = getenv("B200_GEMM_EXACT_AK");   // dev A/B knob
    ak = (e && atoi(e) == 2) ? 2 : 4;
  }
  auto k = ak == 2 ? gemm_exact_full_kernel<2> : gemm_exact_full_kernel<4>;
  static bool attr[2] = {false, false};
  if (!attr[ak == 2]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFullSmem);
    attr[ak == 2] = true;
  }
  dim3 grid((unsigned)(g.N / FBN), (unsigned)(g.M / FBM));
  k<<<grid, kThreads, kFullSmem, static_cast<cudaStream_t>(stream)>>>(g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

template <typename T, typename Addr, int BM, int BN, int TM, int TN, bool VEC, int MINB>
void *kernel_ptr() {
  auto k = contract_exact_kernel<T, Addr, BM, BN, TM, TN, VEC, MINB>;
  constexpr size_t smem = smem_bytes<T, BM, BN>();
  if (smem > 48 * 1024) {
    static bool done = false;   // opt in once per instantiation
    if (!done) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      done = true;
    }
  }
  return reinterpret_cast<void *>(k);
}

template <typename T, typename Addr, int BM, int BN, int TM, int TN, bool VEC = false,
          int MINB = MinBlocks<T, TM, TN>::value>
int launch_tile(const Args<T, Addr> &g, void *stream) {
  dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM));
  if (grid.y > 65535u) return B200_EINVAL;
  kernel_ptr<T, Addr, BM, BN, TM, TN, VEC, MINB>();
  contract_exact_kernel<T, Addr, BM, BN, TM, TN, VEC, MINB>
      <<<grid, kThreads, smem_bytes<T, BM, BN>(), static_cast<cudaStream_t>(stream)>>>(g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

template <typename T, typename Addr, int BM, int BN, int TM, int TN, bool VEC = false,
          int MINB = MinBlocks<T, TM, TN>::value>
int launch_linear(const Args<T, Addr> &g, int64_t blocks, void *stream) {
  if (blocks <= 0) return B200_OK;
  if (blocks >= (int64_t(1) << 31)) return B200_EINVAL;
  kernel_ptr<T, Addr, BM, BN, TM, TN, VEC, MINB>();
  contract_exact_kernel<T, Addr, BM, BN, TM, TN, VEC, MINB>
      <<<(unsigned)blocks, kThreads, smem_bytes<T, BM, BN>(),
         static_cast<cudaStream_t>(stream)>>>(g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// 128 x 128 tiles.  Optional balanced last round (B200_GEMM_EXACT_TAIL=1):
// 2 CTAs per SM give S slots; T = q S + r tiles run as q full rounds of whole
// tiles and, when 2 r <= S, one round of 2 r half-width (128 x 64, 8 x 4 per
// thread) tiles.  Measured at 4096^3 (1024 tiles, S = 296): no gain (5.12 vs
// 5.08 ms) — a CTA left alone on an SM in the last round runs faster, so the
// last round is not a whole round's time — hence off by default.  Every
// output keeps its full-K chain either way.
template <typename Addr, bool VEC>
int launch_128(const Args<float, Addr> &g, void *stream) {
  const int64_t tn = (g.N + 127) / 128, tiles = ((g.M + 127) / 128) * tn;
  const int64_t slots = 2 * (int64_t)sm_count();
  const int64_t rem = tiles % slots;
  if (tiles <= slots || rem == 0 || 2 * rem > slots || !getenv("B200_GEMM_EXACT_TAIL"))
    return launch_tile<float, Addr, 128, 128, 8, 8, VEC>(g, stream);
  Args<float, Addr> g1 = g, g2 = g;
  g1.ntn = tn, g1.tile_base = 0, g1.sub = 1;
  g2.ntn = tn, g2.tile_base = tiles - rem, g2.sub = 2;
  const int rc = launch_linear<float, Addr, 128, 128, 8, 8, VEC>(g1, tiles - rem, stream);
  if (rc != B200_OK) return rc;
  return launch_linear<float, Addr, 128, 64, 8, 4, VEC>(g2, 2 * rem, stream);
}

// 16-byte staging applies (see contract_exact_kernel's VEC)
inline bool vec_ok(const Args<float, Strided> &g) {
  const auto &a = g.ad;
  return a.sAk == 1 && a.sBn == 1 && a.sAm % 4 == 0 && a.sBk % 4 == 0 && g.K % 4 == 0 &&
         g.N % 4 == 0 && (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(g.B) & 15) == 0 && !getenv("B200_GEMM_EXACT_NOVEC");
}

template <typename Addr>
int launch(const Args<float, Addr> &g, void *stream) {
  if (g.M < 0 || g.N < 0 || g.K < 0) return B200_EINVAL;
  if (g.M == 0 || g.N == 0) return B200_OK;
  // tile choice: big tiles amortise staging; when they would leave most SMs
  // idle (or compute mostly padding) use smaller ones — each output's
  // k-chain is identical for every tile shape, so results do not change.
  const int64_t big_ctas = ((g.M + 127) / 128) * ((g.N + 127) / 128);
  if (g.M * g.N <= 64 * 64) return launch_tile<float, Addr, 32, 32, 2, 2>(g, stream);
  if (big_ctas < 148) return launch_tile<float, Addr, 64, 64, 4, 4>(g, stream);
  if (g.N <= 64) return launch_tile<float, Addr, 256, 64, 8, 8>(g, stream);
  // (measured at 4096^3, tools/probe_exact.py: one CTA per SM with 255
  // registers — 128x128, 128x256 at 8x16 or 256x128 at 16x8 per thread —
  // ran 7-17 % slower than two 128-register CTAs: the FMUL -> FADD and LDS
  // latencies need the second CTA's warps more than the extra registers)
  if constexpr (std::is_same<Addr, Strided>::value) {
    if (full_ok(g) && !getenv("B200_GEMM_EXACT_OLD")) return launch_full(g, stream);
    if (vec_ok(g)) return launch_128<Addr, true>(g, stream);
  }
  return launch_128<Addr, false>(g, stream);
}

// An explicit CTA tile (b200_gemm_f32_exact_tiled): the tile sizes of a
// tiled nest pick the CTA tile shape (paper_2307_16080_b200/runtime.py
// cta_tile).  Every shape computes each output's k-chain identically.
int launch_cta(const Args<float, Strided> &g, int cta_m, int cta_n, void *stream) {
  if (g.M < 0 || g.N < 0 || g.K < 0) return B200_EINVAL;
  if (g.M == 0 || g.N == 0) return B200_OK;
  const bool vec = vec_ok(g);
  if (cta_m == 128 && cta_n == 128 && full_ok(g) && !getenv("B200_GEMM_EXACT_OLD"))
    return launch_full(g, stream);
  if (cta_m == 128 && cta_n == 128)
    return vec ? launch_tile<float, Strided, 128, 128, 8, 8, true>(g, stream)
               : launch_tile<float, Strided, 128, 128, 8, 8>(g, stream);
  // whole-tile shapes: the TMA kernel with a 4 x 16 / 16 x 4 micro-tile
  // (round 2; the general kernel measured 26.8 / 24.9 TFLOP/s at 4096^3)
  const bool tma = !getenv("B200_GEMM_EXACT_OLD");
  if (cta_m == 64 && cta_n == 256 && tma && g.ntn == 0 && full_ok(g, 64, 256)) {
    const int rc = launch_tma_shape<4, 4, 16, 2>(g, stream);   // 31.8 TFLOP/s
    if (rc != 1) return rc;
  }
  if (cta_m == 256 && cta_n == 64 && tma && g.ntn == 0 && full_ok(g, 256, 64)) {
    // <AK 2, unroll 1>: 29.5 TFLOP/s (<1, 1> 28.8, <2, 2> 27.6: a 16-row
    // micro-tile's A operands crowd the 128 registers)
    const int rc = launch_tma_shape<2, 16, 4, 2, false, 1>(g, stream);
    if (rc != 1) return rc;
  }
  if (cta_m == 64 && cta_n == 64 && tma && g.ntn == 0 && full_ok(g, 64, 64)) {
    const int rc = launch_tma_shape<4, 4, 4, 3>(g, stream);   // four CTAs per SM
    if (rc != 1) return rc;
  }
  if (cta_m == 64 && cta_n == 256)
    return vec ? launch_tile<float, Strided, 64, 256, 8, 8, true>(g, stream)
               : launch_tile<float, Strided, 64, 256, 8, 8>(g, stream);
  if (cta_m == 256 && cta_n == 64)
    return vec ? launch_tile<float, Strided, 256, 64, 8, 8, true>(g, stream)
               : launch_tile<float, Strided, 256, 64, 8, 8>(g, stream);
  if (cta_m == 64 && cta_n == 64) return launch_tile<float, Strided, 64, 64, 4, 4>(g, stream);
  if (cta_m == 32 && cta_n == 32) return launch_tile<float, Strided, 32, 32, 2, 2>(g, stream);
  return B200_EUNSUPPORTED;
}

template <typename Addr>
int launch(const Args<double, Addr> &g, void *stream) {
  if (g.M < 0 || g.N < 0 || g.K < 0) return B200_EINVAL;
  if (g.M == 0 || g.N == 0) return B200_OK;
  return launch_tile<double, Addr, 64, 64, 4, 4>(g, stream);
}

}  // namespace

extern "C" int b200_gemm_f32_exact(const float *A, int64_t sAm, int64_t sAk, const float *B,
                                   int64_t sBk, int64_t sBn, float *C, int64_t sCm, int64_t sCn,
                                   int64_t M, int64_t N, int64_t K, int32_t init,
                                   float init_value, const float *bias, int64_t bias_stride,
                                   void *stream) {
  Args<float, Strided> g{A, B, C, bias, bias_stride, M, N, K, init, init_value,
                         Strided{sAm, sAk, sBk, sBn, sCm, sCn, sAk == 1, sBn == 1}};
  return launch(g, stream);
}

extern "C" int b200_gemm_f32_exact_tiled(const float *A, int64_t sAm, int64_t sAk,
                                         const float *B, int64_t sBk, int64_t sBn, float *C,
                                         int64_t sCm, int64_t sCn, int64_t M, int64_t N,
                                         int64_t K, int32_t init, float init_value,
                                         const float *bias, int64_t bias_stride, int32_t cta_m,
                                         int32_t cta_n, void *stream) {
  Args<float, Strided> g{A, B, C, bias, bias_stride, M, N, K, init, init_value,
                         Strided{sAm, sAk, sBk, sBn, sCm, sCn, sAk == 1, sBn == 1}};
  if (cta_m <= 0 || cta_n <= 0) return launch(g, stream);
  return launch_cta(g, cta_m, cta_n, stream);
}

extern "C" int b200_contract_exact(int32_t dtype, const void *A, const int64_t *a_m,
                                   const int64_t *a_k, const void *B, const int64_t *b_k,
                                   const int64_t *b_n, void *C, const int64_t *c_m,
                                   const int64_t *c_n, int64_t M, int64_t N, int64_t K,
                                   int32_t a_k_fast, int32_t b_n_fast, int32_t init,
                                   double init_value, const void *bias, int64_t bias_stride,
                                   void *stream) {
  Tables t{a_m, a_k, b_k, b_n, c_m, c_n, a_k_fast != 0, b_n_fast != 0};
  if (dtype == B200_F32) {
    Args<float, Tables> g{static_cast<const float *>(A), static_cast<const float *>(B),
                          static_cast<float *>(C), static_cast<const float *>(bias), bias_stride,
                          M, N, K, init, (float)init_value, t};
    return launch(g, stream);
  }
  if (dtype == B200_F64) {
    Args<double, Tables> g{static_cast<const double *>(A), static_cast<const double *>(B),
                           static_cast<double *>(C), static_cast<const double *>(bias),
                           bias_stride, M, N, K, init, init_value, t};
    return launch(g, stream);
  }
  return B200_EUNSUPPORTED;
}
