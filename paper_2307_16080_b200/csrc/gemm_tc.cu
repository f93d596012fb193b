// Tensor-core contraction for sm_100a: TMA -> SMEM -> tcgen05.mma -> TMEM.
//
// C[m,n] = (init ? init_value : C[m,n]) + sum_k A[m,k] * B[k,n]  (+ bias[n])
//
// Replaces run_tape on a recognised matmul / Linear contraction nest
// (reference tests/kernels.py:24-38) when the engine runs
// with precision "bf16" or "tf32".  Products of bf16/tf32 inputs are exact in
// fp32; the tensor core accumulates in fp32 in K order, so the only deviation
// from the reference's sequential f32 chain is accumulation rounding (bound
// stated in DESIGN.md and tests/test_gpu_tc.py).
//
// Two schedules share the operand format (K-major, 128B-swizzled TMA boxes):
//   * gemm_tc2.cu — CTA pair, UMMA 256x256 (cta_group::2): the default for
//     large problems (half the per-SM shared-memory traffic);
//   * this file — single CTA, UMMA 128x256 (cta_group::1): small problems
//     (fewer than ~2 waves of 256x256 tiles) and tests.
// Single-CTA structure (one CTA per SM, persistent over output tiles):
//   warp 0        TMA producer, 4-stage mbarrier ring (A 16 KB + B 32 KB)
//   warp 1        MMA issuer (one lane): 4 x tcgen05.mma per stage
//   warp 2        TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4..7    epilogue: tcgen05.ld 32x32b.x32 -> +C / init, +bias ->
//                 128-bit global stores; releases the TMEM buffer so the MMA
//                 of tile i+1 overlaps the epilogue of tile i
// Operands are packed K-major by b200_pack_operand (convert / transpose).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"
#include "tc_common.cuh"

using namespace b200tc;

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * 128;  // 16 KB
constexpr int B_STAGE = BN * 128;  // 32 KB
constexpr int TMEM_COLS = 512;
constexpr int kThreads = 256;
constexpr size_t SMEM_BYTES = 1024 + STAGES * (A_STAGE + B_STAGE) + 256;

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   Epi ep, int64_t M, int64_t N, int64_t K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * A_STAGE;
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + STAGES * (A_STAGE + B_STAGE));
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  constexpr int ELEM = KIND == 0 ? 2 : 4;
  constexpr int BK = 128 / ELEM;  // elements of K per stage
  constexpr int UK = 32 / ELEM;   // K per tcgen05.mma (32 bytes)

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
  const int64_t tiles = mt * nt;
  const int64_t kb_total = (K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int32_t m0 = (int32_t)((t / nt) * BM), n0 = (int32_t)((t % nt) * BN);
        for (int64_t kb = 0; kb < kb_total; ++kb) {
          mbar_wait(empty(s), ph ^ 1);
          mbar_expect_tx(full(s), A_STAGE + B_STAGE);
          tma_load_2d(&tma_a, full(s), sA + s * A_STAGE, (int32_t)(kb * BK), m0);
          tma_load_2d(&tma_b, full(s), sB + s * B_STAGE, (int32_t)(kb * BK), n0);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int64_t kb = 0; kb < kb_total; ++kb) {
          mbar_wait(full(s), ph);
          tc_fence_after();
          const uint32_t a_addr = sA + s * A_STAGE, b_addr = sB + s * B_STAGE;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma<KIND, 1>(tmem_d, smem_desc(a_addr + 32 * k), smem_desc(b_addr + 32 * k), idesc,
                          (kb | k) != 0);
          umma_commit(empty(s));
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter of this warp
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t m0 = (t / nt) * BM, n0 = (t % nt) * BN;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int64_t m = m0 + q * 32 + lane;
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(trow + (uint32_t)(c * 32), r);
        epilogue_row32(ep, m, n0 + c * 32, M, N, r);
      }
      tc_fence_before();
      mbar_arrive(tempty(acc));
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// -- operand packing: dst[r][c] (row-major, K-major for the GEMM) --------------

template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ float cvt<float>(float v) {
  // round-to-nearest-even to tf32 (10 explicit mantissa bits), NaN/Inf kept
  uint32_t u = __float_as_uint(v);
  if ((u & 0x7f800000u) != 0x7f800000u) {
    u += 0xfffu + ((u >> 13) & 1u);
    u &= 0xffffe000u;
  }
  return __uint_as_float(u);
}

// Split packing for the fp32-accurate "f32x3" contraction (3xTF32): x =
// hi + lo + d with hi = tf32(x), lo = tf32(x - hi) (x - hi is exact in f32),
// |d| <= 2^-22 |x|.  A row of the packed operand holds three K-segments, so
// one tf32 GEMM over K' = 3K sums hiA.hiB + hiA.loB + loA.hiB (the dropped
// loA.loB is <= 2^-22 |ab|): SPLIT 1 writes [hi | hi | lo] (the A operand),
// SPLIT 2 writes [hi | lo | hi] (B^T).  SPLIT 0 is the plain pack.
template <int SPLIT>
__device__ __forceinline__ void seg_offsets(int64_t cols, int64_t &hi0, int64_t &hi1,
                                            int64_t &lo) {
  if (SPLIT == 1) hi0 = 0, hi1 = cols, lo = 2 * cols;
  else hi0 = 0, hi1 = 2 * cols, lo = cols;
}

// 8 consecutive converted elements of row r, columns c .. c + 7 (16-byte
// aligned destination rows of pitch ld)
template <typename T, int SPLIT>
__device__ __forceinline__ void store8(T *__restrict__ dst, int64_t r, int64_t c, int64_t cols,
                                       int64_t ld, const float v[8]) {
  if constexpr (SPLIT == 0) {
    if (sizeof(T) == 2) {
      __nv_bfloat162 o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      *reinterpret_cast<uint4 *>(dst + r * ld + c) = *reinterpret_cast<uint4 *>(o);
    } else {
      float4 *d = reinterpret_cast<float4 *>(reinterpret_cast<float *>(dst) + r * ld + c);
      d[0] = make_float4(cvt<float>(v[0]), cvt<float>(v[1]), cvt<float>(v[2]), cvt<float>(v[3]));
      d[1] = make_float4(cvt<float>(v[4]), cvt<float>(v[5]), cvt<float>(v[6]), cvt<float>(v[7]));
    }
  } else {
    float hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hi[j] = cvt<float>(v[j]);
      lo[j] = cvt<float>(__fsub_rn(v[j], hi[j]));
    }
    int64_t o_hi0, o_hi1, o_lo;
    seg_offsets<SPLIT>(cols, o_hi0, o_hi1, o_lo);
    float *row = reinterpret_cast<float *>(dst) + r * ld + c;
    const float4 h0 = make_float4(hi[0], hi[1], hi[2], hi[3]);
    const float4 h1 = make_float4(hi[4], hi[5], hi[6], hi[7]);
    const float4 l0 = make_float4(lo[0], lo[1], lo[2], lo[3]);
    const float4 l1 = make_float4(lo[4], lo[5], lo[6], lo[7]);
    reinterpret_cast<float4 *>(row + o_hi0)[0] = h0;
    reinterpret_cast<float4 *>(row + o_hi0)[1] = h1;
    reinterpret_cast<float4 *>(row + o_hi1)[0] = h0;
    reinterpret_cast<float4 *>(row + o_hi1)[1] = h1;
    reinterpret_cast<float4 *>(row + o_lo)[0] = l0;
    reinterpret_cast<float4 *>(row + o_lo)[1] = l1;
  }
}

template <typename T, int SPLIT>
__device__ __forceinline__ void store1(T *__restrict__ dst, int64_t r, int64_t c, int64_t cols,
                                       int64_t ld, float v) {
  if constexpr (SPLIT == 0) {
    dst[r * ld + c] = cvt<T>(v);
  } else {
    const float hi = cvt<float>(v), lo = cvt<float>(__fsub_rn(v, hi));
    int64_t o_hi0, o_hi1, o_lo;
    seg_offsets<SPLIT>(cols, o_hi0, o_hi1, o_lo);
    float *row = reinterpret_cast<float *>(dst) + r * ld + c;
    row[o_hi0] = hi;
    row[o_hi1] = hi;
    row[o_lo] = lo;
  }
}

// Row-contiguous source (s_col == 1, rows 16-byte aligned): 8 elements per
// thread, 2 x 128-bit loads -> one 128-bit (bf16) or two (tf32) stores.
template <typename T, int SPLIT = 0>
__global__ void __launch_bounds__(256) pack_rows_kernel(const float *__restrict__ src, int64_t s_row,
                                                        T *__restrict__ dst, int64_t rows,
                                                        int64_t cols, int64_t ld) {
  const int64_t per_row = cols / 8;
  const int64_t total = rows * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row, c = (i % per_row) * 8;
    const float4 *s = reinterpret_cast<const float4 *>(src + r * s_row + c);
    float4 a = __ldcs(s), b = __ldcs(s + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    store8<T, SPLIT>(dst, r, c, cols, ld, v);
  }
}

// Column-contiguous source (s_row == 1): a 64 x 64 tile transposed through
// shared memory; 128-bit coalesced loads along the source rows and 128-bit
// coalesced stores along the destination rows.
template <typename T, int SPLIT = 0>
__global__ void __launch_bounds__(256) pack_transpose_kernel(const float *__restrict__ src,
                                                             int64_t s_col, T *__restrict__ dst,
                                                             int64_t rows, int64_t cols,
                                                             int64_t ld) {
  __shared__ float tile[64][65];  // [c][r]
  const int64_t r0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  const int t = threadIdx.x;
  // load: source row c (dst column) holds dst rows r contiguously
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = t + i * 256;   // 0..1023 float4 slots: 64 c x 16 float4
    const int cc = e / 16, rr = (e % 16) * 4;
    const int64_t c = c0 + cc, r = r0 + rr;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < cols && r + 3 < rows) {
      v = __ldcs(reinterpret_cast<const float4 *>(src + c * s_col + r));
    } else if (c < cols) {
      float tmp[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < 4; ++j)
        if (r + j < rows) tmp[j] = src[c * s_col + r + j];
      v = make_float4(tmp[0], tmp[1], tmp[2], tmp[3]);
    }
    tile[cc][rr + 0] = v.x;
    tile[cc][rr + 1] = v.y;
    tile[cc][rr + 2] = v.z;
    tile[cc][rr + 3] = v.w;
  }
  __syncthreads();
  // store: each thread writes 8 consecutive dst columns of one dst row
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int e = t + i * 256;   // 0..511: 64 r x 8 chunks of 8
    const int rr = e / 8, cc = (e % 8) * 8;
    const int64_t r = r0 + rr, c = c0 + cc;
    if (r >= rows) continue;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = tile[cc + j][rr];
    if (c + 7 < cols && ((cols % 8) == 0)) {
      store8<T, SPLIT>(dst, r, c, cols, ld, v);
    } else {
      for (int j = 0; j < 8; ++j)
        if (c + j < cols) store1<T, SPLIT>(dst, r, c + j, cols, ld, v[j]);
    }
  }
}

// General strides: 32x32 tiles through shared memory.
template <typename T, int SPLIT = 0>
__global__ void pack_kernel(const float *__restrict__ src, int64_t s_row, int64_t s_col,
                            T *__restrict__ dst, int64_t rows, int64_t cols, int64_t ld) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const bool row_fast = s_col != 1 && s_row == 1;
  for (int i = ty; i < 32; i += 8) {
    int64_t r, c;
    if (row_fast) { r = r0 + tx; c = c0 + i; } else { r = r0 + i; c = c0 + tx; }
    float v = 0.f;
    if (r < rows && c < cols) v = src[r * s_row + c * s_col];
    if (row_fast) tile[tx][i] = v; else tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    if (r < rows && c < cols) store1<T, SPLIT>(dst, r, c, cols, ld, tile[i][tx]);
  }
}

template <typename T, int SPLIT = 0>
int pack(const float *src, int64_t s_row, int64_t s_col, T *dst, int64_t rows, int64_t cols,
         cudaStream_t s) {
  const int64_t ld = SPLIT ? 3 * cols : cols;
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (s_col == 1 && aligned && cols % 8 == 0 && s_row % 4 == 0) {
    const int64_t work = rows * (cols / 8);
    int64_t blocks = (work + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    pack_rows_kernel<T, SPLIT><<<(unsigned)blocks, 256, 0, s>>>(src, s_row, dst, rows, cols, ld);
  } else if (s_row == 1 && aligned && s_col % 4 == 0) {
    dim3 grid((unsigned)((rows + 63) / 64), (unsigned)((cols + 63) / 64));
    pack_transpose_kernel<T, SPLIT><<<grid, 256, 0, s>>>(src, s_col, dst, rows, cols, ld);
  } else {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    pack_kernel<T, SPLIT><<<grid, dim3(32, 8), 0, s>>>(src, s_row, s_col, dst, rows, cols, ld);
  }
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace

extern "C" int b200_pack_operand(int32_t kind, const float *src, int64_t s_row, int64_t s_col,
                                 void *dst, int64_t rows, int64_t cols, void *stream) {
  if (rows <= 0 || cols <= 0) return B200_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (kind == 0)
    return pack<__nv_bfloat16>(src, s_row, s_col, static_cast<__nv_bfloat16 *>(dst), rows, cols, s);
  if (kind == 2)
    return pack<float, 1>(src, s_row, s_col, static_cast<float *>(dst), rows, cols, s);
  if (kind == 3)
    return pack<float, 2>(src, s_row, s_col, static_cast<float *>(dst), rows, cols, s);
  if (kind != 1) return B200_EINVAL;
  return pack<float>(src, s_row, s_col, static_cast<float *>(dst), rows, cols, s);
}

namespace {

int gemm_tc(int32_t kind, const void *A, const void *Bt, float *C, int64_t sCm, int64_t sCn,
            int64_t M, int64_t N, int64_t K, int32_t init, float init_value, const float *bias,
            int64_t bias_stride, int32_t max_ctas, int32_t variant, __nv_bfloat16 *c16,
            int64_t ld16, void *stream, const void *Bkn = nullptr) {
  if (M <= 0 || N <= 0) return B200_OK;
  if (K <= 0 || (kind != 0 && kind != 1)) return B200_EINVAL;
  const int elem = kind == 0 ? 2 : 4;
  if ((K * elem) % 16 != 0) return B200_EUNSUPPORTED;  // TMA row stride alignment
  Epi ep{C, sCm, sCn, bias, bias_stride, init, init_value, c16, ld16};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int sms = num_sms();
  if (variant == 0) {
    // pairs pay off once there are enough 256x256 tiles to fill the pairs
    const int64_t pair_tiles = ((M + 255) / 256) * ((N + 255) / 256);
    variant = pair_tiles >= sms / 2 ? 2 : 1;
  }
  if (Bkn) return launch_gemm_tc2(kind, A, nullptr, ep, M, N, K, max_ctas / 2, s, Bkn, false);
  if (variant == 2) return launch_gemm_tc2(kind, A, Bt, ep, M, N, K, max_ctas / 2, s, nullptr,
                                           false);
  // variant 3: 128 x 256 CTA tiles as cta_group::1 MMAs in 2-CTA clusters
  // sharing the B tile by multicast (gemm_tc2.cu SOLO); variant 1: the
  // stand-alone single-CTA kernel below
  if (variant == 3 && !getenv("B200_TC_SOLO_OFF"))
    return launch_gemm_tc2(kind, A, Bt, ep, M, N, K, max_ctas / 2, s, nullptr, true);
  CUtensorMap ma, mb;
  if (!make_map(&ma, kind, A, M, K, BM) || !make_map(&mb, kind, Bt, N, K, BN))
    return B200_ELAUNCH;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int ctas = sms;
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  if (tiles < ctas) ctas = (int)tiles;
  if (kind == 0) {
    cudaFuncSetAttribute(gemm_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SMEM_BYTES);
    gemm_tc_kernel<0><<<ctas, kThreads, SMEM_BYTES, s>>>(ma, mb, ep, M, N, K);
  } else {
    cudaFuncSetAttribute(gemm_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SMEM_BYTES);
    gemm_tc_kernel<1><<<ctas, kThreads, SMEM_BYTES, s>>>(ma, mb, ep, M, N, K);
  }
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace

extern "C" int b200_gemm_tc(int32_t kind, const void *A, const void *Bt, float *C, int64_t sCm,
                            int64_t sCn, int64_t M, int64_t N, int64_t K, int32_t init,
                            float init_value, const float *bias, int64_t bias_stride,
                            int32_t max_ctas, int32_t variant, void *stream) {
  return gemm_tc(kind, A, Bt, C, sCm, sCn, M, N, K, init, init_value, bias, bias_stride,
                 max_ctas, variant, nullptr, 0, stream);
}

extern "C" int b200_gemm_tc_shadow(int32_t kind, const void *A, const void *Bt, float *C,
                                   int64_t sCm, int64_t sCn, int64_t M, int64_t N, int64_t K,
                                   int32_t init, float init_value, const float *bias,
                                   int64_t bias_stride, void *c16, int64_t ld16,
                                   void *stream) {
  if (!c16 || ld16 < N) return B200_EINVAL;
  return gemm_tc(kind, A, Bt, C, sCm, sCn, M, N, K, init, init_value, bias, bias_stride, 0, 0,
                 static_cast<__nv_bfloat16 *>(c16), ld16, stream);
}

// C (+)= A . B with B given as a K x N row-major bf16 tensor (the matmul
// nest's own B layout, converted but not transposed), read MN-major by the
// CTA-pair kernel; c16 / ld16 as in b200_gemm_tc_shadow (c16 may be null).
extern "C" int b200_gemm_tc_kn(int32_t kind, const void *A, const void *B, float *C,
                               int64_t sCm, int64_t sCn, int64_t M, int64_t N, int64_t K,
                               int32_t init, float init_value, const float *bias,
                               int64_t bias_stride, void *c16, int64_t ld16, void *stream) {
  if (kind != 0) return B200_EUNSUPPORTED;   // MN-major is bf16-only (see gemm_tc2.cu)
  if (c16 && ld16 < N) return B200_EINVAL;
  return gemm_tc(kind, A, nullptr, C, sCm, sCn, M, N, K, init, init_value, bias, bias_stride, 0,
                 2, static_cast<__nv_bfloat16 *>(c16), ld16, stream, B);
}
