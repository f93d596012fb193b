// Tensor-core contraction for sm_100a: TMA -> SMEM -> tcgen05.mma -> TMEM.
//
// C[m,n] = (init ? init_value : C[m,n]) + sum_k A[m,k] * B[k,n]  (+ bias[n])
//
// This replaces run_tape on a recognised matmul / Linear contraction nest
// (reference tests/kernels.py:24-38) when the engine runs
// with precision "bf16" or "tf32".  Products of bf16/tf32 inputs are exact in
// fp32; the tensor core accumulates in fp32 in K order, so the only deviation
// from the reference's sequential f32 chain is accumulation rounding (bound
// stated in DESIGN.md and tests/test_gpu_tc.py).
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0        TMA producer: A tile 128 x 128B and B^T tile 256 x 128B per
//                 stage (both K-major, 128B swizzle), 4-stage mbarrier ring
//   warp 1        MMA issuer (one elected lane): 4 x tcgen05.mma per stage
//                 (UMMA 128x256, K=16 bf16 / K=8 tf32), commits free the
//                 stage and, at the last k-block, publish the accumulator
//   warp 2        TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4..7    epilogue: tcgen05.ld 32x32b.x32 -> +C / init, +bias ->
//                 128-bit global stores; releases the TMEM buffer so the MMA
//                 of tile i+1 overlaps the epilogue of tile i
// Operands must be packed K-major by b200_pack_operand (convert / transpose).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK_BYTES = 128;          // one 128B swizzle row of K per stage
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BK_BYTES; // 16 KB
constexpr int B_STAGE = BN * BK_BYTES; // 32 KB
constexpr int TMEM_COLS = 512;
constexpr int kThreads = 256;
constexpr size_t SMEM_BYTES = 1024 + STAGES * (A_STAGE + B_STAGE) + 256;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint32_t bar, uint32_t dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major, 128B-swizzled operand tile: rows of 128B, 8-row atoms 1024B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                          // LBO (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;                          // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}

template <int KIND>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  if (KIND == 0) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Epi {
  float *C;
  int64_t sCm, sCn;
  const float *bias;
  int64_t bias_stride;
  int init;
  float init_value;
};

// Instruction descriptor: fp32 accumulate, A/B format, K-major both, M=128, N=256.
template <int KIND>
__device__ __forceinline__ uint32_t make_idesc() {
  uint32_t fmt = KIND == 0 ? 1u : 2u;  // BF16 : TF32
  uint32_t d = 0;
  d |= 1u << 4;            // c_format F32
  d |= fmt << 7;           // a_format
  d |= fmt << 10;          // b_format
  d |= (uint32_t)(BN >> 3) << 17;
  d |= (uint32_t)(BM >> 4) << 24;
  return d;
}

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
  // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2], then tmem addr
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  constexpr int ELEM = KIND == 0 ? 2 : 4;
  constexpr int BK = BK_BYTES / ELEM;          // elements of K per stage
  constexpr int UK = 32 / ELEM;                // K per tcgen05.mma (32 bytes)

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
      const uint32_t idesc = make_idesc<KIND>();
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
          for (int k = 0; k < BK / UK; ++k) {
            umma<KIND>(tmem_d, smem_desc(a_addr + 32 * k), smem_desc(b_addr + 32 * k), idesc,
                       (kb | k) != 0);
          }
          umma_commit(empty(s));
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;                 // TMEM lane quarter of this warp
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
        const int64_t nb = n0 + c * 32;
        if (m < M) {
          float *crow = ep.C + m * ep.sCm;
          const bool vec = ep.sCn == 1 && nb + 32 <= N &&
                           ((reinterpret_cast<uintptr_t>(crow + nb) & 15) == 0);
          if (vec) {
            float4 *p = reinterpret_cast<float4 *>(crow + nb);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 o = ep.init ? make_float4(ep.init_value, ep.init_value, ep.init_value,
                                               ep.init_value)
                                 : p[j];
              o.x += __uint_as_float(r[4 * j + 0]);
              o.y += __uint_as_float(r[4 * j + 1]);
              o.z += __uint_as_float(r[4 * j + 2]);
              o.w += __uint_as_float(r[4 * j + 3]);
              if (ep.bias) {
                const float *b = ep.bias + (nb + 4 * j) * ep.bias_stride;
                o.x += b[0];
                o.y += b[ep.bias_stride];
                o.z += b[2 * ep.bias_stride];
                o.w += b[3 * ep.bias_stride];
              }
              p[j] = o;
            }
          } else {
            for (int j = 0; j < 32; ++j) {
              const int64_t n = nb + j;
              if (n >= N) break;
              float *dst = crow + n * ep.sCn;
              float o = ep.init ? ep.init_value : *dst;
              o += __uint_as_float(r[j]);
              if (ep.bias) o += ep.bias[n * ep.bias_stride];
              *dst = o;
            }
          }
        }
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

// 32x32 tiles through shared memory so both the read (along whichever source
// dimension is contiguous) and the write (along c) are coalesced.
template <typename T>
__global__ void pack_kernel(const float *__restrict__ src, int64_t s_row, int64_t s_col,
                            T *__restrict__ dst, int64_t rows, int64_t cols) {
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
    if (r < rows && c < cols) dst[r * cols + c] = cvt<T>(tile[i][tx]);
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled get_encode() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

bool make_map(CUtensorMap *map, int kind, const void *ptr, int64_t rows, int64_t k,
              uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  const int elem = kind == 0 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(k * elem)};
  cuuint32_t box[2] = {(cuuint32_t)(BK_BYTES / elem), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

extern "C" int b200_pack_operand(int32_t kind, const float *src, int64_t s_row, int64_t s_col,
                                 void *dst, int64_t rows, int64_t cols, void *stream) {
  if (rows <= 0 || cols <= 0) return B200_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  dim3 block(32, 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (kind == 0)
    pack_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(src, s_row, s_col,
                                                      static_cast<__nv_bfloat16 *>(dst), rows, cols);
  else
    pack_kernel<float><<<grid, block, 0, s>>>(src, s_row, s_col, static_cast<float *>(dst), rows,
                                              cols);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

extern "C" int b200_gemm_tc(int32_t kind, const void *A, const void *Bt, float *C, int64_t sCm,
                            int64_t sCn, int64_t M, int64_t N, int64_t K, int32_t init,
                            float init_value, const float *bias, int64_t bias_stride,
                            int32_t max_ctas, void *stream) {
  if (M <= 0 || N <= 0) return B200_OK;
  if (K <= 0 || (kind != 0 && kind != 1)) return B200_EINVAL;
  const int elem = kind == 0 ? 2 : 4;
  if ((K * elem) % 16 != 0) return B200_EUNSUPPORTED;  // TMA row stride alignment
  CUtensorMap ma, mb;
  if (!make_map(&ma, kind, A, M, K, BM) || !make_map(&mb, kind, Bt, N, K, BN))
    return B200_ELAUNCH;
  Epi ep{C, sCm, sCn, bias, bias_stride, init, init_value};
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int ctas = num_sms();
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  if (tiles < ctas) ctas = (int)tiles;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
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
