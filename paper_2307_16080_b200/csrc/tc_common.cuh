// Shared sm_100a building blocks for the tensor-core kernels: mbarriers, TMA,
// tcgen05 fences / commits / TMEM loads, UMMA descriptors, tensor maps and
// the fp32 epilogue.  Inline PTX only (no CUTLASS); bit layouts follow the
// PTX ISA tcgen05 descriptor tables (SM100 smem / instruction descriptors).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace b200tc {

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
// arrive on an mbarrier given by a shared::cluster address (peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
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
// cluster-scope acquire wait (for barriers arrived on by the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
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
// 2-SM variant: the completed bytes are counted on `bar` (a shared::cluster
// address, normally the leader CTA's barrier) while data lands in local smem.
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap *map, uint32_t bar,
                                                 uint32_t dst, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(const CUtensorMap *map, uint32_t bar,
                                                 uint32_t dst, int32_t c0, int32_t c1,
                                                 int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA store (bulk group) from local smem to global, OOB elements clipped.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// make generic-proxy shared-memory writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 2-D fp32 tensor map over C (row-major, unit column stride) with boxes of
// 32 columns (128 B, swizzled) x box_rows rows, for the staged epilogue.
inline bool make_map_c(CUtensorMap *map, const float *C, int64_t rows, int64_t cols,
                       int64_t row_stride, uint32_t box_rows);

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major, 128B-swizzled operand tile: rows of 128B, 8-row atoms 1024B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                  // LBO (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;                  // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// MN-major, 128B-swizzled B operand (rows = K, 64 contiguous N per 128-byte
// row): the canonical ((8 x 16 B, n), (8 rows, k)) layout with the 64-wide N
// chunks `lbo` bytes apart and 8-row K groups 1024 bytes apart.
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;   // LBO: next 64-wide N chunk
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: next 8 K rows
  d |= (uint64_t)1 << 46;                  // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: fp32 accumulate, bf16 (kind 0) / tf32 (kind 1)
// operands, both K-major, shape M x N (bit 16 = B MN-major, set by callers).
__host__ __device__ constexpr uint32_t make_idesc(int kind, int M, int N) {
  return (1u << 4) | ((kind == 0 ? 1u : 2u) << 7) | ((kind == 0 ? 1u : 2u) << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int KIND, int CTAS>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  if (KIND == 0 && CTAS == 1)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if (KIND == 1 && CTAS == 1)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if (KIND == 0)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
// 2-SM commit arriving on the same barrier offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(mask)
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
  // optional bf16 shadow of the final C (row-major, leading dimension ld16):
  // the next contraction's packed A operand, written by the same epilogue
  __nv_bfloat16 *c16 = nullptr;
  int64_t ld16 = 0;
};

// 32 consecutive final values of row m, columns [nb, nb + 32), into the bf16
// shadow (4 x 16-byte stores when the whole run is in range).
__device__ __forceinline__ void shadow_store32(const Epi &ep, int64_t m, int64_t nb, int64_t M,
                                               int64_t N, const float (&v)[32]) {
  if (m >= M) return;
  __nv_bfloat16 *dst = ep.c16 + m * ep.ld16 + nb;
  if (nb + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(v[8 * q + 2 * j], v[8 * q + 2 * j + 1]);
      reinterpret_cast<uint4 *>(dst)[q] = *reinterpret_cast<uint4 *>(b);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)   // fully unrolled: v stays in registers
      if (nb + j < N) dst[j] = __float2bfloat16_rn(v[j]);
  }
}

// One thread owns output row m; writes columns [nb, nb+32) from r[].
__device__ __forceinline__ void epilogue_row32(const Epi &ep, int64_t m, int64_t nb, int64_t M,
                                               int64_t N, const uint32_t (&r)[32]) {
  if (m >= M) return;
  float *crow = ep.C + m * ep.sCm;
  const bool vec = ep.sCn == 1 && nb + 32 <= N &&
                   ((reinterpret_cast<uintptr_t>(crow + nb) & 15) == 0);
  if (ep.c16) {
    // with the bf16 shadow: final values gathered, then both outputs written
    // (kept apart from the plain path below, whose code it would bloat)
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t n = nb + j;
      float o = 0.f;
      if (n < N) {
        o = ep.init ? ep.init_value : crow[n * ep.sCn];
        o += __uint_as_float(r[j]);
        if (ep.bias) o += ep.bias[n * ep.bias_stride];
        crow[n * ep.sCn] = o;
      }
      v[j] = o;
    }
    shadow_store32(ep, m, nb, M, N, v);
    return;
  }
  if (vec) {
    float4 *p = reinterpret_cast<float4 *>(crow + nb);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 o = ep.init ? make_float4(ep.init_value, ep.init_value, ep.init_value, ep.init_value)
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

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiled get_encode() {
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

// 2-D K-major tensor map: rows x k elements, box = (128 bytes of K) x box_rows.
inline bool make_map(CUtensorMap *map, int kind, const void *ptr, int64_t rows, int64_t k,
                     uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  const int elem = kind == 0 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(k * elem)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline bool make_map_c(CUtensorMap *map, const float *C, int64_t rows, int64_t cols,
                       int64_t row_stride, uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(row_stride * 4)};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(C), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D bf16 tensor map over the shadow (row-major, leading dimension ld16) with
// boxes of 32 columns (64 B, 64B swizzle) x box_rows rows: the staged shadow
// chunk of the epilogue, written back by one TMA store.
inline bool make_map_s16(CUtensorMap *map, void *c16, int64_t rows, int64_t cols, int64_t ld16,
                         uint32_t box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld16 * 2)};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c16, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Epilogue over one 32-column chunk staged in shared memory by TMA with the
// 128B swizzle: row r's 16-byte unit j lives at unit j ^ (r & 7).  The
// thread owning row r adds its accumulator (and bias) in place.
// m / M: the global row of r and the row count (for the bf16 shadow only).
// sbias (optional): the chunk's 32 bias values already staged in shared
// memory (zero past N).  s16 (optional): the chunk's bf16 shadow buffer in
// shared memory (32 columns = 64 B per row, 64B swizzle: row r's 16-byte
// unit q lives at unit q ^ ((r >> 1) & 3)), stored by TMA afterwards;
// without it the shadow goes straight to global memory.
__device__ __forceinline__ void epilogue_chunk_smem(unsigned char *chunk, int r, int64_t nb,
                                                    int64_t N, const Epi &ep,
                                                    const uint32_t (&acc)[32], int64_t m = 0,
                                                    int64_t M = 0,
                                                    const float *sbias = nullptr,
                                                    unsigned char *s16 = nullptr) {
  float4 *row = reinterpret_cast<float4 *>(chunk + r * 128);
  // the chunk's 32 bias values, loaded up front (the same addresses for the
  // whole warp: one broadcast transaction each): 8 x 16-byte loads when the
  // bias is unit-stride and aligned, element loads otherwise
  float4 bv[8];
  if (sbias) {
#pragma unroll
    for (int j = 0; j < 8; ++j) bv[j] = reinterpret_cast<const float4 *>(sbias)[j];
  } else if (ep.bias) {
    const float *b = ep.bias + nb * ep.bias_stride;
    if (ep.bias_stride == 1 && nb + 32 <= N && (reinterpret_cast<uintptr_t>(b) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) bv[j] = __ldg(reinterpret_cast<const float4 *>(b) + j);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t n = nb + 4 * j;
        bv[j].x = n + 0 < N ? __ldg(b + (4 * j + 0) * ep.bias_stride) : 0.f;
        bv[j].y = n + 1 < N ? __ldg(b + (4 * j + 1) * ep.bias_stride) : 0.f;
        bv[j].z = n + 2 < N ? __ldg(b + (4 * j + 2) * ep.bias_stride) : 0.f;
        bv[j].w = n + 3 < N ? __ldg(b + (4 * j + 3) * ep.bias_stride) : 0.f;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float4 *p = row + (j ^ (r & 7));
    float4 o = ep.init ? make_float4(ep.init_value, ep.init_value, ep.init_value, ep.init_value)
                       : *p;
    o.x += __uint_as_float(acc[4 * j + 0]);
    o.y += __uint_as_float(acc[4 * j + 1]);
    o.z += __uint_as_float(acc[4 * j + 2]);
    o.w += __uint_as_float(acc[4 * j + 3]);
    if (ep.bias) {
      o.x += bv[j].x;
      o.y += bv[j].y;
      o.z += bv[j].z;
      o.w += bv[j].w;
    }
    *p = o;
    bv[j] = o;   // reused as the final values for the shadow
  }
  if (s16) {
    uint4 *srow = reinterpret_cast<uint4 *>(s16 + r * 64);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 b[4];
      b[0] = __floats2bfloat162_rn(bv[2 * q].x, bv[2 * q].y);
      b[1] = __floats2bfloat162_rn(bv[2 * q].z, bv[2 * q].w);
      b[2] = __floats2bfloat162_rn(bv[2 * q + 1].x, bv[2 * q + 1].y);
      b[3] = __floats2bfloat162_rn(bv[2 * q + 1].z, bv[2 * q + 1].w);
      srow[q ^ ((r >> 1) & 3)] = *reinterpret_cast<uint4 *>(b);
    }
  } else if (ep.c16) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[4 * j] = bv[j].x, v[4 * j + 1] = bv[j].y, v[4 * j + 2] = bv[j].z, v[4 * j + 3] = bv[j].w;
    shadow_store32(ep, m, nb, M, N, v);
  }
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// 2-CTA launcher (gemm_tc2.cu).  Bkn (bf16 only): B as a K x N row-major
// tensor read MN-major, instead of the K-major N x K pack Bt.  solo: 128 x
// 256 CTA tiles with cta_group::1 MMAs, the cluster's B tile multicast.
int launch_gemm_tc2(int kind, const void *A, const void *Bt, const Epi &ep, int64_t M, int64_t N,
                    int64_t K, int max_clusters, cudaStream_t s, const void *Bkn = nullptr,
                    bool solo = false);

}  // namespace b200tc
