// 2-SM tensor-core contraction: a CTA pair (cluster of 2) computes a 256x256
// output tile with tcgen05.mma.cta_group::2 (UMMA M=256, N=256).
//
// Each CTA stages its own half of the operands — 128 rows of A and 128 rows of
// B^T per 128-byte K slice — so per SM the TMA traffic per MMA is half of the
// single-CTA 128x256 kernel's.  B comes either K-major (the transposed N x K
// pack) or, for bf16, MN-major straight from its K x N layout (BMN: one 3-D
// TMA box of two 64-wide N chunks x 64 K rows per stage, descriptor LBO = the
// 8 KB chunk stride, SBO = 1 KB per 8 K rows, instruction bit 16 set).  Only the leader CTA (cluster rank 0) issues
// MMAs; both CTAs' TMA loads complete on the leader's full-barrier, MMA
// commits are multicast to both CTAs' empty / tmem-full barriers, and both
// CTAs' epilogues release the accumulator buffer on the leader's tmem-empty
// barrier.  Each CTA's TMEM holds its 128 rows x 256 columns of the fp32
// accumulator (2 buffers = 512 columns, epilogue of tile i overlaps the MMAs
// of tile i+1).
//
// Work schedule: persistent clusters walk full tiles round-robin; the tiles of
// the last, partial wave are split S = floor(clusters / remaining) ways along
// N into 256 x (256/S) sub-tiles (UMMA N = 256/S, same efficiency per flop),
// so the tail wave is balanced while every output keeps one full-K chain
// (deterministic, no partial sums, no workspace).
//
// Epilogue (C = C + acc [+ bias]): C is staged through shared memory in
// 128-row x 32-column chunks by TMA (128B swizzle, 4 buffers): the loads of
// upcoming chunks — including the next tile's — are issued ahead, each thread
// adds its TMEM row in place, and a TMA bulk store writes the chunk back.
// The tile's bias is staged in shared memory once per tile (its loads are
// issued before the accumulator wait); a bf16 shadow of C, when requested,
// is staged per chunk in shared memory (64B swizzle) and TMA-stored with the
// chunk.  (Strided C falls back to per-row 128-bit stores.)
//
// Replaces run_tape on a recognised matmul / Linear contraction nest
// (reference tests/kernels.py:24-38) at bf16/tf32 precision.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/b200k.h"
#include "tc_common.cuh"

namespace b200tc {

namespace {

constexpr int PA = 128 * 128;   // A half: 128 rows x 128 B
constexpr int PB = 128 * 128;   // B half: 128 rows x 128 B
constexpr int CBUF = 128 * 128; // C chunk: 128 rows x 32 fp32
constexpr int NCBUF = 4;
#ifndef B200_SOLO_STAGES
#define B200_SOLO_STAGES 4
#endif
constexpr int SOLO_STAGES = B200_SOLO_STAGES;
constexpr int SBUF = 128 * 64;  // bf16 shadow chunk: 128 rows x 32 bf16
constexpr int BIASB = 256 * 4;  // the tile's bias values
constexpr int PTHREADS = 256;
// Shared memory layout: operand stages | C chunks | [shadow chunks] | bias |
// barriers.  The shadow variant trades one operand stage for two staged
// shadow chunks (the shadow's TMA stores are coalesced; per-thread row
// stores of 64 B were not).
// SOLO (the 128 x 256 CTA tile of (4, 16)-style tilings): each CTA of the
// cluster runs its own cta_group::1 MMAs on its 128 rows and the cluster's
// whole 256-column B tile, whose two halves the two CTAs load once and
// multicast to both — a stage holds all 256 rows of B^T.
template <bool SH, bool SOLO = false>
struct Lay {
  static constexpr int PBS = SOLO ? 2 * PB : PB;   // B bytes per stage
  // SOLO: 48 KB stages; four of them leave room for two C chunks only (the
  // epilogue of a K = 4096 tile is a small share of its 24 us)
  static constexpr int STAGES = SOLO ? (SH ? 3 : SOLO_STAGES) : (SH ? 4 : 5);
  static constexpr int NCB = SOLO && STAGES == 4 ? 2 : NCBUF;
  static constexpr int NSBUF = SH ? 2 : 0;
  static constexpr size_t C_OFF = (size_t)STAGES * (PA + PBS);
  static constexpr size_t S_OFF = C_OFF + NCB * CBUF;
  static constexpr size_t BIAS_OFF = S_OFF + NSBUF * SBUF;
  static constexpr size_t BAR_OFF = BIAS_OFF + BIASB;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 256;
};
static_assert(Lay<false>::SMEM <= 232448 && Lay<true>::SMEM <= 232448, "smem");
static_assert(Lay<false, true>::SMEM <= 232448 && Lay<true, true>::SMEM <= 232448, "smem");

// TMA load multicast to every CTA of `mask` (same shared offsets; each
// destination's barrier at `bar` receives its bytes)
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap *map, uint32_t bar, uint32_t dst,
                                               int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// single-CTA MMA commit arriving on the same barrier in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

struct Sched {
  int64_t tiles, nt, kb_total, ncl;
  int64_t group_m;   // M-blocks walked together by the grouped raster
  int64_t waves;   // full waves of whole tiles
  int64_t rem;     // tiles in the partial wave
  int64_t split;   // N sub-tiles per tail tile (1, 2, 4 or 8)
};

struct Item {
  int64_t m0, n0;  // pair tile origin
  int ncols;       // 256 or 256 / split
};

__device__ __forceinline__ bool get_item(const Sched &s, int64_t cid, int64_t i, Item &it) {
  int64_t t, sub = 0;
  if (i < s.waves) {
    t = cid + i * s.ncl;
    it.ncols = 256;
  } else if (i == s.waves && cid < s.rem * s.split) {
    t = s.waves * s.ncl + cid / s.split;
    sub = cid % s.split;
    it.ncols = (int)(256 / s.split);
  } else {
    return false;
  }
  // grouped raster: GROUP_M consecutive M-blocks walk N together, so one wave
  // of tiles touches ~GROUP_M A panels and ~waves/GROUP_M B panels (L2 reuse)
  const int64_t GROUP_M = s.group_m;
  const int64_t mt = s.tiles / s.nt;
  const int64_t group = t / (GROUP_M * s.nt);
  const int64_t first_m = group * GROUP_M;
  const int64_t gm = (mt - first_m) < GROUP_M ? (mt - first_m) : GROUP_M;
  const int64_t tin = t - group * GROUP_M * s.nt;
  it.m0 = (first_m + tin % gm) * 256;
  it.n0 = (tin / gm) * 256 + sub * it.ncols;
  return true;
}

template <int KIND, bool SH, bool BMN, bool SOLO = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tma_a,
                    const __grid_constant__ CUtensorMap tma_b,
                    const __grid_constant__ CUtensorMap tma_bs,
                    const __grid_constant__ CUtensorMap tma_c,
                    const __grid_constant__ CUtensorMap tma_s, int use_tma_c, Epi ep, int64_t M,
                    int64_t N, Sched sch) {
  using L = Lay<SH, SOLO>;
  constexpr int PSTAGES = L::STAGES;
  constexpr int NCB = L::NCB;
  static_assert(!(SOLO && BMN), "SOLO reads B K-major");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t sA = base;
  const uint32_t sB = base + PSTAGES * PA;
  const uint32_t sC = base + (uint32_t)L::C_OFF;
  unsigned char *gC = gbase + L::C_OFF;
  const uint32_t sS = base + (uint32_t)L::S_OFF;
  unsigned char *gS = gbase + L::S_OFF;
  float *sBias = reinterpret_cast<float *>(gbase + L::BIAS_OFF);
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + L::BAR_OFF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * PSTAGES + 4 + NCB);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (PSTAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * PSTAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * PSTAGES + 2 + a); };
  auto cbar = [&](int b) { return bar0 + 8u * (2 * PSTAGES + 4 + b); };

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  constexpr int ELEM = KIND == 0 ? 2 : 4;
  constexpr int BK = 128 / ELEM;
  constexpr int UK = 32 / ELEM;
  constexpr int CH = 128 / ELEM;        // MN-major B: N elements per 128-byte row
  constexpr uint32_t CHB = BK * 128;    // bytes of one N chunk (BK rows)
  const int64_t kb_total = sch.kb_total;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(full(s), 1);
      // SOLO: a stage's B halves come from both CTAs, so both MMAs release it
      mbar_init(empty(s), SOLO ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), SOLO ? 128 : 256);
    }
    for (int b = 0; b < NCB; ++b) mbar_init(cbar(b), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 2) {
    if (SOLO) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t cid = blockIdx.x / 2;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      Item it;
      for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
        // each CTA stages half of the item's columns of B^T
        const int brows = it.ncols / 2;
        const CUtensorMap *mb = brows == 128 ? &tma_b : &tma_bs;
        // MN-major B: chunks of CH (N) x BK (K) (128-byte rows), at least
        // one (a narrow tail item reads a whole chunk and uses its first
        // brows columns)
        const int nbox = brows >= CH ? brows / CH : 1;
        const uint32_t bytes = BMN ? 2u * (PA + nbox * CHB) : 2u * (PA + brows * 128);
        const int32_t m0 = (int32_t)(it.m0 + rank * 128);
        const int32_t n0 = (int32_t)(it.n0 + rank * brows);
        if (SOLO) {
          // own A rows; this CTA's half of the item's B^T rows to both CTAs
          const int32_t nh = (int32_t)(it.n0 + rank * brows);
          for (int64_t kb = 0; kb < kb_total; ++kb) {
            mbar_wait(empty(s), ph ^ 1);
            mbar_expect_tx(full(s), (uint32_t)(PA + 2 * brows * 128));
            tma_load_2d(&tma_a, full(s), sA + s * PA, (int32_t)(kb * BK), m0);
            tma_load_2d_mc(mb, full(s), sB + s * L::PBS + rank * (uint32_t)(brows * 128),
                           (int32_t)(kb * BK), nh, (uint16_t)0x3);
            if (++s == PSTAGES) { s = 0; ph ^= 1; }
          }
          continue;
        }
        for (int64_t kb = 0; kb < kb_total; ++kb) {
          mbar_wait(empty(s), ph ^ 1);
          if (leader) mbar_expect_tx(full(s), bytes);
          const uint32_t lf = map_to_rank(full(s), 0);
          tma_load_2d_pair(&tma_a, lf, sA + s * PA, (int32_t)(kb * BK), m0);
          if (BMN) {
            // one box: nbox N chunks x BK K rows (chunks CHB bytes apart)
            tma_load_3d_pair(brows == 128 ? &tma_b : &tma_bs, lf, sB + s * PB, n0 % CH,
                             (int32_t)(kb * BK), n0 / CH);
          } else {
            tma_load_2d_pair(mb, lf, sB + s * PB, (int32_t)(kb * BK), n0);
          }
          if (++s == PSTAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (SOLO && lane == 0) {
      // every CTA: 128 x ncols from its own A rows and the shared B tile;
      // a stage is released to both producers (their multicasts wrote it)
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      Item it;
      for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
        const uint32_t idesc = make_idesc(KIND, 128, it.ncols);
        mbar_wait(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * 256);
        for (int64_t kb = 0; kb < kb_total; ++kb) {
          mbar_wait(full(s), ph);
          tc_fence_after();
          const uint32_t a_addr = sA + s * PA, b_addr = sB + s * L::PBS;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma<KIND, 1>(tmem_d, smem_desc(a_addr + 32 * k), smem_desc(b_addr + 32 * k), idesc,
                          (kb | k) != 0);
          umma_commit_mc(empty(s), 0x3);
          if (++s == PSTAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    } else if (!SOLO && leader && lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      Item it;
      for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
        const uint32_t idesc = make_idesc(KIND, 256, it.ncols) | (BMN ? 1u << 16 : 0u);
        mbar_wait_cluster(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * 256);
        for (int64_t kb = 0; kb < kb_total; ++kb) {
          mbar_wait(full(s), ph);
          tc_fence_after();
          const uint32_t a_addr = sA + s * PA, b_addr = sB + s * PB;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma<KIND, 2>(tmem_d, smem_desc(a_addr + 32 * k),
                          BMN ? smem_desc_mn(b_addr + 128 * UK * k, CHB)
                              : smem_desc(b_addr + 32 * k),
                          idesc, (kb | k) != 0);
          umma_commit_pair(empty(s), 0x3);
          if (++s == PSTAGES) { s = 0; ph ^= 1; }
        }
        umma_commit_pair(tfull(acc), 0x3);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int et = threadIdx.x - 128;  // TMEM lane / row within the CTA's 128 rows
    const int q = warp - 4;
    const bool lead_t = et == 0;
    const bool load_c = use_tma_c && !ep.init;
    // chunk g of this CTA: work item g / 8, columns (g % 8) * 32 of the item
    auto chunk_coords = [&](int64_t g, int32_t &col, int32_t &row) -> bool {
      Item ci;
      if (!get_item(sch, cid, g / 8, ci) || (g % 8) * 32 >= ci.ncols) return false;
      row = (int32_t)(ci.m0 + rank * 128);
      col = (int32_t)(ci.n0 + (g % 8) * 32);
      return true;
    };
    auto issue_load = [&](int64_t g) {
      int32_t col, row;
      if (!chunk_coords(g, col, row)) return;
      const int b = (int)(g % NCB);
      mbar_expect_tx(cbar(b), CBUF);
      tma_load_2d(&tma_c, cbar(b), sC + b * CBUF, col, row);
    };
    if (load_c && lead_t)
      for (int64_t g = 0; g < NCB - 1; ++g) issue_load(g);
    int acc = 0;
    uint32_t aph = 0;
    int64_t g = 0;
    const uint32_t lead_tempty0 = map_to_rank(tempty(0), 0);
    const uint32_t lead_tempty1 = map_to_rank(tempty(1), 0);
    Item it;
    for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
      const int64_t m_base = it.m0 + rank * 128;
      // the tile's bias: loads issued before the accumulator wait (their
      // latency hides behind it), staged in shared memory once per tile
      float b0 = 0.f, b1 = 0.f;
      if (ep.bias) {
        const int64_t n0 = it.n0 + et, n1 = n0 + 128;
        if (n0 < N && et < it.ncols) b0 = __ldg(ep.bias + n0 * ep.bias_stride);
        if (n1 < N && et + 128 < it.ncols) b1 = __ldg(ep.bias + n1 * ep.bias_stride);
      }
      mbar_wait_cluster(tfull(acc), aph);
      tc_fence_after();
      if (ep.bias) {
        // every reader of the previous tile's values passed that tile's
        // last chunk barrier
        sBias[et] = b0;
        sBias[et + 128] = b1;
        named_bar_sync(1, 128);
      }
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256);
      const int nchunks = it.ncols / 32;
#pragma unroll 1
      for (int c = 0; c < nchunks; ++c, ++g) {
        uint32_t r[32];
        tmem_ld32(trow + (uint32_t)(c * 32), r);
        const int64_t nb = it.n0 + c * 32;
        if (use_tma_c) {
          const int b = (int)(g % NCB);
          if (load_c) {
            mbar_wait(cbar(b), (uint32_t)((g / NCB) & 1));
          } else {
            // no C load: make sure the store of chunk g-4 (shadow: g-2) has
            // left this buffer
            if (lead_t) bulk_wait_read<SH ? 1 : NCB - 1>();
            named_bar_sync(1, 128);
          }
          const int sb = (int)(g & 1);
          epilogue_chunk_smem(gC + b * CBUF, et, nb, N, ep, r, m_base + et, M,
                              ep.bias ? sBias + c * 32 : nullptr,
                              SH ? gS + sb * SBUF : nullptr);
          fence_proxy_async();
          named_bar_sync(1, 128);
          if (lead_t) {
            tma_store_2d(&tma_c, sC + b * CBUF, (int32_t)nb, (int32_t)m_base);
            if (SH) tma_store_2d(&tma_s, sS + sb * SBUF, (int32_t)nb, (int32_t)m_base);
            bulk_commit();
            if (load_c) {
              bulk_wait_read<1>();  // store of chunk g-1 has read buffer (g+3) % 4
              issue_load(g + NCB - 1);
            }
          }
        } else {
          epilogue_row32(ep, m_base + et, nb, M, N, r);
        }
      }
      g += 8 - nchunks;  // keep one 8-chunk slot per item (only the last item is narrower)
      tc_fence_before();
      if (SOLO)
        mbar_arrive(tempty(acc));   // this CTA's own accumulator
      else
        mbar_arrive_cluster(acc == 0 ? lead_tempty0 : lead_tempty1);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lead_t && use_tma_c) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if (SOLO)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(512));
  }
}

}  // namespace

template <int KIND, bool SH, bool BMN = false, bool SOLO = false>
int launch(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbs,
           const CUtensorMap &mc, const CUtensorMap &ms, int use_tma_c, const Epi &ep, int64_t M,
           int64_t N, const Sched &sch, int clusters, cudaStream_t s) {
  constexpr size_t smem = Lay<SH, SOLO>::SMEM;
  auto kernel = gemm_tc2_kernel<KIND, SH, BMN, SOLO>;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kernel<<<2 * clusters, PTHREADS, smem, s>>>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

// K x N row-major bf16 B viewed as [N / 64][K][64] (a 64-wide N chunk's
// rows are its 128-byte swizzled K rows): boxes of `chunks` x 64 K x 64 N.
// N must be a multiple of 64 for the view (host-checked); the K tail is
// zero-filled.
bool make_map_kn(CUtensorMap *map, int kind, const void *B, int64_t K, int64_t N,
                 uint32_t chunks) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  const int elem = kind == 0 ? 2 : 4;
  const cuuint32_t ch = 128 / elem;     // N per chunk row; K rows per box = BK = ch too
  cuuint64_t dims[3] = {ch, (cuuint64_t)K, (cuuint64_t)(N / ch)};
  cuuint64_t strides[2] = {(cuuint64_t)(N * elem), 128};
  cuuint32_t box[3] = {ch, ch, chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             3, const_cast<void *>(B), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_gemm_tc2(int kind, const void *A, const void *Bt, const Epi &ep, int64_t M, int64_t N,
                    int64_t K, int max_clusters, cudaStream_t s, const void *Bkn, bool solo) {
  if (solo && Bkn) return B200_EUNSUPPORTED;
  // MN-major operands are a 16-bit-type feature: tf32 B read MN-major came
  // out wrong on the B200 (tools/probe_gemm_kn.py --kind 1), so kind 0 only
  if (Bkn && (kind != 0 || N % 64 != 0)) return B200_EUNSUPPORTED;
  Sched sch;
  sch.nt = (N + 255) / 256;
  sch.tiles = ((M + 255) / 256) * sch.nt;
  sch.kb_total = (K * (kind == 0 ? 2 : 4) + 127) / 128;
  int clusters = num_sms() / 2;
  if (max_clusters > 0 && max_clusters < clusters) clusters = max_clusters;
  if (sch.tiles < clusters) clusters = (int)sch.tiles;
  sch.ncl = clusters;
  sch.waves = sch.tiles / clusters;
  sch.rem = sch.tiles - sch.waves * clusters;
  sch.split = 1;
  const char *genv = getenv("B200_TC2_GROUP");   // dev A/B knob
  sch.group_m = genv ? atoi(genv) : 8;
  if (sch.group_m < 1) sch.group_m = 1;
  const char *env = getenv("B200_TC2_SPLIT");
  if (sch.rem > 0 && !(env && env[0] == '0')) {
    const int64_t S = clusters / sch.rem;
    sch.split = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1));
  }
  CUtensorMap ma, mb, mbs, mc;
  if (!make_map(&ma, kind, A, M, K, 128)) return B200_ELAUNCH;
  if (Bkn) {
    // whole halves: 128 N = 128 / CH chunks; tail items: their brows in chunks
    const int64_t ch = kind == 0 ? 64 : 32, tail = 128 / sch.split;
    if (!make_map_kn(&mb, kind, Bkn, K, N, (uint32_t)(128 / ch)) ||
        !make_map_kn(&mbs, kind, Bkn, K, N, (uint32_t)(tail >= ch ? tail / ch : 1)))
      return B200_ELAUNCH;
  } else if (!make_map(&mb, kind, Bt, N, K, 128) ||
             !make_map(&mbs, kind, Bt, N, K, (uint32_t)(128 / sch.split))) {
    return B200_ELAUNCH;
  }
  // staged epilogue needs unit column stride and 16-byte aligned rows
  int use_tma_c = ep.sCn == 1 && (ep.sCm * 4) % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(ep.C) & 15) == 0 && ep.sCm >= N;
  if (use_tma_c && !make_map_c(&mc, ep.C, M, N, ep.sCm, 128)) use_tma_c = 0;
  if (!use_tma_c) mc = ma;  // unused placeholder
  // staged shadow: TMA-storable bf16 rows (16-byte aligned base and pitch)
  CUtensorMap ms = ma;
  const bool sh = use_tma_c && ep.c16 && (ep.ld16 * 2) % 16 == 0 && ep.ld16 >= N &&
                  (reinterpret_cast<uintptr_t>(ep.c16) & 15) == 0 &&
                  make_map_s16(&ms, ep.c16, M, N, ep.ld16, 128);
  if (Bkn)
    return sh ? launch<0, true, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters, s)
              : launch<0, false, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters,
                                       s);
  if (solo) {
    if (kind == 0)
      return sh ? launch<0, true, false, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch,
                                               clusters, s)
                : launch<0, false, false, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch,
                                                clusters, s);
    return sh ? launch<1, true, false, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch,
                                             clusters, s)
              : launch<1, false, false, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch,
                                              clusters, s);
  }
  if (kind == 0)
    return sh ? launch<0, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters, s)
              : launch<0, false>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters, s);
  return sh ? launch<1, true>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters, s)
            : launch<1, false>(ma, mb, mbs, mc, ms, use_tma_c, ep, M, N, sch, clusters, s);
}

}  // namespace b200tc
