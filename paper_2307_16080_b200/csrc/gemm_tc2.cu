// 2-SM tensor-core contraction: a CTA pair (cluster of 2) computes a 256x256
// output tile with tcgen05.mma.cta_group::2 (UMMA M=256, N=256).
//
// Each CTA stages its own half of the operands — 128 rows of A and 128 rows of
// B^T per 128-byte K slice — so per SM the TMA traffic per MMA is half of the
// single-CTA 128x256 kernel's.  Only the leader CTA (cluster rank 0) issues
// MMAs; both CTAs' TMA loads complete on the leader's full-barrier, MMA
// commits are multicast to both CTAs' empty / tmem-full barriers, and both
// CTAs' epilogues release the accumulator buffer on the leader's tmem-empty
// barrier.  Each CTA's TMEM holds its 128 rows x 256 columns of the fp32
// accumulator (2 buffers = 512 columns, epilogue of tile i overlaps the MMAs
// of tile i+1).
//
// Work schedule: persistent clusters walk full tiles round-robin; the tiles of
// the last, partial wave are split S = floor(clusters / remaining) ways along
// K so the tail wave is balanced.  Split parts write fp32 partials to a
// workspace and take a ticket; the last part to finish combines
// C + P_0 + ... + P_{S-1} in fixed order (deterministic, no inter-CTA waits).
//
// Epilogue (C = C + acc [+ bias]): C is staged through shared memory in
// 128-row x 32-column chunks by TMA (128B swizzle, 4 buffers): the loads of
// upcoming chunks — including the next tile's — are issued ahead, each thread
// adds its TMEM row in place, and a TMA bulk store writes the chunk back.
// (Strided C falls back to per-row 128-bit stores.)
//
// Replaces run_tape on a recognised matmul / Linear contraction nest
// (reference tests/kernels.py:24-38) at bf16/tf32 precision.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"
#include "tc_common.cuh"

namespace b200tc {

namespace {

constexpr int PSTAGES = 5;
constexpr int PA = 128 * 128;   // A half: 128 rows x 128 B
constexpr int PB = 128 * 128;   // B half: 128 rows x 128 B
constexpr int CBUF = 128 * 128; // C chunk: 128 rows x 32 fp32
constexpr int NCBUF = 4;
constexpr int PTHREADS = 256;
constexpr size_t PSMEM = 1024 + PSTAGES * (PA + PB) + NCBUF * CBUF + 256;

struct Sched {
  int64_t tiles, nt, kb_total, ncl;
  int64_t waves;   // full waves of whole tiles
  int64_t rem;     // tiles in the partial wave
  int64_t split;   // parts per tail tile (1 = no split)
};

struct Item {
  int64_t t;       // tile index
  int64_t kb0, kb1;
  int part;        // -1 whole tile, else split part
  int64_t tail;    // tail tile ordinal (split items)
};

__device__ __forceinline__ bool get_item(const Sched &s, int64_t cid, int64_t i, Item &it) {
  if (i < s.waves) {
    it.t = cid + i * s.ncl;
    it.kb0 = 0;
    it.kb1 = s.kb_total;
    it.part = -1;
    it.tail = -1;
    return true;
  }
  if (i == s.waves && cid < s.rem * s.split) {
    const int64_t tt = cid / s.split;
    it.t = s.waves * s.ncl + tt;
    if (s.split == 1) {
      it.kb0 = 0;
      it.kb1 = s.kb_total;
      it.part = -1;
      it.tail = -1;
    } else {
      it.part = (int)(cid % s.split);
      it.tail = tt;
      it.kb0 = it.part * s.kb_total / s.split;
      it.kb1 = (it.part + 1) * s.kb_total / s.split;
    }
    return true;
  }
  return false;
}

template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tma_a,
                    const __grid_constant__ CUtensorMap tma_b,
                    const __grid_constant__ CUtensorMap tma_c, int use_tma_c, Epi ep, int64_t M,
                    int64_t N, Sched sch, float *ws, int *ws_cnt) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t sA = base;
  const uint32_t sB = base + PSTAGES * PA;
  const uint32_t sC = base + PSTAGES * (PA + PB);
  unsigned char *gC = gbase + PSTAGES * (PA + PB);
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + PSTAGES * (PA + PB) + NCBUF * CBUF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * PSTAGES + 4 + NCBUF);
  int *ticket_slot = reinterpret_cast<int *>(tmem_slot + 1);
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

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 256);
    }
    for (int b = 0; b < NCBUF; ++b) mbar_init(cbar(b), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t cid = blockIdx.x / 2;
  const int64_t nt = sch.nt;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      Item it;
      for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
        const int32_t m0 = (int32_t)((it.t / nt) * 256 + rank * 128);
        const int32_t n0 = (int32_t)((it.t % nt) * 256 + rank * 128);
        for (int64_t kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait(empty(s), ph ^ 1);
          if (leader) mbar_expect_tx(full(s), 2 * (PA + PB));
          const uint32_t lf = map_to_rank(full(s), 0);
          tma_load_2d_pair(&tma_a, lf, sA + s * PA, (int32_t)(kb * BK), m0);
          tma_load_2d_pair(&tma_b, lf, sB + s * PB, (int32_t)(kb * BK), n0);
          if (++s == PSTAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, 256, 256);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      Item it;
      for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
        mbar_wait_cluster(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * 256);
        for (int64_t kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait(full(s), ph);
          tc_fence_after();
          const uint32_t a_addr = sA + s * PA, b_addr = sB + s * PB;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma<KIND, 2>(tmem_d, smem_desc(a_addr + 32 * k), smem_desc(b_addr + 32 * k), idesc,
                          (kb != it.kb0 || k != 0));
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
    // chunk g of this CTA: work item g / 8, columns (g % 8) * 32 (whole tiles only)
    auto chunk_coords = [&](int64_t g, int32_t &col, int32_t &row) -> bool {
      Item ci;
      if (!get_item(sch, cid, g / 8, ci) || ci.part >= 0) return false;
      row = (int32_t)((ci.t / nt) * 256 + rank * 128);
      col = (int32_t)((ci.t % nt) * 256 + (g % 8) * 32);
      return true;
    };
    auto issue_load = [&](int64_t g) {
      int32_t col, row;
      if (!chunk_coords(g, col, row)) return;
      const int b = (int)(g % NCBUF);
      mbar_expect_tx(cbar(b), CBUF);
      tma_load_2d(&tma_c, cbar(b), sC + b * CBUF, col, row);
    };
    if (load_c && lead_t)
      for (int64_t g = 0; g < NCBUF - 1; ++g) issue_load(g);
    int acc = 0;
    uint32_t aph = 0;
    int64_t g = 0;
    const uint32_t lead_tempty0 = map_to_rank(tempty(0), 0);
    const uint32_t lead_tempty1 = map_to_rank(tempty(1), 0);
    Item it;
    for (int64_t i = 0; get_item(sch, cid, i, it); ++i) {
      const int64_t m_base = (it.t / nt) * 256 + rank * 128;
      const int64_t n0 = (it.t % nt) * 256;
      mbar_wait_cluster(tfull(acc), aph);
      tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256);
      if (it.part >= 0) {
        // split part: fp32 partial of this CTA's 128 x 256 block -> workspace
        float *P = ws + ((it.tail * sch.split + it.part) * 2 + rank) * (128 * 256);
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t r[32];
          tmem_ld32(trow + (uint32_t)(c * 32), r);
          float4 *dst = reinterpret_cast<float4 *>(P + et * 256 + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        g += 8;
        tc_fence_before();
        mbar_arrive_cluster(acc == 0 ? lead_tempty0 : lead_tempty1);
        __threadfence();
        named_bar_sync(1, 128);
        if (lead_t) *ticket_slot = atomicAdd(&ws_cnt[it.tail * 2 + rank], 1);
        named_bar_sync(1, 128);
        if (*ticket_slot == sch.split - 1) {
          // last part: C = C + P_0 + ... + P_{S-1} in part order
          __threadfence();
          const int64_t m = m_base + et;
          if (m < M) {
            for (int c = 0; c < 256; c += 4) {
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              for (int p = 0; p < sch.split; ++p) {
                // L2 (coherent) loads: the partials were written by other SMs
                const float4 w = __ldcg(reinterpret_cast<const float4 *>(
                    ws + ((it.tail * sch.split + p) * 2 + rank) * (128 * 256) + et * 256 + c));
                v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
              }
              for (int j = 0; j < 4; ++j) {
                const int64_t n = n0 + c + j;
                if (n >= N) break;
                float *dst = ep.C + m * ep.sCm + n * ep.sCn;
                float o = ep.init ? ep.init_value : *dst;
                o += (&v.x)[j];
                if (ep.bias) o += ep.bias[n * ep.bias_stride];
                *dst = o;
              }
            }
          }
          named_bar_sync(1, 128);
          if (lead_t) ws_cnt[it.tail * 2 + rank] = 0;  // reset for the next launch
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < 8; ++c, ++g) {
          uint32_t r[32];
          tmem_ld32(trow + (uint32_t)(c * 32), r);
          if (use_tma_c) {
            const int b = (int)(g % NCBUF);
            if (load_c) {
              mbar_wait(cbar(b), (uint32_t)((g / NCBUF) & 1));
            } else {
              // no C load: make sure the store of chunk g-4 has left this buffer
              if (lead_t) bulk_wait_read<NCBUF - 1>();
              named_bar_sync(1, 128);
            }
            epilogue_chunk_smem(gC + b * CBUF, et, n0 + c * 32, N, ep, r);
            fence_proxy_async();
            named_bar_sync(1, 128);
            if (lead_t) {
              tma_store_2d(&tma_c, sC + b * CBUF, (int32_t)(n0 + c * 32), (int32_t)m_base);
              bulk_commit();
              if (load_c) {
                bulk_wait_read<1>();  // store of chunk g-1 has read buffer (g+3) % 4
                issue_load(g + NCBUF - 1);
              }
            }
          } else {
            epilogue_row32(ep, m_base + et, n0 + c * 32, M, N, r);
          }
        }
        tc_fence_before();
        mbar_arrive_cluster(acc == 0 ? lead_tempty0 : lead_tempty1);
      }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lead_t && use_tma_c) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
}

// split-K workspace: fp32 partials + per-(tail tile, rank) tickets (zeroed
// once; the last part of every tile resets its ticket).  One launch at a time.
float *g_ws = nullptr;
int *g_cnt = nullptr;
size_t g_ws_floats = 0, g_cnt_n = 0;

bool ensure_ws(size_t floats, size_t cnt, cudaStream_t s) {
  if (floats > g_ws_floats) {
    if (g_ws) cudaFree(g_ws);
    if (cudaMalloc(&g_ws, floats * sizeof(float)) != cudaSuccess) {
      g_ws = nullptr;
      g_ws_floats = 0;
      return false;
    }
    g_ws_floats = floats;
  }
  if (cnt > g_cnt_n) {
    if (g_cnt) cudaFree(g_cnt);
    if (cudaMalloc(&g_cnt, cnt * sizeof(int)) != cudaSuccess) {
      g_cnt = nullptr;
      g_cnt_n = 0;
      return false;
    }
    cudaMemsetAsync(g_cnt, 0, cnt * sizeof(int), s);
    g_cnt_n = cnt;
  }
  return true;
}

}  // namespace

int launch_gemm_tc2(int kind, const void *A, const void *Bt, const Epi &ep, int64_t M, int64_t N,
                    int64_t K, int max_clusters, cudaStream_t s) {
  CUtensorMap ma, mb, mc;
  if (!make_map(&ma, kind, A, M, K, 128) || !make_map(&mb, kind, Bt, N, K, 128))
    return B200_ELAUNCH;
  // staged epilogue needs unit column stride and 16-byte aligned rows
  int use_tma_c = ep.sCn == 1 && (ep.sCm * 4) % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(ep.C) & 15) == 0 && ep.sCm >= N;
  if (use_tma_c && !make_map_c(&mc, ep.C, M, N, ep.sCm, 128)) use_tma_c = 0;
  if (!use_tma_c) mc = ma;  // unused placeholder
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
  if (sch.rem > 0) {
    int64_t S = clusters / sch.rem;
    if (S > sch.kb_total) S = sch.kb_total;
    if (S > 8) S = 8;
    if (S >= 2) sch.split = S;
  }
  if (sch.split > 1 &&
      !ensure_ws((size_t)sch.rem * sch.split * 2 * 128 * 256, (size_t)sch.rem * 2, s))
    sch.split = 1;
  if (kind == 0) {
    cudaFuncSetAttribute(gemm_tc2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)PSMEM);
    gemm_tc2_kernel<0><<<2 * clusters, PTHREADS, PSMEM, s>>>(ma, mb, mc, use_tma_c, ep, M, N, sch,
                                                            g_ws, g_cnt);
  } else {
    cudaFuncSetAttribute(gemm_tc2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)PSMEM);
    gemm_tc2_kernel<1><<<2 * clusters, PTHREADS, PSMEM, s>>>(ma, mb, mc, use_tma_c, ep, M, N, sch,
                                                            g_ws, g_cnt);
  }
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace b200tc
