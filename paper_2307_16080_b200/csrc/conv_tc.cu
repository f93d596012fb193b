// Tensor-core implicit-GEMM convolution (NCHW / FCHW, valid, stride 1) on sm_100a.
//
//   out[n, f, ho, wo] (+)= sum_{ci, ki, kj} in[n, ci, ho+ki, wo+kj] * w[f, ci, ki, kj]
//
// Replaces run_tape on the conv_2d_nchw_fchw nest (reference
// tests/kernels.py:50-64; the engine recognises it from
// the separable contraction's index maps) when the engine precision is bf16.
// The tensor core accumulates in fp32; the only deviations from the
// reference's (ci, ki, kj)-ordered f32 chain are accumulation order and the
// bf16 operand rounding (tolerance: DESIGN.md, tests/test_gpu_conv.py).
//
// Halo reuse.  The input is repacked once per call to NHWC bf16, channels
// padded to a multiple of 64 (b200_pack_conv_input), so one pixel of one
// 64-channel block is a 128-byte row.  Each output tile's input patch arrives
// as ONE 128B-swizzled TMA box per channel block, and every filter tap is a
// K-major SW128 UMMA descriptor over that same patch (start shifted by the
// tap, SBO = one patch row): A traffic per tile is the patch, not one
// shifted tile per tap.  The 128B swizzle is a function of absolute shared
// memory address bits, so shifted starts need no descriptor base offset.
//
// Two tilings (template R, struct Tiling):
//  R == 1   tile 16 rows x 8 columns (M = 128 = row * 8 + col), patch rows of
//           PW = 8 + KW - 1 pixels; one UMMA 128 x F x 16 per (tap, 16
//           channels).
//  R == KW  (KW * F <= 256) the KW horizontal taps are merged into N: tile
//           4 rows x 28 columns over patch rows of 32 pixels (M = 128 =
//           row * 32 + col), one UMMA 128 x (KW * F) x 16 per (ki, 16
//           channels) against the KW weight slices stacked as B rows
//           (kj, f).  The epilogue sums the KW partial products of output
//           (h, w) from TMEM lanes (h, w + kj), columns kj * F + f, with warp
//           shuffles.  At F = 64 a 128 x 64 x 16 UMMA is paced by a per-
//           instruction cost (~110 cycles measured, 32 of math); N = 192
//           amortises it over 3x the work.
//
// Weights ([F][KH][KW][Cp] bf16, K-major) stay resident in shared memory for
// the whole kernel.  Output blocks [F][TH][TW] fp32 are staged through
// shared memory: TMA-loaded ahead by a loader warp (out += conv reads the
// previous output), updated in place by the epilogue, TMA-stored (rows and
// columns past the image clipped).  Outputs that are not a legal tensor map
// (unaligned strides) take a direct register path instead.
// Structure per CTA (persistent over tiles):
//   warp 0  TMA producer (weights once; one patch per (tile, channel block))
//   warp 1  MMA issuer
//   warp 2  TMEM allocator (2 accumulator buffers of R * F columns)
//   warp 3  output-block loader (ring of up to 3 blocks)
//   warps 4-11 epilogue, two warpgroups splitting the output channels:
//           thread = TMEM lane = tile pixel
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/b200k.h"
#include "tc_common.cuh"

using namespace b200tc;

namespace {

constexpr int kMaxStages = 6;             // patch pipeline depth (runtime, smem permitting)
constexpr int kMaxOut = 3;                // staged output blocks (runtime)
constexpr int kThreads = 384;              // 4 control warps + 2 epilogue warpgroups
constexpr int kConvThreads = 128;          // fused: + 1 converter warpgroup (warps 12-15)
constexpr int kMaxRaw = 8;                 // fused: raw f32 chunk buffers (runtime, smem permitting)
constexpr int kRawCh = 8;                  // fused: channels per raw chunk
constexpr size_t kSmemMax = 232448;
int *b200_conv_trace_host = nullptr;

// Tile geometry of tiling R.  ROWLEN: pixels per patch row = per M row group
// (M = 128 = TH * ROWLEN); TW: output columns per tile — R > 1 loses the
// last KW - 1 columns of each row to the merged taps' halo, rounded down so
// that a tile's row is a whole number of 16-byte units (TMA store boxes).
template <int F, int R>
struct Tiling {
  static constexpr int ROWLEN = R == 1 ? 8 : 32;
  static constexpr int TH = 128 / ROWLEN;
  static constexpr int TW = R == 1 ? 8 : 28;
  static constexpr int TPIX = TH * TW;                // staged output pixels per channel
  static constexpr int OUTBUF = F * TPIX * 4;         // staged output block [F][TH][TW] fp32
};

struct ConvGeo {
  int64_t nb, cp, hp, wp, f, ho, wo, kh, kw;
  int64_t so_n, so_f, so_h, so_w;   // output element strides
  int64_t th_tiles, tw_tiles, tiles;
  int th, tw;        // output tile rows / valid columns
  int ph, prow;      // patch rows / patch row length in pixels
  int cblocks, stages;
  int nout;          // staged output blocks: previous output TMA-loaded, updated in
                     // shared memory, TMA-stored (0: unaligned output, the epilogue
                     // reads and writes global memory directly)
  int patch_bytes;   // bytes one patch box delivers (transaction count)
  int pstage;        // smem stride of a patch stage (1024-aligned)
  int init;
  float init_value;
  unsigned long long *stats;   // dev: per-role wait cycles (B200_CONV_STATS), or null
  // fused (NCHW f32 input read by the kernel): a raw chunk is ONE TMA box
  // over the input viewed as [N][C][H / 2][2 W] (row pairs: a 16-byte
  // multiple pitch where single rows are not): `npair` row pairs x `blen`
  // pixels (W + prow, rounded to 4) x kRawCh channels; `rstages` buffers of
  // `raw_bytes`
  int blen, npair, raw_bytes, rstages, c;
  // dev: per-CTA progress counters in mapped host memory (B200_CONV_TRACE),
  // [cta][8]: producer units, converter patches, mma patches, epilogue
  // tiles, loader tiles; or null
  volatile int *trace;
};
#define TRACE(slot, v)                                           \
  do {                                                           \
    if (g.trace) {                                               \
      g.trace[blockIdx.x * 8 + (slot)] = (v);                    \
    }                                                            \
  } while (0)

// dev instrumentation: cycles spent in a wait, per role slot
#define TIMED(slot, stmt)                          \
  do {                                             \
    if (g.stats) {                                 \
      const long long t0_ = clock64();             \
      stmt;                                        \
      st[slot] += clock64() - t0_;                 \
    } else {                                       \
      stmt;                                        \
    }                                              \
  } while (0)

__device__ __forceinline__ void tma_load_4d(const CUtensorMap *map, uint32_t bar, uint32_t dst,
                                            int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, uint32_t src, int32_t c0,
                                             int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// K-major SW128 operand whose 8-row groups are `sbo` bytes apart; the start
// may sit anywhere on a 16-byte boundary inside the swizzle atom.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 16 TMEM columns of this warp's 32 lanes, without the completion wait.
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// PAIR (fused only, launched as 2-CTA clusters): the two column tiles of a
// row band run on the two CTAs of a cluster as ONE cta_group::2 MMA
// (M = 2 x 128 pixels, N = KW x F): each CTA keeps only half of the stacked
// weight rows (B is split along N across the pair), which frees the shared
// memory for a third patch stage; each CTA converts its own tile's patch
// from its own copy of the band; the leader issues the MMAs.
template <int F, int R, bool FUSED = false, bool PAIR = false>
__global__ void __launch_bounds__(kThreads + (FUSED ? kConvThreads : 0), 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tma_in,
                   const __grid_constant__ CUtensorMap tma_w,
                   const __grid_constant__ CUtensorMap tma_out, float *__restrict__ out,
                   ConvGeo g) {
  constexpr int N = R * F;                   // UMMA N
  constexpr int SLICE = F * 128;             // one (tap, channel block) weight slice
  constexpr uint32_t TCOLS = 2 * N <= 32 ? 32 : (2 * N <= 64 ? 64 : (2 * N <= 128 ? 128 :
                                                  (2 * N <= 256 ? 256 : 512)));
  using T = Tiling<F, R>;
  constexpr int ROWLEN = T::ROWLEN;          // pixels per tile row in the M ordering
  constexpr int TPIX = T::TPIX;
  constexpr int OUTBUF = T::OUTBUF;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const int taps = (int)(g.kh * g.kw);
  const int nslices = taps * g.cblocks;
  const int stages = g.stages;
  const uint32_t pstage = (uint32_t)g.pstage;
  constexpr int WSL = PAIR ? SLICE / 2 : SLICE;  // this CTA's bytes of a weight slice
  const uint32_t sB = base;                                   // nslices x WSL
  const uint32_t sP = base + nslices * WSL;                   // stages x patch
  const uint32_t sO = sP + stages * pstage;                   // nout x OUTBUF
  float *gO = reinterpret_cast<float *>(gbase + (sO - base));
  const uint32_t sR = sO + g.nout * OUTBUF;                   // fused: rstages raw chunks
  const float *gR = reinterpret_cast<const float *>(gbase + (sR - base));
  uint64_t *bars = reinterpret_cast<uint64_t *>(
      gbase + (sR - base) + (FUSED ? g.rstages * g.raw_bytes : 0));
  uint32_t *tmem_slot =
      reinterpret_cast<uint32_t *>(bars + 2 * kMaxStages + 5 + 2 * kMaxOut + 2 * kMaxRaw);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (kMaxStages + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * kMaxStages + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * kMaxStages + 2 + a); };
  const uint32_t wbar = bar0 + 8u * (2 * kMaxStages + 4);
  auto ofull = [&](int b) { return bar0 + 8u * (2 * kMaxStages + 5 + b); };
  auto oempty = [&](int b) { return bar0 + 8u * (2 * kMaxStages + 5 + kMaxOut + b); };
  auto rfull = [&](int r) { return bar0 + 8u * (2 * kMaxStages + 5 + 2 * kMaxOut + r); };
  auto rempty = [&](int r) {
    return bar0 + 8u * (2 * kMaxStages + 5 + 2 * kMaxOut + kMaxRaw + r);
  };

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  long long st[5] = {0, 0, 0, 0, 0};
  const long long t_start = clock64();
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      // fused: the converter warps fill a patch stage and each arrives
      // (PAIR: both CTAs' converters, on the leader's barrier)
      mbar_init(full(s), FUSED ? (PAIR ? 2 : 1) * kConvThreads / 32 : 1);
      mbar_init(empty(s), 1);
    }
    if (FUSED)
      for (int r = 0; r < g.rstages; ++r) {
        mbar_init(rfull(r), 1);
        mbar_init(rempty(r), 1);   // the one converter warp that owns the chunk
      }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), PAIR ? 512 : 256);   // PAIR: both CTAs' epilogues, on the leader
    }
    for (int b = 0; b < g.nout; ++b) {
      mbar_init(ofull(b), 1);
      mbar_init(oempty(b), 1);   // the storing thread, once the block's store has read it
    }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // 32-bit tile decomposition (tiles < 2^31, checked on the host): 64-bit
  // division is a long software sequence on the epilogue's critical path
  const uint32_t per_img = (uint32_t)(g.th_tiles * g.tw_tiles);
  const uint32_t twt = (uint32_t)g.tw_tiles;
  auto tile_coords = [&](int64_t t, int32_t &n, int32_t &h0, int32_t &w0) {
    const uint32_t tt = (uint32_t)t;
    const uint32_t nn = tt / per_img, r = tt - nn * per_img;
    const uint32_t ty = r / twt;
    n = (int32_t)nn;
    h0 = (int32_t)(ty * g.th);
    w0 = (int32_t)((r - ty * twt) * g.tw);
  };

  // this CTA's tile sequence: strided tiles, or (fused) whole row bands — a
  // band's tw_tiles tiles back to back, so its input rows are loaded and
  // converted once for all of them
  const int64_t twt64 = g.tw_tiles;
  const int64_t nbands = g.tiles / twt64;
  auto tile_at = [&](int64_t i) -> int64_t {   // -1: no more tiles
    if (PAIR) {   // band cid + i * clusters; this CTA's column tile = its rank
      const int64_t band = blockIdx.x / 2 + i * (int64_t)(gridDim.x / 2);
      return band < nbands ? band * twt64 + rank : -1;
    }
    if (!FUSED) {
      const int64_t t = blockIdx.x + i * (int64_t)gridDim.x;
      return t < g.tiles ? t : -1;
    }
    const int64_t band = blockIdx.x + (i / twt64) * (int64_t)gridDim.x;
    return band < nbands ? band * twt64 + i % twt64 : -1;
  };

  if (warp == 0) {
    if (lane == 0) {
      // resident weights: slice (ki, kj, cb) = rows f of columns
      // [(ki * KW + kj) * cp + cb * 64, +64); R == 1 orders slices
      // (tap, cb), R > 1 orders them (ki, cb, kj) so that the KW slices of
      // one (ki, cb) stack into the N = KW * F rows of a single B operand
      if (PAIR) {
        // this CTA's half of each (ki, cb) group's stacked rows (kj, f):
        // half-slices hs = 2 kj + (f >= F / 2) in [rank R, rank R + R),
        // counted on the leader's weight barrier (both halves)
        if (leader) mbar_expect_tx(wbar, (uint32_t)(nslices * SLICE));
        const uint32_t lw = map_to_rank(wbar, 0);
        for (int ki = 0; ki < (int)g.kh; ++ki)
          for (int cb = 0; cb < g.cblocks; ++cb)
            for (int h = 0; h < R; ++h) {
              const int hs = (int)rank * R + h, kj = hs / 2, hf = hs % 2;
              const int tap = ki * (int)g.kw + kj;
              tma_load_2d_pair(&tma_w, lw,
                               sB + (ki * g.cblocks + cb) * R * WSL + h * (F / 2) * 128,
                               (int32_t)(tap * g.cp + cb * 64), hf * (F / 2));
            }
      } else {
        mbar_expect_tx(wbar, (uint32_t)(nslices * SLICE));
        for (int tap = 0; tap < taps; ++tap) {
          const int ki = tap / (int)g.kw, kj = tap % (int)g.kw;
          for (int cb = 0; cb < g.cblocks; ++cb) {
            const int slot = R == 1 ? tap * g.cblocks + cb : (ki * g.cblocks + cb) * R + kj;
            tma_load_2d(&tma_w, wbar, sB + slot * SLICE, (int32_t)(tap * g.cp + cb * 64), 0);
          }
        }
      }
      int s = 0;
      uint32_t ph = 0;
      int64_t rq = 0;   // fused: raw chunk stream index
      for (int64_t i = 0, t; (t = tile_at(i)) >= 0; ++i) {
        int32_t n, h0, w0;
        tile_coords(t, n, h0, w0);
        for (int cb = 0; cb < g.cblocks; ++cb) {
          if (FUSED) {
            // raw f32 chunks of kRawCh channels, once per row band (its
            // first tile): one box of whole row pairs h0 / 2 .. + npair - 1.
            // Chunk q of the stream goes to converter warp q % 4's own ring
            // (rstages / 4 buffers): a buffer is only ever waited on by one
            // warp, in order — the mbarrier parity test cannot tell use k
            // from use k - 2, so two warps sharing a buffer would race
            if (!PAIR && i % twt64 != 0) continue;
            const int pw = g.rstages / 4;
            for (int j = 0; j < 64 / kRawCh; ++j) {
              const int64_t q = (rq++);
              const int64_t k = q / 4;
              const int rb = (int)(q % 4) * pw + (int)(k % pw);
              const uint32_t rph = (uint32_t)((k / pw) & 1);
              TIMED(0, mbar_wait(rempty(rb), rph ^ 1));
              mbar_expect_tx(rfull(rb), (uint32_t)g.raw_bytes);
              tma_load_4d(&tma_in, rfull(rb), sR + rb * g.raw_bytes, 0, h0 / 2,
                          cb * 64 + j * kRawCh, n);
              TRACE(0, (int)(q + 1));
            }
            continue;
          }
          TIMED(0, mbar_wait(empty(s), ph ^ 1));
          mbar_expect_tx(full(s), (uint32_t)g.patch_bytes);
          tma_load_4d(&tma_in, full(s), sP + s * pstage, cb * 64, w0, h0, n);
          if (++s == stages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (PAIR && lane == 0 && leader) {
      // one cta_group::2 MMA per (ki, 16 channels): A = each CTA's own
      // patch (M 2 x 128), B = the (ki, cb) group's stacked rows split across
      // the pair (N / 2 per CTA); commits reach both CTAs
      constexpr uint32_t idesc = make_idesc(0, 256, N);
      mbar_wait_cluster(wbar, 0);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t i = 0, t; (t = tile_at(i)) >= 0; ++i) {
        TIMED(2, mbar_wait_cluster(tempty(acc), aph ^ 1));
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * N);
        for (int cb = 0; cb < g.cblocks; ++cb) {
          TIMED(1, mbar_wait_cluster(full(s), ph));
          tc_fence_after();
          const uint64_t a0 = desc_sw128(sP + s * pstage, 1024);
          uint32_t acc_flag = cb != 0;
          for (int ki = 0; ki < (int)g.kh; ++ki) {
            const uint64_t ad = a0 + (uint64_t)ki * g.prow * 8;
            const uint64_t bd = desc_sw128(sB + (ki * g.cblocks + cb) * R * WSL, 1024);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              umma<0, 2>(tmem_d, ad + 2 * k, bd + 2 * k, idesc, acc_flag);
              acc_flag = 1;
            }
          }
          umma_commit_pair(empty(s), 0x3);
          if (++s == stages) { s = 0; ph ^= 1; }
        }
        umma_commit_pair(tfull(acc), 0x3);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    } else if (!PAIR && lane == 0) {
      constexpr uint32_t idesc = make_idesc(0, 128, N);
      // 8-pixel M groups: one patch row apart (R == 1), or back to back
      // (R > 1: two groups per 16-pixel patch row)
      const uint32_t sbo = R == 1 ? (uint32_t)g.prow * 128 : 1024;
      mbar_wait(wbar, 0);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t i = 0, t; (t = tile_at(i)) >= 0; ++i) {
        TIMED(2, mbar_wait(tempty(acc), aph ^ 1));
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * N);
        for (int cb = 0; cb < g.cblocks; ++cb) {
          TIMED(1, mbar_wait(full(s), ph));
          tc_fence_after();
          // descriptors advance in 16-byte units of their start-address
          // field: +2 per 16-channel k step
          const uint64_t a0 = desc_sw128(sP + s * pstage, sbo);
          uint32_t acc_flag = cb != 0;
          if (R == 1) {
            // per tap: A shifted by (ki * PW + kj) pixels, B = slice (tap, cb)
            uint64_t ad = a0;
            uint64_t bd = desc_sw128(sB + cb * SLICE, 1024);
            const uint64_t b_tap = (uint64_t)(g.cblocks * SLICE) >> 4;
            for (int ki = 0; ki < (int)g.kh; ++ki) {
              for (int kj = 0; kj < (int)g.kw; ++kj) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  umma<0, 1>(tmem_d, ad + 2 * k, bd + 2 * k, idesc, acc_flag);
                  acc_flag = 1;
                }
                ad += 8;
                bd += b_tap;
              }
              ad += (uint64_t)(g.prow - g.kw) * 8;
            }
          } else {
            // per ki: A shifted by ki patch rows, B = the KW stacked slices
            // of (ki, cb)
            for (int ki = 0; ki < (int)g.kh; ++ki) {
              const uint64_t ad = a0 + (uint64_t)ki * g.prow * 8;
              const uint64_t bd =
                  desc_sw128(sB + (ki * g.cblocks + cb) * R * SLICE, 1024);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                umma<0, 1>(tmem_d, ad + 2 * k, bd + 2 * k, idesc, acc_flag);
                acc_flag = 1;
              }
            }
          }
          umma_commit(empty(s));
          if (++s == stages) { s = 0; ph ^= 1; }
          TRACE(2, (int)i * 4 + cb + 1);
        }
        umma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp == 3) {
    if (lane == 0 && g.nout > 0) {
      // output-tile loader: the previous output block [F][TH][TW] of each
      // tile, TMA-loaded into a ring of nout buffers (for init, the buffer
      // is only handed over once its last store has drained)
      int b = 0;
      uint32_t ph = 0;
      for (int64_t i = 0, t; (t = tile_at(i)) >= 0; ++i) {
        int32_t n, h0, w0;
        tile_coords(t, n, h0, w0);
        mbar_wait(oempty(b), ph ^ 1);
        if (g.init) {
          mbar_arrive(ofull(b));
        } else {
          mbar_expect_tx(ofull(b), (uint32_t)OUTBUF);
          tma_load_4d(&tma_out, ofull(b), sO + b * OUTBUF, w0, h0, 0, n);
        }
        if (++b == g.nout) { b = 0; ph ^= 1; }

      }
    }
  } else if (FUSED && warp >= 12) {
    // converter warpgroup: raw f32 [kRawCh][npair][blen] chunks -> the bf16
    // patch stage ([ph][ROWLEN px][64 ch], 128-byte pixel rows, 128B swizzle:
    // the 16-byte channel group k of pixel p sits at k ^ (p & 7)).  The four
    // warps convert different chunks at once — chunk q of the stream goes to
    // warp q % 4 — so their load-to-store latencies overlap; a warp releases
    // its raw buffer alone (rempty count 1) and the patch is full once all
    // four have arrived.  Lane task = a pixel pair of one patch row: 8 LDS.64
    // (channel rows of the chunk), 8 packs, two 16-byte stores.  Patch row y
    // is row pair y / 2 at offset (y % 2) W; W even keeps pairs 8-byte aligned.
    const int cw = warp - 12;
    constexpr int NCH = 64 / kRawCh;   // chunks per 64-channel patch (cblocks == 1)
    const int npairs = g.ph * ROWLEN / 2;
    const int cstride = g.npair * g.blen;   // floats between a chunk's channels
    // the band's tiles this CTA converts: all of them, or (PAIR) its own
    const int twt = PAIR ? 1 : (int)twt64;
    const int tx0 = PAIR ? (int)rank : 0;
    int s = 0;
    uint32_t ph = 0;
    int64_t bi = 0;   // band index of this CTA's stream
    for (int64_t i = 0, t; (t = tile_at(i)) >= 0; i += twt, ++bi) {
      // the band's tiles take the next twt patch stages
      for (int k = 0, ss = s; k < twt; ++k) {
        mbar_wait(empty(ss), (ss >= s ? ph : ph ^ 1) ^ 1);
        if (++ss == stages) ss = 0;
      }
      for (int j = cw; j < NCH; j += 4) {
        const int64_t q = bi * NCH + j;   // q % 4 == cw: this warp's ring
        const int64_t k = q / 4;
        const int pw = g.rstages / 4;
        const int rs = cw * pw + (int)(k % pw);
        mbar_wait(rfull(rs), (uint32_t)((k / pw) & 1));
        const float *raw = gR + rs * (g.raw_bytes / 4);
        for (int tx = 0, ss = s; tx < twt; ++tx) {
          unsigned char *patch = gbase + (sP - base) + ss * pstage;
          const int w0 = (tx0 + tx) * g.tw;
          for (int tp = lane; tp < npairs; tp += 32) {
            const int p = 2 * tp;
            const int y = p / ROWLEN, x = p % ROWLEN;
            const float *src = raw + (y >> 1) * g.blen + (y & 1) * (int)g.wp + w0 + x;
            __nv_bfloat162 v0[4], v1[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float2 a = *reinterpret_cast<const float2 *>(src + (2 * c) * cstride);
              const float2 b = *reinterpret_cast<const float2 *>(src + (2 * c + 1) * cstride);
              v0[c] = __floats2bfloat162_rn(a.x, b.x);
              v1[c] = __floats2bfloat162_rn(a.y, b.y);
            }
            *reinterpret_cast<uint4 *>(patch + p * 128 + ((j ^ (p & 7)) << 4)) =
                *reinterpret_cast<uint4 *>(v0);
            *reinterpret_cast<uint4 *>(patch + (p + 1) * 128 + ((j ^ ((p + 1) & 7)) << 4)) =
                *reinterpret_cast<uint4 *>(v1);
          }
          if (++ss == stages) ss = 0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(rempty(rs));
      }
      fence_proxy_async();   // generic-proxy stores -> the tensor cores' reads
      __syncwarp();
      for (int k = 0; k < twt; ++k) {
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(map_to_rank(full(s), 0));   // the leader issues the MMA
          else
            mbar_arrive(full(s));
        }
        if (++s == stages) { s = 0; ph ^= 1; }
      }
      if (lane == 0) TRACE(cw == 0 ? 1 : 4 + cw, (int)(i + twt));
    }
  } else if (warp >= 4) {
    // two epilogue warpgroups: warp w reads TMEM lanes 32 * (w % 4) + [0, 32)
    // (its lane quadrant) and warpgroup e takes the 16-column chunks
    // e, e + 2, e + 4, ... of the F output channels
    const int m = (warp % 4) * 32 + lane;   // TMEM lane = tile pixel (row * ROWLEN + col)
    const int e = (warp - 4) / 4;
    const int hr = m / ROWLEN, wc = m % ROWLEN;
    const bool lane_ok = wc < g.tw;         // R > 1: the last KW - 1 (+ pad) columns are halo
    const int sf = (int)g.so_f;   // channel stride in elements (< 2^31 / F, host-checked)
    constexpr int CH = F / 32 > 0 ? F / 32 : 1;   // 16-column chunks per warpgroup
    int acc = 0;
    uint32_t aph = 0;
    int ob = 0;
    uint32_t oph = 0;
    for (int64_t i = 0, t; (t = tile_at(i)) >= 0; ++i) {
      int32_t n, h0, w0;
      tile_coords(t, n, h0, w0);
      const bool valid = lane_ok && h0 + hr < g.ho && w0 + wc < g.wo;
      float *const o = out + n * g.so_n + (h0 + hr) * g.so_h + (w0 + wc) * g.so_w;
      if (PAIR)
        TIMED(3, mbar_wait_cluster(tfull(acc), aph));
      else
        TIMED(3, mbar_wait(tfull(acc), aph));
      tc_fence_after();
      // staged: this pixel's [c][row][col] slot of the TMA-loaded block,
      // updated in place and stored back by TMA
      float *st_px = gO + ob * (OUTBUF / 4) + hr * T::TW + wc;
      if (g.nout > 0) TIMED(4, mbar_wait(ofull(ob), oph));
      const uint32_t trow = tmem_base + ((uint32_t)((warp % 4) * 32) << 16) + (uint32_t)(acc * N);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int c0 = 16 * e + 32 * c;
        if (c0 >= F) break;
        uint32_t v[R][16];
#pragma unroll
        for (int kj = 0; kj < R; ++kj) tmem_ld16_nowait(trow + (uint32_t)(kj * F + c0), v[kj]);
        float prev[16];
        if (g.nout > 0 && !g.init) {
#pragma unroll
          for (int j = 0; j < 16; ++j) prev[j] = lane_ok ? st_px[(c0 + j) * TPIX] : 0.f;
        } else if (!g.init && valid) {
#pragma unroll
          for (int j = 0; j < 16; ++j) prev[j] = o[(c0 + j) * sf];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) prev[j] = g.init_value;
        }
        tmem_wait_ld();
        // all 16 results first (independent shuffles interleave), then one
        // branch around the stores
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float sum = __uint_as_float(v[0][j]);
#pragma unroll
          for (int kj = 1; kj < R; ++kj)
            sum += __shfl_down_sync(0xffffffffu, __uint_as_float(v[kj][j]), kj);
          prev[j] += sum;
        }
        if (g.nout > 0) {
          if (lane_ok) {
#pragma unroll
            for (int j = 0; j < 16; ++j) st_px[(c0 + j) * TPIX] = prev[j];
          }
        } else if (valid) {
          float *pc = o + c0 * sf;
#pragma unroll
          for (int j = 0; j < 16; ++j) pc[j * sf] = prev[j];
        }
      }
      tc_fence_before();
      if (PAIR)
        mbar_arrive_cluster(map_to_rank(tempty(acc), 0));
      else
        mbar_arrive(tempty(acc));
      if (++acc == 2) { acc = 0; aph ^= 1; }
      if (threadIdx.x == 128) TRACE(3, (int)i * 2 + 1);
      if (g.nout > 0) {
        // the block goes back by one TMA store (out-of-range rows/columns
        // clipped); buffer ob - 1 is released once its own store has read it
        fence_proxy_async();
        named_bar_sync(1, 256);
        if (threadIdx.x == 128) {
          tma_store_4d(&tma_out, sO + ob * OUTBUF, w0, h0, 0, n);
          bulk_commit();
          if (g.nout == 1) {
            // a single buffer: the next tile's load waits for this store
            bulk_wait_read<0>();
            mbar_arrive(oempty(0));
          } else if (i != 0) {
            bulk_wait_read<1>();
            mbar_arrive(oempty(ob == 0 ? g.nout - 1 : ob - 1));
          }
        }
        if (++ob == g.nout) { ob = 0; oph ^= 1; }
        if (threadIdx.x == 128) TRACE(3, (int)i * 2 + 2);
      }
    }
    if (g.nout > 0 && threadIdx.x == 128) bulk_wait_all();
  }
  if (g.stats && lane == 0) {
    const unsigned long long tot = (unsigned long long)(clock64() - t_start);
    if (warp == 0) {
      atomicAdd(&g.stats[0], (unsigned long long)st[0]);
      atomicAdd(&g.stats[8], tot);
    } else if (warp == 1) {
      atomicAdd(&g.stats[1], (unsigned long long)st[1]);
      atomicAdd(&g.stats[2], (unsigned long long)st[2]);
      atomicAdd(&g.stats[9], tot);
    } else if (warp == 4) {
      atomicAdd(&g.stats[3], (unsigned long long)st[3]);
      atomicAdd(&g.stats[4], (unsigned long long)st[4]);
      atomicAdd(&g.stats[10], tot);
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TCOLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TCOLS));
  }
}

// NCHW f32 (any strides) -> NHWC bf16 with channels padded to cp (zeros).
// Register transpose, no shared memory.  The input is a set of `lines` of
// `len` pixels (an image's whole H * W plane when its rows are contiguous,
// else one row) and a work unit is (line, block of 32 * WI pixels, 64-channel
// pass).  Warp k of a CTA owns the unit's 8-channel chunk k: its lanes read
// the 8 channel runs (8 * WI coalesced loads in flight per thread) and each
// lane writes one pixel's 8 channels as a 16-byte bf16 vector.  The 8 warps
// of the CTA fill each pixel's 128-byte line within the same few hundred
// cycles, so L2 merges the 16-byte pieces before DRAM.  Units are
// grid-strided and the next unit's loads are issued before the current
// unit's converts and stores (the kernel is latency-bound otherwise).
constexpr int PACK_MAXW = 256;
constexpr int PACK_WI = 4;
template <int WI>
__global__ void __launch_bounds__(256) pack_nhwc_kernel(const float *__restrict__ src, int64_t sN,
                                                        int64_t sC, int64_t sH, int64_t sP,
                                                        __nv_bfloat16 *__restrict__ dst, int C,
                                                        int lines_per_img, int len, int cp,
                                                        int64_t lines) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int passes = cp / 64;
  const int blocks = (len + 32 * WI - 1) / (32 * WI);
  const int64_t units = lines * blocks * passes;
  float v[2][8][WI];
  auto coords = [&](int64_t u, int64_t &line, int &p0, int &c0) {
    const int64_t lb = u / passes;
    c0 = (int)(u - lb * passes) * 64 + warp * 8;
    line = lb / blocks;
    p0 = (int)(lb - line * blocks) * 32 * WI;
  };
  auto load = [&](float (&r)[8][WI], int64_t u) {
    int64_t line;
    int p0, c0;
    coords(u, line, p0, c0);
    const float *base = src + (line / lines_per_img) * sN + (line % lines_per_img) * sH;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < WI; ++i) {
        const int p = p0 + lane + 32 * i;
        r[k][i] = (c0 + k < C && p < len)
                      ? __ldg(base + (int64_t)(c0 + k) * sC + (int64_t)p * sP) : 0.f;
      }
  };
  auto store = [&](const float (&r)[8][WI], int64_t u) {
    int64_t line;
    int p0, c0;
    coords(u, line, p0, c0);
    __nv_bfloat16 *base = dst + line * (int64_t)len * cp + c0;
#pragma unroll
    for (int i = 0; i < WI; ++i) {
      const int p = p0 + lane + 32 * i;
      if (p < len) {
        __nv_bfloat162 b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(r[2 * j][i], r[2 * j + 1][i]);
        *reinterpret_cast<uint4 *>(base + (int64_t)p * cp) = *reinterpret_cast<uint4 *>(b);
      }
    }
  };
  int64_t u = blockIdx.x;
  if (u < units) load(v[0], u);
  for (; u < units; u += 2 * (int64_t)gridDim.x) {
    const int64_t u1 = u + gridDim.x;
    if (u1 < units) load(v[1], u1);
    store(v[0], u);
    if (u1 >= units) break;
    if (u1 + gridDim.x < units) load(v[0], u1 + gridDim.x);
    store(v[1], u1);
  }
}

// Same units and register transpose as pack_nhwc_kernel, but the CTA's
// [32 WI pixels][64 channels] bf16 tile is assembled in shared memory (128B
// swizzle: pixel p's 16-byte chunk k at k ^ (p & 7), so a quarter warp's
// 16-byte stores hit 8 distinct bank groups) and written by ONE TMA store of
// whole 128-byte pixel rows (pixels past the line clipped by the tensor
// map), instead of 16-byte pieces from eight warps that L2 has to merge.
// Two tiles alternate; a tile is rewritten only after its store has read it.
template <int WI>
__global__ void __launch_bounds__(256) pack_nhwc_tma_kernel(
    const float *__restrict__ src, int64_t sN, int64_t sC, int64_t sH, int64_t sP,
    const __grid_constant__ CUtensorMap tmap, int C, int lines_per_img, int len, int cp,
    int64_t lines) {
  constexpr int TILE = 32 * WI * 128;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int passes = cp / 64;
  const int blocks = (len + 32 * WI - 1) / (32 * WI);
  const int64_t units = lines * blocks * passes;
  float v[2][8][WI];
  auto coords = [&](int64_t u, int64_t &line, int &p0, int &c0) {
    const int64_t lb = u / passes;
    c0 = (int)(u - lb * passes) * 64;
    line = lb / blocks;
    p0 = (int)(lb - line * blocks) * 32 * WI;
  };
  auto load = [&](float (&r)[8][WI], int64_t u) {
    int64_t line;
    int p0, c0;
    coords(u, line, p0, c0);
    c0 += warp * 8;
    const float *bp = src + (line / lines_per_img) * sN + (line % lines_per_img) * sH;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < WI; ++i) {
        const int p = p0 + lane + 32 * i;
        r[k][i] = (c0 + k < C && p < len)
                      ? __ldg(bp + (int64_t)(c0 + k) * sC + (int64_t)p * sP) : 0.f;
      }
  };
  int b = 0;
  auto put = [&](const float (&r)[8][WI], int64_t u) {
    if (threadIdx.x == 0) bulk_wait_read<1>();   // the store of this tile's last use has read it
    __syncthreads();
    unsigned char *tile = gbase + b * TILE;
#pragma unroll
    for (int i = 0; i < WI; ++i) {
      const int p = lane + 32 * i;
      __nv_bfloat162 h[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(r[2 * j][i], r[2 * j + 1][i]);
      *reinterpret_cast<uint4 *>(tile + p * 128 + ((warp ^ (p & 7)) << 4)) =
          *reinterpret_cast<uint4 *>(h);
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t line;
      int p0, c0;
      coords(u, line, p0, c0);
      tma_store_4d(&tmap, base + b * TILE, c0, p0, (int32_t)line, 0);
      bulk_commit();
    }
    b ^= 1;
  };
  int64_t u = blockIdx.x;
  if (u < units) load(v[0], u);
  for (; u < units; u += 2 * (int64_t)gridDim.x) {
    const int64_t u1 = u + gridDim.x;
    if (u1 < units) load(v[1], u1);
    put(v[0], u);
    if (u1 >= units) break;
    if (u1 + gridDim.x < units) load(v[0], u1 + gridDim.x);
    put(v[1], u1);
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// All-bulk variant for whole-plane lines (the usual dense NCHW input): the
// unit's [64 channels][128 pixels] f32 block arrives by one TMA load (rows of
// 512 bytes; pixels past the plane and channels past C zero-filled, which is
// the channel padding), double-buffered; each thread reads its 4 pixels' 8
// channels from shared memory (consecutive pixels across lanes: no bank
// conflicts), converts, and assembles the swizzled bf16 tile that one TMA
// store writes back.  No global loads by threads: the HBM stream is all TMA.
constexpr int BULK_PX = 128;
// FCHW f32 weights -> [F][KH][KW][cp] bf16, optionally packed by the same
// launch as the input (b200_pack_conv: the weights are a few hundred KB, so
// their share of each CTA hides behind its first TMA load)
struct WPack {
  const float *src;
  int64_t sF, sC, sKH, sKW;
  __nv_bfloat16 *dst;   // null: no weights in this launch
  int F, C, KH, KW, cp;
};
__device__ __forceinline__ void pack_weights(const WPack &w, int64_t first, int64_t stride) {
  const int total = w.F * w.KH * w.KW * w.cp, taps = w.KH * w.KW;
  for (int64_t i = first; i < total; i += stride) {
    const int c = (int)(i % w.cp), ft = (int)(i / w.cp);
    const int tap = ft % taps, f = ft / taps;
    const int ki = tap / w.KW, kj = tap - ki * w.KW;
    w.dst[i] = __float2bfloat16_rn(
        c < w.C ? w.src[f * w.sF + c * w.sC + ki * w.sKH + kj * w.sKW] : 0.f);
  }
}

__global__ void __launch_bounds__(256) pack_nhwc_bulk_kernel(
    const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int len,
    int cp, int64_t lines, WPack wp) {
  constexpr int IN_TILE = 64 * BULK_PX * 4, OUT_TILE = BULK_PX * 128;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t sIn = base, sOut = base + 2 * IN_TILE;
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + 2 * IN_TILE + 2 * OUT_TILE);
  const uint32_t bar0 = smem_u32(bars);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int passes = cp / 64;
  const int blocks = (len + BULK_PX - 1) / BULK_PX;
  const int64_t units = lines * blocks * passes;
  auto coords = [&](int64_t u, int64_t &line, int &p0, int &c0) {
    const int64_t lb = u / passes;
    c0 = (int)(u - lb * passes) * 64;
    line = lb / blocks;
    p0 = (int)(lb - line * blocks) * BULK_PX;
  };
  auto issue = [&](int64_t u, int st) {
    int64_t line;
    int p0, c0;
    coords(u, line, p0, c0);
    mbar_expect_tx(bar0 + 8u * st, IN_TILE);
    tma_load_4d(&tin, bar0 + 8u * st, sIn + st * IN_TILE, p0, c0, (int32_t)line, 0);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = blockIdx.x, step = gridDim.x;
  if (threadIdx.x == 0) {
    if (u0 < units) issue(u0, 0);
    if (u0 + step < units) issue(u0 + step, 1);
  }
  if (wp.dst)   // while the first loads are in flight
    pack_weights(wp, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                 (int64_t)gridDim.x * blockDim.x);
  int st = 0, ob = 0;
  uint32_t ph = 0;
  for (int64_t u = u0; u < units; u += step) {
    mbar_wait(bar0 + 8u * st, ph);
    if (threadIdx.x == 0) bulk_wait_read<1>();   // the store of out tile ob's last use has read it
    __syncthreads();
    const float *in = reinterpret_cast<const float *>(gbase + st * IN_TILE);   // [64][128]
    unsigned char *tile = gbase + 2 * IN_TILE + ob * OUT_TILE;
#pragma unroll
    for (int i = 0; i < BULK_PX / 32; ++i) {
      const int p = lane + 32 * i;
      __nv_bfloat162 h[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        h[j] = __floats2bfloat162_rn(in[(8 * warp + 2 * j) * BULK_PX + p],
                                     in[(8 * warp + 2 * j + 1) * BULK_PX + p]);
      *reinterpret_cast<uint4 *>(tile + p * 128 + ((warp ^ (p & 7)) << 4)) =
          *reinterpret_cast<uint4 *>(h);
    }
    fence_proxy_async();
    __syncthreads();   // input stage st consumed, out tile ob complete
    if (threadIdx.x == 0) {
      int64_t line;
      int p0, c0;
      coords(u, line, p0, c0);
      tma_store_4d(&tout, sOut + ob * OUT_TILE, c0, p0, (int32_t)line, 0);
      bulk_commit();
      if (u + 2 * step < units) issue(u + 2 * step, st);
    }
    ob ^= 1;
    if (++st == 2) { st = 0; ph ^= 1; }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// FCHW f32 weights -> [F][KH][KW][cp] bf16 (K order: tap, channel).
// One thread per destination element; 32-bit index math (the tensor is at
// most F * KH * KW * cp < 2^31 elements, host-checked).
__global__ void pack_wt_kernel(const float *__restrict__ src, int64_t sF, int64_t sC,
                               int64_t sKH, int64_t sKW, __nv_bfloat16 *__restrict__ dst,
                               int F, int C, int KH, int KW, int cp) {
  const int total = F * KH * KW * cp;
  const int taps = KH * KW;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % cp, ft = i / cp;
    const int tap = ft % taps, f = ft / taps;
    const int ki = tap / KW, kj = tap - ki * KW;
    dst[i] = __float2bfloat16_rn(c < C ? src[f * sF + c * sC + ki * sKH + kj * sKW] : 0.f);
  }
}

bool make_map_4d(CUtensorMap *map, CUtensorMapDataType dt, const void *ptr, const cuuint64_t *dims,
                 const cuuint64_t *strides_bytes, const cuuint32_t *box, CUtensorMapSwizzle sw) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, dt, 4, const_cast<void *>(ptr), dims, strides_bytes, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Merge factor: the KW horizontal taps go into N when KW * F fits one UMMA
// (instantiated for 3x3 at F <= 64 and 5x5 at F = 32).  Mirrored by
// runtime.conv_tc_supported.
int conv_merge(int64_t f, int64_t kw) {
  if (getenv("B200_CONV_NOMERGE")) return 1;   // dev knob: force the 16 x 8 tiling
  return (kw == 3 && (f == 32 || f == 64)) || (kw == 5 && f == 32) ? (int)kw : 1;
}

// Shared memory of the kernel (weights, `stages` patch stages, `nout` staged
// output blocks of `outbuf` bytes, barriers, alignment).  Mirrored by
// runtime.conv_tc_supported (2 stages, no staged output blocks).
size_t conv_smem(int64_t f, int64_t kh, int64_t kw, int64_t cp, int64_t pstage, int stages,
                 int nout, int64_t outbuf, int64_t raw_bytes = 0, int rstages = 0,
                 bool pair = false) {
  return 1024 + kh * kw * (cp / 64) * f * 128 / (pair ? 2 : 1) + stages * pstage +
         nout * outbuf +
         rstages * raw_bytes + 512;   // barriers (39 x 8 bytes) + the TMEM slot
}

// FUSED: `in` is the NCHW f32 input itself (dense planes; see
// b200_conv2d_tc_fused), read by TMA as [N][C][H * W] and converted in the
// kernel; otherwise `in` is the NHWC bf16 repack.
template <int F, int R, bool FUSED = false, bool PAIR = false>
int launch_conv(const void *in, const int64_t *in_strides, const void *wt, float *out,
                ConvGeo &g, cudaStream_t s) {
  using T = Tiling<F, R>;
  const int64_t raw = FUSED ? g.raw_bytes : 0;
  // fused: at least 2 raw chunk buffers; the staged output blocks are capped
  // at 2 so the rest of shared memory deepens the raw ring (its TMA loads
  // are what hides the input's latency)
  const int rmin = FUSED ? 4 : 0;
  auto smem_of = [&](int stages, int nout, int rst = -1) {
    return conv_smem(F, g.kh, g.kw, g.cp, g.pstage, stages, nout, T::OUTBUF, raw,
                     rst < 0 ? rmin : rst, PAIR);
  };
  CUtensorMap mi, mw, mo;
  if (FUSED) {
    // [N][C][H / 2][2 W] f32: row pairs of 8 W bytes (16-byte multiples)
    cuuint64_t di[4] = {(cuuint64_t)(2 * g.wp), (cuuint64_t)(g.hp / 2), (cuuint64_t)g.c,
                        (cuuint64_t)g.nb};
    cuuint64_t si[3] = {(cuuint64_t)(2 * g.wp * 4), (cuuint64_t)(in_strides[1] * 4),
                        (cuuint64_t)(in_strides[0] * 4)};
    cuuint32_t bi[4] = {(cuuint32_t)g.blen, (cuuint32_t)g.npair, (cuuint32_t)kRawCh, 1};
    if (!make_map_4d(&mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, in, di, si, bi,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
      return B200_ELAUNCH;
  } else {
    cuuint64_t di[4] = {(cuuint64_t)g.cp, (cuuint64_t)g.wp, (cuuint64_t)g.hp, (cuuint64_t)g.nb};
    cuuint64_t si[3] = {(cuuint64_t)(g.cp * 2), (cuuint64_t)(g.wp * g.cp * 2),
                        (cuuint64_t)(g.hp * g.wp * g.cp * 2)};
    // the whole patch of one 64-channel block per box, rows of 128 B, swizzled
    cuuint32_t bi[4] = {64, (cuuint32_t)g.prow, (cuuint32_t)g.ph, 1};
    if (!make_map_4d(&mi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in, di, si, bi,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return B200_ELAUNCH;
  }
  // PAIR: each CTA loads half-slices of F / 2 rows
  if (!make_map(&mw, 0, wt, F, g.kh * g.kw * g.cp, PAIR ? F / 2 : F)) return B200_ELAUNCH;
  if (smem_of(2, 0) > kSmemMax) return B200_EUNSUPPORTED;
  // output blocks staged through shared memory (TMA load, in-place update,
  // TMA store) when the NCHW output is a legal tensor map: 16-byte aligned
  // base and strides, unit w stride.  Box origins are multiples of TW
  // columns = 32 bytes.
  g.nout = 0;
  const bool tma_ok = g.so_w == 1 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                      (g.so_h * 4) % 16 == 0 && (g.so_f * 4) % 16 == 0 &&
                      (g.so_n * 4) % 16 == 0;
  if (tma_ok) {
    cuuint64_t dout[4] = {(cuuint64_t)g.wo, (cuuint64_t)g.ho, (cuuint64_t)F, (cuuint64_t)g.nb};
    cuuint64_t sout[3] = {(cuuint64_t)(g.so_h * 4), (cuuint64_t)(g.so_f * 4),
                          (cuuint64_t)(g.so_n * 4)};
    cuuint32_t bout[4] = {(cuuint32_t)T::TW, (cuuint32_t)T::TH, F, 1};
    if (make_map_4d(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, dout, sout, bout,
                    CU_TENSOR_MAP_SWIZZLE_NONE)) {
      const char *env = getenv("B200_CONV_NOUT");   // dev knob
      g.nout = env ? atoi(env) : (FUSED ? 2 : kMaxOut);
      if (g.nout > kMaxOut) g.nout = kMaxOut;
      while (g.nout > 0 && smem_of(2, g.nout) > kSmemMax) --g.nout;
    }
  }
  if (g.nout == 0) mo = mi;   // unused placeholder
  g.stages = kMaxStages;
  if (FUSED) {
    const char *env = getenv("B200_CONV_RAW");   // dev knob
    g.rstages = env ? atoi(env) : kMaxRaw;
    if (g.rstages > kMaxRaw) g.rstages = kMaxRaw;
    g.rstages &= ~3;   // one ring per converter warp
    while (g.rstages > 4 && smem_of(2, g.nout, g.rstages) > kSmemMax) g.rstages -= 4;
    if (g.rstages < 4) g.rstages = 4;
  }
  while (smem_of(g.stages, g.nout, g.rstages) > kSmemMax) --g.stages;
  const size_t smem = smem_of(g.stages, g.nout, g.rstages);
  if (FUSED && !PAIR && g.stages < g.tw_tiles) return B200_EUNSUPPORTED;   // a band's patches
  int ctas = num_sms();
  const int64_t units = FUSED ? g.tiles / g.tw_tiles : g.tiles;   // fused: row bands
  if (PAIR) {
    ctas = 2 * (int)(units < num_sms() / 2 ? units : num_sms() / 2);   // clusters of 2
  } else if (units < ctas) {
    ctas = (int)units;
  }
  cudaFuncSetAttribute(conv_tc_kernel<F, R, FUSED, PAIR>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (getenv("B200_CONV_TRACE")) {   // dev: progress counters the host can read while it runs
    static int *host_trace = nullptr;
    if (!host_trace) cudaHostAlloc(&host_trace, 8 * 1024 * sizeof(int), cudaHostAllocMapped);
    memset(host_trace, 0, 8 * 1024 * sizeof(int));
    int *dev = nullptr;
    cudaHostGetDevicePointer(&dev, host_trace, 0);
    g.trace = dev;
    b200_conv_trace_host = host_trace;
  }
  const bool stats = getenv("B200_CONV_STATS") != nullptr;   // dev: print role wait cycles
  if (stats) {
    cudaMalloc(&g.stats, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(g.stats, 0, 16 * sizeof(unsigned long long), s);
  }
  if (PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(kThreads + kConvThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, conv_tc_kernel<F, R, FUSED, PAIR>, mi, mw, mo, out, g);
  } else {
    conv_tc_kernel<F, R, FUSED>
        <<<ctas, kThreads + (FUSED ? kConvThreads : 0), smem, s>>>(mi, mw, mo, out, g);
  }
  if (stats) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, g.stats, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(g.stats);
    const double c = ctas;
    fprintf(stderr,
            "conv stats (kcycles/CTA): producer total %.1f wait-empty %.1f | mma total %.1f "
            "wait-full %.1f wait-tempty %.1f | epilogue total %.1f wait-tfull %.1f "
            "wait-out %.1f | "
            "R %d stages %d staged output blocks %d raw stages %d tiles %lld\n",
            h[8] / c / 1e3, h[0] / c / 1e3, h[9] / c / 1e3, h[1] / c / 1e3, h[2] / c / 1e3,
            h[10] / c / 1e3, h[3] / c / 1e3, h[4] / c / 1e3, R, g.stages, g.nout, g.rstages,
            (long long)g.tiles);
  }
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace

namespace {
// The input pack; `wp` (dst non-null) is folded into the launch when the
// all-bulk kernel applies (*wp_done set), else left to the caller.
int pack_input(const float *src, const int64_t *sstr, void *dst, int64_t nb, int64_t c,
               int64_t h, int64_t w, int64_t cp, cudaStream_t stream, WPack wp, bool *wp_done) {
  *wp_done = false;
  if (nb == 0) return B200_OK;   // an empty batch shard: nothing to convert
  if (nb < 0 || h <= 0 || w <= 0 || cp < c || cp % 64 || w > PACK_MAXW) return B200_EINVAL;
  // rows contiguous (h stride = W * w stride): one line per image plane
  const bool plane = sstr[2] == w * sstr[3];
  const int lines_per_img = plane ? 1 : (int)h;
  const int len = plane ? (int)(h * w) : (int)w;
  const int64_t lines = nb * lines_per_img;
  const int64_t units = lines * ((len + 32 * PACK_WI - 1) / (32 * PACK_WI)) * (cp / 64);
  // the TMA-stored variant: dst rows of cp bf16 (a 16-byte multiple) as a
  // [lines][len][cp] tensor, 1024-byte-aligned shared tiles
  CUtensorMap tmap;
  const cuuint64_t dims[4] = {(cuuint64_t)cp, (cuuint64_t)len, (cuuint64_t)lines, 1};
  const cuuint64_t strides[3] = {(cuuint64_t)(cp * 2), (cuuint64_t)(len * cp * 2),
                                 (cuuint64_t)(lines * len * cp * 2)};
  const cuuint32_t box[4] = {64, 32 * PACK_WI, 1, 1};
  const bool tma_out = !getenv("B200_PACK_OLD") && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                       make_map_4d(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dst, dims, strides,
                                   box, CU_TENSOR_MAP_SWIZZLE_128B);
  // all-bulk loads: whole-plane lines with unit pixel stride and 16-byte
  // channel / image strides, viewed as [nb][C][len] f32
  CUtensorMap imap;
  const cuuint64_t idims[4] = {(cuuint64_t)len, (cuuint64_t)c, (cuuint64_t)nb, 1};
  const cuuint64_t istr[3] = {(cuuint64_t)(sstr[1] * 4), (cuuint64_t)(sstr[0] * 4),
                              (cuuint64_t)(nb * sstr[0] * 4)};
  const cuuint32_t ibox[4] = {BULK_PX, 64, 1, 1};
  const cuuint32_t obox[4] = {64, BULK_PX, 1, 1};
  CUtensorMap omap;
  if (tma_out && plane && sstr[3] == 1 && sstr[1] % 4 == 0 && sstr[0] % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(src) & 15) == 0 && !getenv("B200_PACK_NOBULK") &&
      make_map_4d(&imap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, src, idims, istr, ibox,
                  CU_TENSOR_MAP_SWIZZLE_NONE) &&
      make_map_4d(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dst, dims, strides, obox,
                  CU_TENSOR_MAP_SWIZZLE_128B)) {
    const int64_t bunits = lines * ((len + BULK_PX - 1) / BULK_PX) * (cp / 64);
    const int smem = 1024 + 2 * 64 * BULK_PX * 4 + 2 * BULK_PX * 128 + 64;
    cudaFuncSetAttribute(pack_nhwc_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pack_nhwc_bulk_kernel, 256, smem);
    int64_t blocks = (int64_t)num_sms() * (per_sm < 1 ? 1 : per_sm);
    if (blocks > bunits) blocks = bunits;
    pack_nhwc_bulk_kernel<<<(unsigned)blocks, 256, smem, stream>>>(imap, omap, len, (int)cp,
                                                                  lines, wp);
    *wp_done = wp.dst != nullptr;
    return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
  }
  if (tma_out) {
    const int smem = 1024 + 2 * 32 * PACK_WI * 128;
    auto kernel = pack_nhwc_tma_kernel<PACK_WI>;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem);
    int64_t blocks = (int64_t)num_sms() * (per_sm < 1 ? 1 : per_sm);
    if (blocks > units) blocks = units;
    kernel<<<(unsigned)blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(
        src, sstr[0], sstr[1], sstr[2], sstr[3], tmap, (int)c, lines_per_img, len, (int)cp,
        lines);
    return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pack_nhwc_kernel<PACK_WI>, 256, 0);
  int64_t blocks = (int64_t)num_sms() * (per_sm < 1 ? 1 : per_sm);
  if (blocks > units) blocks = units;
  pack_nhwc_kernel<PACK_WI><<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, sstr[0], sstr[1], sstr[2], sstr[3], static_cast<__nv_bfloat16 *>(dst), (int)c,
      lines_per_img, len, (int)cp, lines);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}
}  // namespace

extern "C" int b200_pack_conv_input(const float *src, const int64_t *sstr, void *dst, int64_t nb,
                                    int64_t c, int64_t h, int64_t w, int64_t cp, void *stream) {
  bool unused;
  return pack_input(src, sstr, dst, nb, c, h, w, cp, static_cast<cudaStream_t>(stream),
                    WPack{}, &unused);
}

extern "C" int b200_pack_conv(const float *src, const int64_t *sstr, void *dst, int64_t nb,
                              int64_t c, int64_t h, int64_t w, int64_t cp, const float *ker,
                              const int64_t *swt, void *wdst, int64_t f, int64_t kh, int64_t kw,
                              void *stream) {
  const int64_t total = f * kh * kw * cp;
  if (total <= 0 || cp % 64) return B200_EINVAL;
  if (total >= (int64_t(1) << 31)) return B200_EUNSUPPORTED;
  WPack wp{ker, swt[0], swt[1], swt[2], swt[3], static_cast<__nv_bfloat16 *>(wdst), (int)f,
           (int)c, (int)kh, (int)kw, (int)cp};
  bool done = false;
  const int rc = pack_input(src, sstr, dst, nb, c, h, w, cp, static_cast<cudaStream_t>(stream),
                            wp, &done);
  if (rc != B200_OK || done) return rc;
  return b200_pack_conv_weight(ker, swt, wdst, f, c, kh, kw, cp, stream);
}

extern "C" int b200_pack_conv_weight(const float *src, const int64_t *sstr, void *dst, int64_t f,
                                     int64_t c, int64_t kh, int64_t kw, int64_t cp,
                                     void *stream) {
  const int64_t total = f * kh * kw * cp;
  if (total <= 0 || cp % 64) return B200_EINVAL;
  if (total >= (int64_t(1) << 31)) return B200_EUNSUPPORTED;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  pack_wt_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, sstr[0], sstr[1], sstr[2], sstr[3], static_cast<__nv_bfloat16 *>(dst), (int)f,
      (int)c, (int)kh, (int)kw, (int)cp);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

namespace {
// Tile / patch geometry shared by both entry points; false: outside the
// kernel's 32-bit index limits.
bool conv_geo(ConvGeo &g, const int64_t *out_strides, int64_t nb, int64_t cp, int64_t hp,
              int64_t wp, int64_t f, int64_t ho, int64_t wo, int64_t kh, int64_t kw, int32_t init,
              float init_value) {
  g = ConvGeo{};
  g.nb = nb; g.cp = cp; g.hp = hp; g.wp = wp; g.f = f; g.ho = ho; g.wo = wo;
  g.kh = kh; g.kw = kw; g.init = init; g.init_value = init_value;
  g.so_n = out_strides[0]; g.so_f = out_strides[1];
  g.so_h = out_strides[2]; g.so_w = out_strides[3];
  const int R = conv_merge(f, kw);
  if (R == 1) {   // Tiling<F, 1>
    g.th = 16; g.tw = 8; g.prow = (int)(8 + kw - 1);
  } else {        // Tiling<F, KW>: 4 rows of 32 patch pixels, 28 output columns
    g.th = 4; g.tw = 28; g.prow = 32;
  }
  g.ph = (int)(g.th + kh - 1);
  g.th_tiles = (ho + g.th - 1) / g.th;
  g.tw_tiles = (wo + g.tw - 1) / g.tw;
  g.tiles = nb * g.th_tiles * g.tw_tiles;
  g.cblocks = (int)(cp / 64);
  g.patch_bytes = g.ph * g.prow * 128;
  g.pstage = (g.patch_bytes + 1023) & ~1023;
  // 32-bit tile indices and per-pixel channel offsets in the kernel
  return !(g.ph > 256 || g.prow > 256 || g.tiles + 2 * 148 >= (int64_t(1) << 31) ||
           out_strides[1] < 0 || out_strides[1] * f >= (int64_t(1) << 31));
}
}  // namespace

extern "C" int b200_conv2d_tc(const void *in_nhwc, const void *wt, float *out,
                              const int64_t *out_strides, int64_t nb, int64_t cp, int64_t hp,
                              int64_t wp, int64_t f, int64_t ho, int64_t wo, int64_t kh,
                              int64_t kw, int32_t init, float init_value, void *stream) {
  if (cp % 64 || ho <= 0 || wo <= 0 || kh <= 0 || kw <= 0 || ho + kh - 1 > hp ||
      wo + kw - 1 > wp || nb < 0)
    return B200_EINVAL;
  if (nb == 0) return B200_OK;   // an empty batch shard (shard.py)
  ConvGeo g;
  if (!conv_geo(g, out_strides, nb, cp, hp, wp, f, ho, wo, kh, kw, init, init_value))
    return B200_EUNSUPPORTED;
  const int R = conv_merge(f, kw);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (f * 16 + R) {
    case 32 * 16 + 1: return launch_conv<32, 1>(in_nhwc, nullptr, wt, out, g, s);
    case 64 * 16 + 1: return launch_conv<64, 1>(in_nhwc, nullptr, wt, out, g, s);
    case 128 * 16 + 1: return launch_conv<128, 1>(in_nhwc, nullptr, wt, out, g, s);
    case 32 * 16 + 3: return launch_conv<32, 3>(in_nhwc, nullptr, wt, out, g, s);
    case 64 * 16 + 3: return launch_conv<64, 3>(in_nhwc, nullptr, wt, out, g, s);
    case 32 * 16 + 5: return launch_conv<32, 5>(in_nhwc, nullptr, wt, out, g, s);
    default: return B200_EUNSUPPORTED;
  }
}

extern "C" int b200_conv2d_tc_fused(const float *in, const int64_t *in_strides, const void *wt,
                                    float *out, const int64_t *out_strides, int64_t nb,
                                    int64_t c, int64_t hp, int64_t wp, int64_t f, int64_t ho,
                                    int64_t wo, int64_t kh, int64_t kw, int32_t init,
                                    float init_value, void *stream) {
  if (c <= 0 || ho <= 0 || wo <= 0 || kh <= 0 || kw <= 0 || ho + kh - 1 > hp ||
      wo + kw - 1 > wp || nb < 0)
    return B200_EINVAL;
  if (nb == 0) return B200_OK;   // an empty batch shard (shard.py)
  const int64_t cp = (c + 63) / 64 * 64;
  ConvGeo g;
  if (!conv_geo(g, out_strides, nb, cp, hp, wp, f, ho, wo, kh, kw, init, init_value))
    return B200_EUNSUPPORTED;
  const int R = conv_merge(f, kw);
  // dense planes read as [N][C][H * W] f32: unit pixel stride, rows back to
  // back, 16-byte channel / image strides and base (TMA)
  if (R == 1 || in_strides[3] != 1 || in_strides[2] != wp || in_strides[1] % 4 ||
      in_strides[0] % 4 || (reinterpret_cast<uintptr_t>(in) & 15) || hp * wp >= (int64_t(1) << 31))
    return B200_EUNSUPPORTED;
  // one TMA box per raw chunk over row pairs ([N][C][H / 2][2 W]): H and W
  // even (pair pitch 8 W bytes), box starts (w0, h0 / 2) on 16-byte
  // boundaries (a misaligned TMA box start faults — measured, "illegal
  // instruction"): tile origins are (4 h, 28 w), so 16 | 112 and h0 is even
  g.c = (int)c;
  g.blen = (int)(2 * wp);   // whole row pairs: a band's tiles share the chunk
  g.npair = (g.ph + 1) / 2;
  if (hp % 2 || wp % 2 || g.blen > 256 || g.th % 2 || g.cblocks != 1 || g.tw_tiles > 2)
    return B200_EUNSUPPORTED;
  g.raw_bytes = kRawCh * g.npair * g.blen * 4;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the CTA-pair variant (opt-in, B200_CONV_PAIR=1) needs both column tiles
  // of every band.  Measured at N = 256: 217 us against 160 for one CTA per
  // band — the freed shared memory buys a third patch stage, but the pair's
  // MMA couples the two CTAs' epilogues (the leader waits for the slower
  // one's TMEM release: 116 of 183 kcycles) and their output-block loads
  // queue behind each other (epilogue wait-out 105 vs 43 kcycles)
  const char *pe = getenv("B200_CONV_PAIR");
  const bool pair = g.tw_tiles == 2 && pe && pe[0] == '1';
  switch (f * 16 + R) {
    case 32 * 16 + 3:
      return pair ? launch_conv<32, 3, true, true>(in, in_strides, wt, out, g, s)
                  : launch_conv<32, 3, true>(in, in_strides, wt, out, g, s);
    case 64 * 16 + 3:
      return pair ? launch_conv<64, 3, true, true>(in, in_strides, wt, out, g, s)
                  : launch_conv<64, 3, true>(in, in_strides, wt, out, g, s);
    default: return B200_EUNSUPPORTED;
  }
}

// dev: the mapped progress counters of the last B200_CONV_TRACE launch
extern "C" int *b200_conv_trace(void) { return b200_conv_trace_host; }
