// Tensor-core implicit-GEMM convolution (NCHW / FCHW, valid, stride 1) on sm_100a.
//
//   out[n, f, ho, wo] (+)= sum_{ci, ki, kj} in[n, ci, ho+ki, wo+kj] * w[f, ci, ki, kj]
//
// Replaces run_tape on the conv_2d_nchw_fchw nest (reference
// tests/kernels.py:50-64; the engine recognises it from
// the separable contraction's index maps) when the engine precision is bf16.
// GEMM view: M = output pixels, N = F, K = (ki, kj, ci-block of 64) — the
// tensor core accumulates in fp32, the only deviation from the reference's
// (ci, ki, kj)-ordered f32 chain being accumulation order and the bf16
// operand rounding (tolerance: DESIGN.md, tests/test_gpu_conv.py).
//
// Layout: the input is repacked once per call to NHWC bf16 with channels
// padded to Cp (a multiple of 64) — b200_pack_conv_input — so the A tile of
// one tap is a single 4-D TMA box {64 ch, 8 w, 16 h, 1 n}: 128 pixel rows of
// 128 bytes, 128B-swizzled, i.e. exactly the canonical K-major UMMA layout.
// Taps are coordinate shifts of that box (the nest's input is pre-padded, out
// of range rows are TMA zero-fill).  Weights ([F][KH][KW][Cp] bf16) stay
// resident in shared memory for the CTA's lifetime.
// Structure per CTA (persistent over 16x8-pixel output tiles):
//   warp 0  TMA producer (weights once, then one A box per k-block, 5 stages)
//   warp 1  MMA issuer: UMMA 128 x F x 16, 4 per k-block, fp32 in TMEM
//   warp 2  TMEM allocator (2 accumulator buffers of F columns)
//   warps 4-7 epilogue: thread = pixel row; TMEM -> +out tile (TMA-loaded
//           into smem as [f][h][w] fp32) -> TMA store back to NCHW
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"
#include "tc_common.cuh"

using namespace b200tc;

namespace {

constexpr int TH = 16, TW = 8;            // output tile: 16 rows x 8 columns = 128 pixels
constexpr int ASTAGES = 5;
constexpr int A_STAGE = 128 * 128;        // 128 pixel rows x 64 bf16
constexpr int kThreads = 256;

struct ConvGeo {
  int64_t nb, cp, hp, wp, f, ho, wo, kh, kw;
  int64_t th_tiles, tw_tiles, tiles, kblocks;   // kblocks = kh*kw*(cp/64)
  int init;
  float init_value;
};

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

template <int F>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tma_in,
                   const __grid_constant__ CUtensorMap tma_w,
                   const __grid_constant__ CUtensorMap tma_out, ConvGeo g) {
  constexpr int B_KBLOCK = F * 128;          // F rows x 64 bf16
  constexpr int CBUF = F * 128 * 4;          // out tile [F][16][8] fp32
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const int kb_total = (int)g.kblocks;
  const uint32_t sB = base;                                   // kb_total x B_KBLOCK
  const uint32_t sA = base + kb_total * B_KBLOCK;             // ASTAGES x A_STAGE
  const uint32_t sC = sA + ASTAGES * A_STAGE;                 // 2 x CBUF
  unsigned char *gC = gbase + (sC - base);
  uint64_t *bars = reinterpret_cast<uint64_t *>(gC + 2 * CBUF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * ASTAGES + 7);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (ASTAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * ASTAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * ASTAGES + 2 + a); };
  auto cbar = [&](int b) { return bar0 + 8u * (2 * ASTAGES + 4 + b); };
  const uint32_t wbar = bar0 + 8u * (2 * ASTAGES + 6);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ASTAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 128);
      mbar_init(cbar(a), 1);
    }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * F < 32 ? 32 : 2 * F));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t per_img = g.th_tiles * g.tw_tiles;
  auto tile_coords = [&](int64_t t, int32_t &n, int32_t &h0, int32_t &w0) {
    n = (int32_t)(t / per_img);
    const int64_t r = t % per_img;
    h0 = (int32_t)((r / g.tw_tiles) * TH);
    w0 = (int32_t)((r % g.tw_tiles) * TW);
  };
  const int cblocks = (int)(g.cp / 64);

  if (warp == 0) {
    if (lane == 0) {
      // resident weights: every (tap, channel-block) K slice of B^T
      mbar_expect_tx(wbar, (uint32_t)(kb_total * B_KBLOCK));
      for (int kb = 0; kb < kb_total; ++kb)
        tma_load_2d(&tma_w, wbar, sB + kb * B_KBLOCK, kb * 64, 0);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
        int32_t n, h0, w0;
        tile_coords(t, n, h0, w0);
        for (int kb = 0; kb < kb_total; ++kb) {
          const int tap = kb / cblocks, cb = kb % cblocks;
          const int ki = (int)(tap / g.kw), kj = (int)(tap % g.kw);
          mbar_wait(empty(s), ph ^ 1);
          mbar_expect_tx(full(s), A_STAGE);
          tma_load_4d(&tma_in, full(s), sA + s * A_STAGE, cb * 64, w0 + kj, h0 + ki, n);
          if (++s == ASTAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(0, 128, F);
      mbar_wait(wbar, 0);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x) {
        mbar_wait(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * F);
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(full(s), ph);
          tc_fence_after();
          const uint32_t a_addr = sA + s * A_STAGE, b_addr = sB + kb * B_KBLOCK;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma<0, 1>(tmem_d, smem_desc(a_addr + 32 * k), smem_desc(b_addr + 32 * k), idesc,
                       (kb | k) != 0);
          umma_commit(empty(s));
          if (++s == ASTAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int r = threadIdx.x - 128;    // pixel row of the tile = TMEM lane
    const int q = warp - 4;
    const bool lead_t = r == 0;
    // out tile as [f][h][w] fp32 (TMA box order: w fastest, then h, then f)
    auto issue_load = [&](int64_t t, int b) {
      int32_t n, h0, w0;
      tile_coords(t, n, h0, w0);
      mbar_expect_tx(cbar(b), CBUF);
      tma_load_4d(&tma_out, cbar(b), sC + b * CBUF, w0, h0, 0, n);
    };
    int acc = 0;
    uint32_t aph = 0;
    int64_t it = 0;
    if (lead_t && !g.init && blockIdx.x < g.tiles) issue_load(blockIdx.x, 0);
    for (int64_t t = blockIdx.x; t < g.tiles; t += gridDim.x, ++it) {
      const int b = (int)(it & 1);
      int32_t n, h0, w0;
      tile_coords(t, n, h0, w0);
      // prefetch the next tile's out block into the other buffer once its
      // previous store has drained
      if (lead_t) {
        bulk_wait_read<0>();
        if (!g.init && t + gridDim.x < g.tiles) issue_load(t + gridDim.x, b ^ 1);
      }
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      if (!g.init) mbar_wait(cbar(b), (uint32_t)((it >> 1) & 1));
      else named_bar_sync(1, 128);   // buffer b is free (its store drained above)
      float *cb = reinterpret_cast<float *>(gC + b * CBUF);
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * F);
#pragma unroll 1
      for (int c0 = 0; c0 < F; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(trow + (uint32_t)c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float *p = cb + (c0 + j) * 128 + r;
          const float o = g.init ? g.init_value : *p;
          *p = o + __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty(acc));
      fence_proxy_async();
      named_bar_sync(1, 128);
      if (lead_t) {
        tma_store_4d(&tma_out, sC + b * CBUF, w0, h0, 0, n);
        bulk_commit();
      }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lead_t) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * F < 32 ? 32 : 2 * F));
  }
}

// NCHW f32 (any strides) -> NHWC bf16 with channels padded to cp (zeros).
// A CTA transposes one (n, h) row slab [cp][W] through shared memory per
// iteration, grid-striding over rows: each warp reads whole channel rows
// (coalesced along w), each thread then writes 8 channels of one pixel as a
// single 16-byte vector.
constexpr int PACK_MAXW = 256;
__global__ void __launch_bounds__(256) pack_nhwc_kernel(const float *__restrict__ src, int64_t sN,
                                                        int64_t sC, int64_t sH, int64_t sW,
                                                        __nv_bfloat16 *__restrict__ dst, int C,
                                                        int H, int W, int cp, int64_t rows) {
  extern __shared__ float slab[];   // [cp][W + 1]
  const int ld = W + 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int chunks = cp / 8;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t n = row / H, h = row % H;
    const float *base = src + n * sN + h * sH;
    for (int c = warp; c < cp; c += 8) {
      const float *p = base + (int64_t)c * sC;
      for (int w = lane; w < W; w += 32) slab[c * ld + w] = c < C ? __ldg(p + w * sW) : 0.f;
    }
    __syncthreads();
    uint4 *out = reinterpret_cast<uint4 *>(dst + row * (int64_t)W * cp);
    for (int i = threadIdx.x; i < W * chunks; i += 256) {
      const int w = i / chunks, c0 = (i % chunks) * 8;
      __nv_bfloat162 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[j] = __floats2bfloat162_rn(slab[(c0 + 2 * j) * ld + w], slab[(c0 + 2 * j + 1) * ld + w]);
      out[i] = *reinterpret_cast<uint4 *>(v);
    }
    __syncthreads();
  }
}

// FCHW f32 weights -> [F][KH][KW][cp] bf16 (K order: tap, channel).
__global__ void pack_wt_kernel(const float *__restrict__ src, int64_t sF, int64_t sC,
                               int64_t sKH, int64_t sKW, __nv_bfloat16 *__restrict__ dst,
                               int64_t F, int64_t C, int64_t KH, int64_t KW, int64_t cp) {
  const int64_t total = F * KH * KW * cp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % cp, tap = (i / cp) % (KH * KW), f = i / (cp * KH * KW);
    const int64_t ki = tap / KW, kj = tap % KW;
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

template <int F>
int launch_conv(const void *in_nhwc, const void *wt, float *out, const int64_t *ostr,
                const ConvGeo &g, cudaStream_t s) {
  CUtensorMap mi, mw, mo;
  cuuint64_t di[4] = {(cuuint64_t)g.cp, (cuuint64_t)g.wp, (cuuint64_t)g.hp, (cuuint64_t)g.nb};
  cuuint64_t si[3] = {(cuuint64_t)(g.cp * 2), (cuuint64_t)(g.wp * g.cp * 2),
                      (cuuint64_t)(g.hp * g.wp * g.cp * 2)};
  cuuint32_t bi[4] = {64, TW, TH, 1};
  if (!make_map_4d(&mi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in_nhwc, di, si, bi,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return B200_ELAUNCH;
  if (!make_map(&mw, 0, wt, F, g.kh * g.kw * g.cp, F)) return B200_ELAUNCH;
  // out: NCHW f32 with element strides ostr = {n, f, h, w} (w must be 1)
  cuuint64_t dout[4] = {(cuuint64_t)g.wo, (cuuint64_t)g.ho, (cuuint64_t)F, (cuuint64_t)g.nb};
  cuuint64_t sout[3] = {(cuuint64_t)(ostr[2] * 4), (cuuint64_t)(ostr[1] * 4),
                        (cuuint64_t)(ostr[0] * 4)};
  cuuint32_t bout[4] = {TW, TH, F, 1};
  if (!make_map_4d(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, dout, sout, bout,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
    return B200_ELAUNCH;
  const size_t smem = 1024 + g.kblocks * F * 128 + ASTAGES * A_STAGE + 2 * F * 128 * 4 + 256;
  if (smem > 232448) return B200_EUNSUPPORTED;
  int ctas = num_sms();
  if (g.tiles < ctas) ctas = (int)g.tiles;
  cudaFuncSetAttribute(conv_tc_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  conv_tc_kernel<F><<<ctas, kThreads, smem, s>>>(mi, mw, mo, g);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace

extern "C" int b200_pack_conv_input(const float *src, const int64_t *sstr, void *dst, int64_t nb,
                                    int64_t c, int64_t h, int64_t w, int64_t cp, void *stream) {
  if (nb <= 0 || h <= 0 || w <= 0 || cp < c || cp % 64 || w > PACK_MAXW) return B200_EINVAL;
  const size_t smem = (size_t)cp * (w + 1) * 4;
  if (smem > 227 * 1024) return B200_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(pack_nhwc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int64_t rows = nb * h;
  const int per_sm = (int)((228 * 1024) / (smem + 1024));
  int64_t blocks = (int64_t)num_sms() * (per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm));
  if (blocks > rows) blocks = rows;
  pack_nhwc_kernel<<<(unsigned)blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      src, sstr[0], sstr[1], sstr[2], sstr[3], static_cast<__nv_bfloat16 *>(dst), (int)c, (int)h,
      (int)w, (int)cp, rows);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

extern "C" int b200_pack_conv_weight(const float *src, const int64_t *sstr, void *dst, int64_t f,
                                     int64_t c, int64_t kh, int64_t kw, int64_t cp,
                                     void *stream) {
  const int64_t total = f * kh * kw * cp;
  if (total <= 0 || cp % 64) return B200_EINVAL;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  pack_wt_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, sstr[0], sstr[1], sstr[2], sstr[3], static_cast<__nv_bfloat16 *>(dst), f, c, kh, kw,
      cp);
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

extern "C" int b200_conv2d_tc(const void *in_nhwc, const void *wt, float *out,
                              const int64_t *out_strides, int64_t nb, int64_t cp, int64_t hp,
                              int64_t wp, int64_t f, int64_t ho, int64_t wo, int64_t kh,
                              int64_t kw, int32_t init, float init_value, void *stream) {
  if (out_strides[3] != 1 || cp % 64 || ho + kh - 1 > hp || wo + kw - 1 > wp)
    return B200_EINVAL;
  ConvGeo g{nb, cp, hp, wp, f, ho, wo, kh, kw, 0, 0, 0, 0, init, init_value};
  g.th_tiles = (ho + TH - 1) / TH;
  g.tw_tiles = (wo + TW - 1) / TW;
  g.tiles = nb * g.th_tiles * g.tw_tiles;
  g.kblocks = kh * kw * (cp / 64);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (f) {
    case 32: return launch_conv<32>(in_nhwc, wt, out, out_strides, g, s);
    case 64: return launch_conv<64>(in_nhwc, wt, out, out_strides, g, s);
    case 128: return launch_conv<128>(in_nhwc, wt, out, out_strides, g, s);
    default: return B200_EUNSUPPORTED;
  }
}
