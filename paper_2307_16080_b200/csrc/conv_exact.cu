// Bit-exact direct convolution (NCHW / FCHW, valid, stride 1) on the FP32 /
// FP64 pipes of sm_100a.
//
//   out[n, f, ho, wo] = out (or init) + sum over ci, ki, kj (nest order) of
//                       round(in[n, ci, ho+ki, wo+kj] * w[f, ci, ki, kj])
//
// Replaces run_tape on the conv_2d_nchw_fchw nest (reference
// tests/kernels.py:50-64) at the exact precision: every product and every
// partial sum is one IEEE op (__fmul_rn / __fadd_rn, never contracted), and
// each output's chain runs ci -> ki -> kj exactly as the reference does
// (interp/_evalpy.py:115-127), so results are bit-identical.  The generic
// table-addressed contraction (gemm_exact.cu) computes the same thing; this
// kernel exists for speed: the conv's operands are re-read KH*KW times, so it
// stages them once per CTA in shared memory instead of gathering through
// offset tables.
//
// CTA tile: 8 output rows x 32 columns x 64 filters.  Warp w owns filters
// [8w, 8w + 8) (its weights are warp-uniform: 16-byte broadcast reads);
// lane l owns rows l / 8 and l / 8 + 4 and columns l % 8 + 8 i (i < 4), so a
// warp's input reads are 4 rows x 8 consecutive pixels — with the patch row
// pitch padded to 8 mod 32 words they hit 32 distinct banks.  Each thread
// keeps 8 pixels x 8 filters of accumulators: 10 shared-memory reads per
// 128 FP32 ops.  Channels are staged 8 at a time (input patch
// [8][8 + KH - 1][pitch], weights [8][KH * KW][64], weights pre-transposed
// to [C][KH * KW][F]) by cp.async into a double buffer, so the next chunk's
// loads overlap this chunk's arithmetic.  Measured (N=256 C=F=64 56² 3×3,
// f32): 21.3 TFLOP/s = 57 % of the 37.2 TFLOP/s no-FMA ceiling (separate,
// individually rounded multiply and add per MAC), vs 13.7 through the
// generic table-addressed kernel.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "../../include/b200k.h"
#include "tc_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int TH = 8, TW = 32;     // output rows x columns per CTA
constexpr int FT = 64, FX = 8;     // filters per CTA / per thread
constexpr int PX = 8;              // output pixels per thread: rows r, r + 4 x 4 columns
constexpr int CC = 8;              // channels per staged chunk

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__device__ __forceinline__ void cp_async(T *dst, const T *src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  // src-size 0 zero-fills the destination (out-of-range patch elements)
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src),
               "n"(sizeof(T)), "r"(valid ? (int)sizeof(T) : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T>
struct ConvArgs {
  const T *in, *w;               // w: the [C][KH * KW][F] transpose (f fastest)
  T *out;
  int64_t si[4], so[4];          // element strides n, c, h, w / n, f, h, w
  int nb, c, hp, wp, f, ho, wo, kh, kw;
  int pitch;                     // patch row pitch (elements)
  int th_tiles, tw_tiles;
  int init;
  T init_value;
};

// KHC / KWC: compile-time filter extent (0 = runtime g.kh / g.kw); the 3x3
// instantiation unrolls the tap loops so shared-memory offsets are
// immediates and the FP pipe is not diluted by loop and address work.
template <typename T, int KHC, int KWC>
__global__ void __launch_bounds__(kThreads) conv_exact_kernel(ConvArgs<T> g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int KH = KHC ? KHC : g.kh, KW = KWC ? KWC : g.kw;
  const int ph = TH + KH - 1;
  const int taps = KH * KW;
  const int in_elems = CC * ph * g.pitch;
  const int w_elems = CC * taps * FT;
  T *in_s = reinterpret_cast<T *>(smem_raw);          // [2][CC][ph][pitch]
  T *w_s = in_s + 2 * in_elems;                       // [2][CC][taps][FT]

  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int r = lane / 8, wl = lane % 8;
  int tile = blockIdx.x;
  const int tw_i = tile % g.tw_tiles;
  tile /= g.tw_tiles;
  const int th_i = tile % g.th_tiles;
  const int n = tile / g.th_tiles;
  const int h0 = th_i * TH, w0 = tw_i * TW;
  const int f0 = blockIdx.y * FT;
  const int fw = f0 + warp * FX;                      // this thread's first filter

  const T *in_n = g.in + (int64_t)n * g.si[0];
  // stage channels [c0, c0 + CC) into buffer b
  auto stage = [&](int c0, int b) {
    T *is = in_s + b * in_elems;
    const int pw = TW + g.kw - 1;
    for (int e = t; e < CC * ph * pw; e += kThreads) {
      const int cc = e / (ph * pw), rem = e - cc * (ph * pw);
      const int y = rem / pw, x = rem - y * pw;
      const int ci = c0 + cc, hy = h0 + y, wx = w0 + x;
      const bool ok = ci < g.c && hy < g.hp && wx < g.wp;
      const T *src = ok ? in_n + ci * g.si[1] + hy * g.si[2] + wx * g.si[3] : g.in;
      cp_async(is + (cc * ph + y) * g.pitch + x, src, ok);
    }
    T *ws = w_s + b * w_elems;
    for (int e = t; e < CC * taps * FT; e += kThreads) {
      const int fi = e % FT, ct = e / FT;   // ct = cc * taps + tap
      const int ff = f0 + fi;
      const bool ok = c0 * taps + ct < g.c * taps && ff < g.f;
      const T *src = ok ? g.w + ((int64_t)c0 * taps + ct) * g.f + ff : g.w;
      cp_async(ws + e, src, ok);
    }
    cp_commit();
  };

  // accumulators start from the output (out += conv) or the fused init value
  T acc[PX][FX];
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int ho = h0 + r + 4 * (i / 4), wo = w0 + wl + 8 * (i % 4);
#pragma unroll
    for (int j = 0; j < FX; ++j) {
      const int ff = fw + j;
      T v = g.init_value;
      if (!g.init && ho < g.ho && wo < g.wo && ff < g.f)
        v = g.out[(int64_t)n * g.so[0] + ff * g.so[1] + ho * g.so[2] + wo * g.so[3]];
      acc[i][j] = v;
    }
  }

  const int chunks = (g.c + CC - 1) / CC;
  stage(0, 0);
  for (int k = 0; k < chunks; ++k) {
    const int b = k & 1;
    if (k + 1 < chunks) {
      stage((k + 1) * CC, b ^ 1);   // buffer b^1 was last read before the barrier below
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const T *is = in_s + b * in_elems + r * g.pitch + wl;
    const T *ws = w_s + b * w_elems + warp * FX;
    const int cn = min(CC, g.c - k * CC);
    for (int cc = 0; cc < cn; ++cc) {
#pragma unroll
      for (int ki = 0; ki < KH; ++ki) {
        const T *irow = is + (cc * ph + ki) * g.pitch;
        const T *wrow = ws + (cc * taps + ki * KW) * FT;
#pragma unroll
        for (int kj = 0; kj < KW; ++kj) {
          T x[PX], wv[FX];
#pragma unroll
          for (int i = 0; i < PX; ++i) x[i] = irow[(i / 4) * 4 * g.pitch + kj + 8 * (i % 4)];
#pragma unroll
          for (int j = 0; j < FX; ++j) wv[j] = wrow[kj * FT + j];
#pragma unroll
          for (int i = 0; i < PX; ++i)
#pragma unroll
            for (int j = 0; j < FX; ++j) acc[i][j] = add_rn(acc[i][j], mul_rn(x[i], wv[j]));
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int ho = h0 + r + 4 * (i / 4), wo = w0 + wl + 8 * (i % 4);
    if (ho >= g.ho || wo >= g.wo) continue;
#pragma unroll
    for (int j = 0; j < FX; ++j) {
      const int ff = fw + j;
      if (ff < g.f) g.out[(int64_t)n * g.so[0] + ff * g.so[1] + ho * g.so[2] + wo * g.so[3]] =
          acc[i][j];
    }
  }
}

// Compile-time KH x KW (KW <= 5) variant, the one the 3x3 conv runs.  Same
// CTA tile, chain order and staging scheme as conv_exact_kernel, but lane l
// owns rows l / 8 and l / 8 + 4 and the 4 CONSECUTIVE columns 4 (l % 8) ..
// +3: per (channel, filter row) a thread reads its 2 x (4 + KW - 1) inputs
// once as 16-byte vectors (a quarter warp reads one 128-byte patch row:
// conflict-free) and reuses them for all KW taps, so the shared-memory reads
// per 128 FP32 ops drop from 10 to ~3.  Channel chunks are staged with
// vector cp.async (input pairs, weight quads) when the layout allows, and
// float outputs are read / written as 16-byte vectors.
constexpr int RPITCH = TW + 8;   // patch row pitch: 4 (l % 8) + 8 <= pitch

template <typename T, int KH, int KW>
__global__ void __launch_bounds__(kThreads) conv_rows_kernel(ConvArgs<T> g, int vec_in,
                                                             int vec_w, int vec_out) {
  static_assert(KW <= 5, "input run of 4 + KW - 1 values must fit two 4-vectors");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PH = TH + KH - 1, PW = TW + KW - 1, TAPS = KH * KW;
  constexpr int IN_ELEMS = CC * PH * RPITCH;
  constexpr int W_ELEMS = CC * TAPS * FT;
  constexpr int RUN = 4 + KW - 1;
  T *in_s = reinterpret_cast<T *>(smem_raw);          // [2][CC][PH][RPITCH]
  T *w_s = in_s + 2 * IN_ELEMS;                       // [2][CC][TAPS][FT]

  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int r = lane / 8, cg = lane % 8;
  int tile = blockIdx.x;
  const int tw_i = tile % g.tw_tiles;
  tile /= g.tw_tiles;
  const int th_i = tile % g.th_tiles;
  const int n = tile / g.th_tiles;
  const int h0 = th_i * TH, w0 = tw_i * TW;
  const int f0 = blockIdx.y * FT;
  const int fw = f0 + warp * FX;

  const T *in_n = g.in + (int64_t)n * g.si[0];
  auto stage = [&](int c0, int b) {
    T *is = in_s + b * IN_ELEMS;
    if (vec_in) {   // pairs: unit column stride, even strides, aligned base
      constexpr int PV = (PW + 1) / 2;
      for (int e = t; e < CC * PH * PV; e += kThreads) {
        const int cc = e / (PH * PV), rem = e - cc * (PH * PV);
        const int y = rem / PV, x = 2 * (rem - y * PV);
        const int ci = c0 + cc, hy = h0 + y, wx = w0 + x;
        const int avail = (ci < g.c && hy < g.hp && wx < g.wp) ? min(2, g.wp - wx) : 0;
        const T *src = avail ? in_n + ci * g.si[1] + hy * g.si[2] + wx : g.in;
        const uint32_t d =
            static_cast<uint32_t>(__cvta_generic_to_shared(is + (cc * PH + y) * RPITCH + x));
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src),
                     "n"(2 * sizeof(T)), "r"(avail * (int)sizeof(T))
                     : "memory");
      }
    } else {
      for (int e = t; e < CC * PH * PW; e += kThreads) {
        const int cc = e / (PH * PW), rem = e - cc * (PH * PW);
        const int y = rem / PW, x = rem - y * PW;
        const int ci = c0 + cc, hy = h0 + y, wx = w0 + x;
        const bool ok = ci < g.c && hy < g.hp && wx < g.wp;
        const T *src = ok ? in_n + ci * g.si[1] + hy * g.si[2] + wx * g.si[3] : g.in;
        cp_async(is + (cc * PH + y) * RPITCH + x, src, ok);
      }
    }
    T *ws = w_s + b * W_ELEMS;
    if (vec_w) {    // 16-byte groups of filters (F a multiple of the group)
      constexpr int WV = 16 / sizeof(T);
      for (int e = t; e < W_ELEMS / WV; e += kThreads) {
        const int fi = (e % (FT / WV)) * WV, ct = e / (FT / WV);
        const int ff = f0 + fi;
        const bool ok = c0 * TAPS + ct < g.c * TAPS && ff < g.f;
        const T *src = ok ? g.w + ((int64_t)c0 * TAPS + ct) * g.f + ff : g.w;
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(ws + ct * FT + fi));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                     "r"(ok ? 16 : 0)
                     : "memory");
      }
    } else {
      for (int e = t; e < W_ELEMS; e += kThreads) {
        const int fi = e % FT, ct = e / FT;
        const int ff = f0 + fi;
        const bool ok = c0 * TAPS + ct < g.c * TAPS && ff < g.f;
        const T *src = ok ? g.w + ((int64_t)c0 * TAPS + ct) * g.f + ff : g.w;
        cp_async(ws + e, src, ok);
      }
    }
    cp_commit();
  };

  // pixel i: row h0 + r + 4 (i / 4), column w0 + 4 cg + i % 4
  T acc[PX][FX];
  const int wo0 = w0 + 4 * cg;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ho = h0 + r + 4 * q;
#pragma unroll
    for (int j = 0; j < FX; ++j) {
      const int ff = fw + j;
      T *o = g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
      if (!g.init && vec_out && ho < g.ho && wo0 + 3 < g.wo && ff < g.f) {
        const float4 v = *reinterpret_cast<const float4 *>(o + wo0);
        acc[4 * q][j] = v.x, acc[4 * q + 1][j] = v.y, acc[4 * q + 2][j] = v.z,
        acc[4 * q + 3][j] = v.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int wo = wo0 + u;
          acc[4 * q + u][j] = (!g.init && ho < g.ho && wo < g.wo && ff < g.f)
                                  ? o[(int64_t)wo * g.so[3]] : g.init_value;
        }
      }
    }
  }

  const int chunks = (g.c + CC - 1) / CC;
  stage(0, 0);
  for (int k = 0; k < chunks; ++k) {
    const int b = k & 1;
    if (k + 1 < chunks) {
      stage((k + 1) * CC, b ^ 1);   // buffer b^1 was last read before the barrier below
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const T *is = in_s + b * IN_ELEMS + r * RPITCH + 4 * cg;
    const T *ws = w_s + b * W_ELEMS + warp * FX;
    const int cn = min(CC, g.c - k * CC);
    for (int cc = 0; cc < cn; ++cc) {
#pragma unroll
      for (int ki = 0; ki < KH; ++ki) {
        T x[2][8];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const T *row = is + (cc * PH + ki + 4 * q) * RPITCH;
#pragma unroll
          for (int u = 0; u < RUN; ++u) x[q][u] = row[u];
        }
        const T *wrow = ws + (cc * TAPS + ki * KW) * FT;
#pragma unroll
        for (int kj = 0; kj < KW; ++kj) {
          T wv[FX];
#pragma unroll
          for (int j = 0; j < FX; ++j) wv[j] = wrow[kj * FT + j];
#pragma unroll
          for (int i = 0; i < PX; ++i)
#pragma unroll
            for (int j = 0; j < FX; ++j)
              acc[i][j] = add_rn(acc[i][j], mul_rn(x[i / 4][i % 4 + kj], wv[j]));
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ho = h0 + r + 4 * q;
    if (ho >= g.ho) continue;
#pragma unroll
    for (int j = 0; j < FX; ++j) {
      const int ff = fw + j;
      if (ff >= g.f) continue;
      T *o = g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
      if (vec_out && wo0 + 3 < g.wo) {
        *reinterpret_cast<float4 *>(o + wo0) =
            make_float4(acc[4 * q][j], acc[4 * q + 1][j], acc[4 * q + 2][j], acc[4 * q + 3][j]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (wo0 + u < g.wo) o[(int64_t)(wo0 + u) * g.so[3]] = acc[4 * q + u][j];
      }
    }
  }
}

// Width-matched variant for output widths that are multiples of 8 * PXW
// (ResNet's 56 = 8 x 7): lane l owns ONE row (l / 8) and PXW consecutive
// columns PXW (l % 8) .. + PXW - 1, so a CTA tile is 4 rows x 8 PXW columns x
// 64 filters with no idle columns (the 32-wide tiles of conv_rows_kernel
// leave 8 of every 64 columns idle at width 56).  Its input run of
// PXW + KW - 1 values per (channel, filter row) is read with scalar loads: at
// a row pitch of 8 (mod 32) the 4 rows x 8 runs (stride PXW, odd) of a warp
// hit 32 distinct banks.
constexpr int PTH = 4;           // rows per CTA

template <typename T, int KH, int KW, int PXW>
__global__ void __launch_bounds__(kThreads) conv_runs_kernel(ConvArgs<T> g, int vec_in,
                                                             int vec_w) {
  constexpr int TWR = 8 * PXW;
  constexpr int PH = PTH + KH - 1, PW = TWR + KW - 1, TAPS = KH * KW;
  constexpr int PITCH = PW + ((8 - PW) % 32 + 32) % 32;
  constexpr int IN_ELEMS = CC * PH * PITCH;
  constexpr int W_ELEMS = CC * TAPS * FT;
  constexpr int RUN = PXW + KW - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *in_s = reinterpret_cast<T *>(smem_raw);          // [2][CC][PH][PITCH]
  T *w_s = in_s + 2 * IN_ELEMS;                       // [2][CC][TAPS][FT]

  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int r = lane / 8, cg = lane % 8;
  int tile = blockIdx.x;
  const int tw_i = tile % g.tw_tiles;
  tile /= g.tw_tiles;
  const int th_i = tile % g.th_tiles;
  const int n = tile / g.th_tiles;
  const int h0 = th_i * PTH, w0 = tw_i * TWR;
  const int f0 = blockIdx.y * FT;
  const int fw = f0 + warp * FX;

  const T *in_n = g.in + (int64_t)n * g.si[0];
  auto stage = [&](int c0, int b) {
    T *is = in_s + b * IN_ELEMS;
    if (vec_in) {
      constexpr int PV = (PW + 1) / 2;
      for (int e = t; e < CC * PH * PV; e += kThreads) {
        const int cc = e / (PH * PV), rem = e - cc * (PH * PV);
        const int y = rem / PV, x = 2 * (rem - y * PV);
        const int ci = c0 + cc, hy = h0 + y, wx = w0 + x;
        const int avail = (ci < g.c && hy < g.hp && wx < g.wp) ? min(2, g.wp - wx) : 0;
        const T *src = avail ? in_n + ci * g.si[1] + hy * g.si[2] + wx : g.in;
        const uint32_t d =
            static_cast<uint32_t>(__cvta_generic_to_shared(is + (cc * PH + y) * PITCH + x));
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src),
                     "n"(2 * sizeof(T)), "r"(avail * (int)sizeof(T))
                     : "memory");
      }
    } else {
      for (int e = t; e < CC * PH * PW; e += kThreads) {
        const int cc = e / (PH * PW), rem = e - cc * (PH * PW);
        const int y = rem / PW, x = rem - y * PW;
        const int ci = c0 + cc, hy = h0 + y, wx = w0 + x;
        const bool ok = ci < g.c && hy < g.hp && wx < g.wp;
        const T *src = ok ? in_n + ci * g.si[1] + hy * g.si[2] + wx * g.si[3] : g.in;
        cp_async(is + (cc * PH + y) * PITCH + x, src, ok);
      }
    }
    T *ws = w_s + b * W_ELEMS;
    if (vec_w) {
      constexpr int WV = 16 / sizeof(T);
      for (int e = t; e < W_ELEMS / WV; e += kThreads) {
        const int fi = (e % (FT / WV)) * WV, ct = e / (FT / WV);
        const int ff = f0 + fi;
        const bool ok = c0 * TAPS + ct < g.c * TAPS && ff < g.f;
        const T *src = ok ? g.w + ((int64_t)c0 * TAPS + ct) * g.f + ff : g.w;
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(ws + ct * FT + fi));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                     "r"(ok ? 16 : 0)
                     : "memory");
      }
    } else {
      for (int e = t; e < W_ELEMS; e += kThreads) {
        const int fi = e % FT, ct = e / FT;
        const int ff = f0 + fi;
        const bool ok = c0 * TAPS + ct < g.c * TAPS && ff < g.f;
        const T *src = ok ? g.w + ((int64_t)c0 * TAPS + ct) * g.f + ff : g.w;
        cp_async(ws + e, src, ok);
      }
    }
    cp_commit();
  };

  // pixel u: row h0 + r, column w0 + PXW cg + u
  T acc[PXW][FX];
  const int ho = h0 + r, wo0 = w0 + PXW * cg;
#pragma unroll
  for (int j = 0; j < FX; ++j) {
    const int ff = fw + j;
    const T *o = g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
#pragma unroll
    for (int u = 0; u < PXW; ++u) {
      const int wo = wo0 + u;
      acc[u][j] = (!g.init && ho < g.ho && wo < g.wo && ff < g.f) ? o[(int64_t)wo * g.so[3]]
                                                                  : g.init_value;
    }
  }

  const int chunks = (g.c + CC - 1) / CC;
  stage(0, 0);
  for (int k = 0; k < chunks; ++k) {
    const int b = k & 1;
    if (k + 1 < chunks) {
      stage((k + 1) * CC, b ^ 1);   // buffer b^1 was last read before the barrier below
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const T *is = in_s + b * IN_ELEMS + r * PITCH + PXW * cg;
    const T *ws = w_s + b * W_ELEMS + warp * FX;
    const int cn = min(CC, g.c - k * CC);
    for (int cc = 0; cc < cn; ++cc) {
#pragma unroll
      for (int ki = 0; ki < KH; ++ki) {
        T x[RUN];
        const T *row = is + (cc * PH + ki) * PITCH;
#pragma unroll
        for (int u = 0; u < RUN; ++u) x[u] = row[u];
        const T *wrow = ws + (cc * TAPS + ki * KW) * FT;
#pragma unroll
        for (int kj = 0; kj < KW; ++kj) {
          T wv[FX];
#pragma unroll
          for (int j = 0; j < FX; ++j) wv[j] = wrow[kj * FT + j];
#pragma unroll
          for (int u = 0; u < PXW; ++u)
#pragma unroll
            for (int j = 0; j < FX; ++j) acc[u][j] = add_rn(acc[u][j], mul_rn(x[u + kj], wv[j]));
        }
      }
    }
    __syncthreads();
  }

  if (ho >= g.ho) return;
#pragma unroll
  for (int j = 0; j < FX; ++j) {
    const int ff = fw + j;
    if (ff >= g.f) continue;
    T *o = g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
#pragma unroll
    for (int u = 0; u < PXW; ++u)
      if (wo0 + u < g.wo) o[(int64_t)(wo0 + u) * g.so[3]] = acc[u][j];
  }
}

// TMA-fed runs kernel (f32, 3x3; the default where its tensor maps apply,
// B200_CONV_EXACT_TMA=0 selects conv_runs_kernel): the same tile, lane
// mapping and arithmetic, staged differently — each 8-channel chunk is two
// TMA boxes issued by thread 0 (the input as whole row pairs of the
// [N][C][H/2][2W] view: single rows of W floats are not 16-byte multiples;
// the transposed weights as [8 x 9][64]) into a 3-stage ring tracked by
// mbarriers.  No per-element copy addressing (division by the patch
// geometry per element in conv_runs_kernel's staging) and no CTA-wide
// barrier: a warp waits only for the chunk it reads, thread 0 refills a
// stage once all eight warps released it.  The patch row pitch is W (rows of
// a pair are back to back), so the ring holds full rows.
constexpr int TSTG = 3;

template <int PXW>
__global__ void __launch_bounds__(kThreads) conv_runs_tma_kernel(
    const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tw,
    ConvArgs<float> g) {
  using namespace b200tc;
  constexpr int KH = 3, KW = 3, TAPS = 9, TWR = 8 * PXW, RUN = PXW + KW - 1;
  constexpr int PH = PTH + KH - 1;                 // 6 rows = 3 pairs
  constexpr int W_ELEMS = CC * TAPS * FT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char *gbase = smem_raw + (base - smem_u32(smem_raw));
  const int W = g.wp;
  const int in_elems = CC * PH * W;                // [CC][3 pairs][2W]
  const uint32_t in_bytes = (uint32_t)in_elems * 4u;
  const uint32_t in_stage = (in_bytes + 127u) & ~127u;
  const float *in_s = reinterpret_cast<const float *>(gbase);
  const float *w_s = reinterpret_cast<const float *>(gbase + TSTG * in_stage);
  const uint32_t sIn = base, sW = base + TSTG * in_stage;
  uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + TSTG * (in_stage + W_ELEMS * 4));
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int st) { return bar0 + 8u * st; };
  auto empty = [&](int st) { return bar0 + 8u * (TSTG + st); };

  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int r = lane / 8, cg = lane % 8;
  int tile = blockIdx.x;
  const int tw_i = tile % g.tw_tiles;
  tile /= g.tw_tiles;
  const int th_i = tile % g.th_tiles;
  const int n = tile / g.th_tiles;
  const int h0 = th_i * PTH, w0 = tw_i * TWR;
  const int f0 = blockIdx.y * FT;
  const int fw = f0 + warp * FX;
  const int chunks = (g.c + CC - 1) / CC;
  auto issue = [&](int k) {
    const int st = k % TSTG;
    mbar_expect_tx(full(st), in_bytes + (uint32_t)W_ELEMS * 4u);
    // input: pairs h0 / 2 .. + 2 of channels k CC .. + CC - 1 (zero past C / H)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(sIn + st * in_stage),
        "l"(reinterpret_cast<uint64_t>(&tin)), "r"(full(st)), "r"(0), "r"(h0 / 2),
        "r"(k * CC), "r"(n)
        : "memory");
    tma_load_2d(&tw, full(st), sW + st * (uint32_t)(W_ELEMS * 4), f0, k * CC * TAPS);
  };
  if (t == 0) {
    for (int st = 0; st < TSTG; ++st) {
      mbar_init(full(st), 1);
      mbar_init(empty(st), kThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int k = 0; k < TSTG && k < chunks; ++k) issue(k);

  float acc[PXW][FX];
  const int ho = h0 + r, wo0 = w0 + PXW * cg;
#pragma unroll
  for (int j = 0; j < FX; ++j) {
    const int ff = fw + j;
    const float *o =
        g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
#pragma unroll
    for (int u = 0; u < PXW; ++u) {
      const int wo = wo0 + u;
      acc[u][j] = (!g.init && ho < g.ho && wo < g.wo && ff < g.f) ? o[(int64_t)wo * g.so[3]]
                                                                  : g.init_value;
    }
  }

  // stage / phase counters; thread 0 refills the stage every warp released
  // one chunk earlier (as in gemm_exact_tma_kernel), so warp 0 runs up to a
  // chunk ahead of the slowest warp instead of stalling on it
  int st = 0, pst = TSTG - 1;
  uint32_t ph = 0, pph = 1;
  for (int k = 0; k < chunks; ++k) {
    if (t == 0 && k > 0 && k - 1 + TSTG < chunks) {
      mbar_wait(empty(pst), pph);
      issue(k - 1 + TSTG);
    }
    mbar_wait(full(st), ph);
    const float *is = in_s + st * (in_stage / 4) + r * W + w0 + PXW * cg;
    const float *ws = w_s + st * W_ELEMS + warp * FX;
    const int cn = min(CC, g.c - k * CC);
    for (int cc = 0; cc < cn; ++cc) {
#pragma unroll
      for (int ki = 0; ki < KH; ++ki) {
        float x[RUN];
        const float *row = is + (cc * PH + ki) * W;
#pragma unroll
        for (int u = 0; u < RUN; ++u) x[u] = row[u];
        const float *wrow = ws + (cc * TAPS + ki * KW) * FT;
#pragma unroll
        for (int kj = 0; kj < KW; ++kj) {
          float wv[FX];
#pragma unroll
          for (int j = 0; j < FX; ++j) wv[j] = wrow[kj * FT + j];
#pragma unroll
          for (int u = 0; u < PXW; ++u)
#pragma unroll
            for (int j = 0; j < FX; ++j)
              acc[u][j] = __fadd_rn(acc[u][j], __fmul_rn(x[u + kj], wv[j]));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty(st));
    pst = st;
    pph = ph;
    if (++st == TSTG) { st = 0; ph ^= 1; }
  }

  if (ho >= g.ho) return;
#pragma unroll
  for (int j = 0; j < FX; ++j) {
    const int ff = fw + j;
    if (ff >= g.f) continue;
    float *o = g.out + (int64_t)n * g.so[0] + (int64_t)ff * g.so[1] + (int64_t)ho * g.so[2];
#pragma unroll
    for (int u = 0; u < PXW; ++u)
      if (wo0 + u < g.wo) o[(int64_t)(wo0 + u) * g.so[3]] = acc[u][j];
  }
}

// The runs-TMA kernel's tensor maps, or false where they do not apply
// (dense even-sized planes with 16-byte strides, rows of <= 128 floats, F a
// multiple of 4, 16-byte aligned bases).
bool runs_tma_maps(CUtensorMap *tin, CUtensorMap *tw, const float *in, const int64_t *si,
                   const float *wt, int64_t nb, int64_t c, int64_t hp, int64_t wp, int64_t f) {
  using namespace b200tc;
  if (si[3] != 1 || si[2] != wp || wp % 2 || hp % 2 || 2 * wp > 256 || si[1] % 4 ||
      si[0] % 4 || f % 4 || (reinterpret_cast<uintptr_t>(in) & 15) ||
      (reinterpret_cast<uintptr_t>(wt) & 15))
    return false;
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  const cuuint64_t di[4] = {(cuuint64_t)(2 * wp), (cuuint64_t)(hp / 2), (cuuint64_t)c,
                            (cuuint64_t)nb};
  const cuuint64_t sti[3] = {(cuuint64_t)(2 * wp * 4), (cuuint64_t)(si[1] * 4),
                             (cuuint64_t)(si[0] * 4)};
  const cuuint32_t bi[4] = {(cuuint32_t)(2 * wp), 3, (cuuint32_t)CC, 1};
  const cuuint32_t e4[4] = {1, 1, 1, 1};
  const cuuint64_t dw[2] = {(cuuint64_t)f, (cuuint64_t)(c * 9)};
  const cuuint64_t stw[1] = {(cuuint64_t)(f * 4)};
  const cuuint32_t bw[2] = {(cuuint32_t)FT, (cuuint32_t)(CC * 9)};
  return enc(tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(in), di, sti, bi, e4,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS &&
         enc(tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(wt), dw, stw, bw, e4,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS;
}

// FCHW weights (any strides) -> [C][KH * KW][F], f fastest.
template <typename T>
__global__ void transpose_w_kernel(const T *__restrict__ w, int64_t s0, int64_t s1, int64_t s2,
                                   int64_t s3, T *__restrict__ dst, int f, int c, int kh, int kw) {
  const int total = f * c * kh * kw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ff = i % f, rest = i / f;
    const int tap = rest % (kh * kw), ci = rest / (kh * kw);
    const int ki = tap / kw, kj = tap - ki * kw;
    dst[i] = w[ff * s0 + ci * s1 + ki * s2 + kj * s3];
  }
}

template <typename T>
int launch(const void *in, const int64_t *si, const void *w, const int64_t *sw, void *w_work,
           void *out,
           const int64_t *so, int64_t nb, int64_t c, int64_t hp, int64_t wp, int64_t f,
           int64_t ho, int64_t wo, int64_t kh, int64_t kw, int32_t init, double init_value,
           cudaStream_t s) {
  ConvArgs<T> g{};
  g.in = static_cast<const T *>(in);
  g.w = static_cast<const T *>(w_work);
  g.out = static_cast<T *>(out);
  for (int d = 0; d < 4; ++d) g.si[d] = si[d], g.so[d] = so[d];
  g.nb = (int)nb; g.c = (int)c; g.hp = (int)hp; g.wp = (int)wp; g.f = (int)f;
  g.ho = (int)ho; g.wo = (int)wo; g.kh = (int)kh; g.kw = (int)kw;
  // pitch >= TW + KW - 1 and = 8 (mod 32): conflict-free 4-row x 8-pixel reads
  const int pw = (int)(TW + kw - 1);
  g.pitch = pw + ((8 - pw) % 32 + 32) % 32;
  g.th_tiles = (int)((ho + TH - 1) / TH);
  g.tw_tiles = (int)((wo + TW - 1) / TW);
  g.init = init;
  g.init_value = (T)init_value;
  const size_t smem =
      2 * (size_t)CC * ((TH + kh - 1) * g.pitch + kh * kw * FT) * sizeof(T);
  if (smem > 227 * 1024) return B200_EUNSUPPORTED;
  const int wt = (int)(f * c * kh * kw);
  transpose_w_kernel<T><<<(wt + 255) / 256 < 1024 ? (wt + 255) / 256 : 1024, 256, 0, s>>>(
      static_cast<const T *>(w), sw[0], sw[1], sw[2], sw[3], static_cast<T *>(w_work), (int)f,
      (int)c, (int)kh, (int)kw);
  dim3 grid((unsigned)(nb * g.th_tiles * g.tw_tiles), (unsigned)((f + FT - 1) / FT));
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<grid, kThreads, smem, s>>>(g);
  };
  const char *variant = getenv("B200_CONV_EXACT");   // dev A/B: "old", "rows", "runs"
  // 56-wide runs tiles when they pad the width less than 32-wide tiles
  const bool runs = kh == 3 && kw == 3 &&
                    (variant ? variant[0] == 'r' && variant[1] == 'u'
                             : (wo + 55) / 56 * 56 <= (wo + 31) / 32 * 32);
  if (runs) {
    auto even = [](int64_t v) { return (v & 1) == 0; };
    const int vec_in = si[3] == 1 && even(si[0]) && even(si[1]) && even(si[2]) &&
                       (reinterpret_cast<uintptr_t>(in) % (2 * sizeof(T))) == 0;
    const int vec_w = (f % (16 / sizeof(T))) == 0 &&
                      (reinterpret_cast<uintptr_t>(w_work) % 16) == 0;
    constexpr int PW = 56 + 2, PITCH = PW + ((8 - PW) % 32 + 32) % 32;
    const size_t rsmem = 2 * (size_t)CC * ((PTH + 2) * PITCH + 9 * FT) * sizeof(T);
    ConvArgs<T> gr = g;
    gr.th_tiles = (int)((ho + PTH - 1) / PTH);
    gr.tw_tiles = (int)((wo + 55) / 56);
    dim3 rgrid((unsigned)(nb * gr.th_tiles * gr.tw_tiles), (unsigned)((f + FT - 1) / FT));
    const char *tv = getenv("B200_CONV_EXACT_TMA");   // dev A/B: "0" = cp.async staging
    if constexpr (std::is_same<T, float>::value) {
      CUtensorMap tin, tw;
      if (!(tv && tv[0] == '0') &&
          runs_tma_maps(&tin, &tw, static_cast<const float *>(in), si,
                        static_cast<const float *>(w_work), nb, c, hp, wp, f)) {
        const size_t in_stage = ((size_t)CC * (PTH + 2) * wp * 4 + 127) / 128 * 128;
        const size_t tsmem = 1024 + TSTG * (in_stage + (size_t)CC * 9 * FT * 4) + 64;
        if (tsmem <= 227 * 1024) {
          auto kernel = conv_runs_tma_kernel<7>;
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tsmem);
          kernel<<<rgrid, kThreads, tsmem, s>>>(tin, tw, gr);
          return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
        }
      }
    }
    auto kernel = conv_runs_kernel<T, 3, 3, 7>;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    kernel<<<rgrid, kThreads, rsmem, s>>>(gr, vec_in, vec_w);
  } else if (kh == 3 && kw == 3 && !(variant && variant[0] == 'o')) {
    // the consecutive-column variant: its own pitch and vector staging flags
    auto even = [](int64_t v) { return (v & 1) == 0; };
    const int vec_in = si[3] == 1 && even(si[0]) && even(si[1]) && even(si[2]) &&
                       (reinterpret_cast<uintptr_t>(in) % (2 * sizeof(T))) == 0;
    const int vec_w = (f % (16 / sizeof(T))) == 0 &&
                      (reinterpret_cast<uintptr_t>(w_work) % 16) == 0;
    const int vec_out = sizeof(T) == 4 && so[3] == 1 && so[0] % 4 == 0 && so[1] % 4 == 0 &&
                        so[2] % 4 == 0 && (reinterpret_cast<uintptr_t>(out) % 16) == 0;
    const size_t rsmem = 2 * (size_t)CC * ((TH + 2) * RPITCH + 9 * FT) * sizeof(T);
    auto kernel = conv_rows_kernel<T, 3, 3>;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    kernel<<<grid, kThreads, rsmem, s>>>(g, vec_in, vec_w, vec_out);
  } else if (kh == 3 && kw == 3) {
    go(conv_exact_kernel<T, 3, 3>);
  } else {
    go(conv_exact_kernel<T, 0, 0>);
  }
  return cudaGetLastError() == cudaSuccess ? B200_OK : B200_ELAUNCH;
}

}  // namespace

extern "C" int b200_conv2d_exact(int32_t dtype, const void *in, const int64_t *in_strides,
                                 const void *w, const int64_t *w_strides, void *w_work,
                                 void *out,
                                 const int64_t *out_strides, int64_t nb, int64_t c, int64_t hp,
                                 int64_t wp, int64_t f, int64_t ho, int64_t wo, int64_t kh,
                                 int64_t kw, int32_t init, double init_value, void *stream) {
  if (nb <= 0 || f <= 0 || ho <= 0 || wo <= 0) return B200_OK;
  if (c <= 0 || kh <= 0 || kw <= 0 || ho + kh - 1 > hp || wo + kw - 1 > wp) return B200_EINVAL;
  // 32-bit index math in the kernel
  const int64_t lim = int64_t(1) << 31;
  if (nb * ((ho + TH - 1) / TH) * ((wo + TW - 1) / TW) >= lim || hp >= lim || wp >= lim ||
      c * in_strides[1] >= lim || f * c * kh * kw >= lim || f * out_strides[1] >= lim ||
      hp * in_strides[2] >= lim || ho * out_strides[2] >= lim)
    return B200_EUNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == B200_F32)
    return launch<float>(in, in_strides, w, w_strides, w_work, out, out_strides, nb, c, hp, wp, f, ho,
                         wo, kh, kw, init, init_value, s);
  if (dtype == B200_F64)
    return launch<double>(in, in_strides, w, w_strides, w_work, out, out_strides, nb, c, hp, wp, f, ho,
                          wo, kh, kw, init, init_value, s);
  return B200_EINVAL;
}
