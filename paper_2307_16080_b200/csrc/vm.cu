// Device tape VM — the generic execution tier of the B200 backend.
//
// Executes the per-thread program produced by paper_2307_16080_b200/vmcode.py:
// one band point per thread, everything below the band in reference order.
// Semantics follow the reference evaluator instruction by instruction
// (reference pkg/src/staircase/interp/_evalpy.py:81-232):
//   * floats are held as doubles (like the reference's Python floats);
//     f32 ops are single IEEE ops via __f*_rn (never contracted into FMA),
//     f64 ops via __d*_rn;
//   * integers are int64 with two's-complement wrap, i32 wrap when flagged
//     (interp/buffer.py:22-24);
//   * loads/stores are row-major with optional per-dimension bounds checks
//     (interp/_evalpy.py:90-114); integer stores wrap to the buffer width;
//   * loop tests count one bookkeeping event per body entry
//     (interp/_evalpy.py:139-148).
// The program, the preload table and the buffer table are staged into shared
// memory once per CTA: every thread of a warp executes the same instruction
// stream, so instruction fetch is a shared-memory broadcast.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/b200k.h"

namespace {

enum {
  V_END = 0, V_CONST, V_BINF, V_BINI, V_CMPF, V_CMPI, V_CAST, V_LOAD, V_STORE,
  V_MOV, V_TEST, V_NEXT, V_JUMP, V_IFF, V_PCHECK, V_NOP, V_ZERO
};

constexpr int kMaxRegs = 256;
constexpr int kMaxBand = 16;
constexpr int kTally = 25;
constexpr int kThreads = 128;

struct VmParams {
  const int32_t *prog;
  const int32_t *init_regs;
  const int64_t *init_vals;
  const b200_buffer *bufs;
  unsigned long long *tally;
  b200_vm_error *err;
  int32_t n_words, n_init, n_regs, n_bufs, nd;
  int32_t band_regs[kMaxBand];
  int64_t band_lb[kMaxBand], band_step[kMaxBand], band_trip[kMaxBand];
  int64_t total;
};

__device__ __forceinline__ double as_f(uint64_t v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ uint64_t from_f(double d) { return (uint64_t)__double_as_longlong(d); }
__device__ __forceinline__ int64_t wrap32(int64_t v) { return (int64_t)(int32_t)(uint32_t)(uint64_t)v; }

__device__ __forceinline__ void report(b200_vm_error *err, int code, int slot, int64_t idx,
                                       int64_t extent, int64_t loc) {
  if (atomicCAS(&err->code, 0, code) == 0) {
    err->slot = slot;
    err->index = idx;
    err->extent = extent;
    err->loc = loc;
  }
}

template <bool COUNT>
__global__ void __launch_bounds__(kThreads) vm_kernel(VmParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  b200_buffer *sbuf = reinterpret_cast<b200_buffer *>(smem);
  int64_t *sinit_v = reinterpret_cast<int64_t *>(sbuf + p.n_bufs);
  int32_t *sinit_r = reinterpret_cast<int32_t *>(sinit_v + p.n_init);
  int32_t *sprog = sinit_r + p.n_init;
  {
    const int32_t *gb = reinterpret_cast<const int32_t *>(p.bufs);
    int32_t *sb = reinterpret_cast<int32_t *>(sbuf);
    int nb = p.n_bufs * (int)(sizeof(b200_buffer) / 4);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = gb[i];
    for (int i = threadIdx.x; i < p.n_init; i += blockDim.x) {
      sinit_v[i] = p.init_vals[i];
      sinit_r[i] = p.init_regs[i];
    }
    for (int i = threadIdx.x; i < p.n_words; i += blockDim.x) sprog[i] = p.prog[i];
  }
  __syncthreads();

  uint64_t R[kMaxRegs];
  unsigned long long cnt[kTally];
  if (COUNT)
    for (int i = 0; i < kTally; ++i) cnt[i] = 0;

  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t pt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pt < p.total; pt += stride) {
    for (int i = 0; i < p.n_init; ++i) R[sinit_r[i]] = (uint64_t)sinit_v[i];
    int64_t rem = pt;
    for (int d = p.nd - 1; d >= 0; --d) {
      int64_t t = rem % p.band_trip[d];
      rem /= p.band_trip[d];
      R[p.band_regs[d]] = (uint64_t)(p.band_lb[d] + p.band_step[d] * t);
    }
    int pc = 0;
    for (;;) {
      const int32_t w = sprog[pc];
      const int op = w & 0xff;
      const int tag = ((w >> 8) & 0xff) - 1;
      const int fl = (w >> 16) & 0xffff;
      if (COUNT && tag >= 0) cnt[tag] += 1;
      switch (op) {
        case V_END:
          goto done;
        case V_CONST: {
          uint64_t lo = (uint32_t)sprog[pc + 2], hi = (uint32_t)sprog[pc + 3];
          R[sprog[pc + 1]] = lo | (hi << 32);
          pc += 4;
          break;
        }
        case V_BINF: {
          double a = as_f(R[sprog[pc + 2]]), b = as_f(R[sprog[pc + 3]]), r;
          const int f = fl & 3;
          if (fl & 4) {
            float fa = (float)a, fb = (float)b, fr;
            if (f == 0) fr = __fadd_rn(fa, fb);
            else if (f == 1) fr = __fsub_rn(fa, fb);
            else if (f == 2) fr = __fmul_rn(fa, fb);
            else fr = __fdiv_rn(fa, fb);
            r = (double)fr;
          } else {
            if (f == 0) r = __dadd_rn(a, b);
            else if (f == 1) r = __dsub_rn(a, b);
            else if (f == 2) r = __dmul_rn(a, b);
            else r = __ddiv_rn(a, b);
          }
          R[sprog[pc + 1]] = from_f(r);
          pc += 4;
          break;
        }
        case V_BINI: {
          uint64_t a = R[sprog[pc + 2]], b = R[sprog[pc + 3]], r;
          const int f = fl & 3;
          r = f == 0 ? a + b : (f == 1 ? a - b : a * b);
          R[sprog[pc + 1]] = (fl & 4) ? (uint64_t)wrap32((int64_t)r) : r;
          pc += 4;
          break;
        }
        case V_CMPF: {
          double a = as_f(R[sprog[pc + 2]]), b = as_f(R[sprog[pc + 3]]);
          bool r;
          switch (fl & 7) {
            case 0: r = a == b; break;
            case 1: r = (a == a) && (b == b) && (a != b); break;
            case 2: r = a < b; break;
            case 3: r = a <= b; break;
            case 4: r = a > b; break;
            default: r = a >= b; break;
          }
          R[sprog[pc + 1]] = r;
          pc += 4;
          break;
        }
        case V_CMPI: {
          int64_t a = (int64_t)R[sprog[pc + 2]], b = (int64_t)R[sprog[pc + 3]];
          bool r;
          switch (fl & 7) {
            case 0: r = a == b; break;
            case 1: r = a != b; break;
            case 2: r = a < b; break;
            case 3: r = a <= b; break;
            case 4: r = a > b; break;
            default: r = a >= b; break;
          }
          R[sprog[pc + 1]] = r;
          pc += 4;
          break;
        }
        case V_CAST: {
          uint64_t v = R[sprog[pc + 2]];
          R[sprog[pc + 1]] = (fl & 1) ? (uint64_t)wrap32((int64_t)v) : v;
          pc += 3;
          break;
        }
        case V_LOAD:
        case V_STORE: {
          const int rank = fl & 15, checked = (fl >> 4) & 1, dt = (fl >> 5) & 3;
          const int slot = sprog[pc + 2];
          const b200_buffer &b = sbuf[slot];
          int64_t off = 0;
          for (int k = 0; k < rank; ++k) {
            int64_t i = (int64_t)R[sprog[pc + 3 + k]];
            if (checked && (i < 0 || i >= b.shape[k])) {
              report(p.err, 1, slot, i, b.shape[k], sprog[pc + 3 + rank]);
              goto fault;
            }
            off += i * b.strides[k];
          }
          const int reg = sprog[pc + 1];
          if (op == V_LOAD) {
            uint64_t v;
            if (dt == 0) v = from_f((double)static_cast<const float *>(b.ptr)[off]);
            else if (dt == 1) v = from_f(static_cast<const double *>(b.ptr)[off]);
            else if (dt == 2) v = (uint64_t)(int64_t) static_cast<const int32_t *>(b.ptr)[off];
            else v = (uint64_t) static_cast<const int64_t *>(b.ptr)[off];
            R[reg] = v;
          } else {
            uint64_t v = R[reg];
            if (dt == 0) static_cast<float *>(b.ptr)[off] = (float)as_f(v);
            else if (dt == 1) static_cast<double *>(b.ptr)[off] = as_f(v);
            else if (dt == 2) static_cast<int32_t *>(b.ptr)[off] = (int32_t)(uint32_t)v;
            else static_cast<int64_t *>(b.ptr)[off] = (int64_t)v;
          }
          pc += 4 + rank;
          break;
        }
        case V_MOV:
          R[sprog[pc + 1]] = R[sprog[pc + 2]];
          pc += 3;
          break;
        case V_TEST:
          if ((int64_t)R[sprog[pc + 1]] >= (int64_t)R[sprog[pc + 2]]) {
            pc = sprog[pc + 3];
          } else {
            if (COUNT && (fl & 1)) cnt[kTally - 1] += 1;
            pc += 4;
          }
          break;
        case V_NEXT: {
          int64_t step = (int64_t)R[sprog[pc + 2]];
          if ((fl & 1) && step <= 0) {
            report(p.err, 2, -1, step, 0, -1);
            goto fault;
          }
          R[sprog[pc + 1]] = (uint64_t)((int64_t)R[sprog[pc + 1]] + step);
          pc = sprog[pc + 3];
          break;
        }
        case V_JUMP:
          pc = sprog[pc + 1];
          break;
        case V_IFF:
          pc = R[sprog[pc + 1]] ? pc + 3 : sprog[pc + 2];
          break;
        case V_PCHECK: {
          const int nd = fl;
          for (int k = 0; k < nd; ++k)
            if ((int64_t)R[sprog[pc + 1 + k]] <= 0) {
              report(p.err, 3, -1, 0, 0, -1);
              goto fault;
            }
          pc += 1 + nd;
          break;
        }
        case V_ZERO: {
          // memref.alloc inside the region: a fresh zero-filled buffer
          // (reference _evalpy.py:209-210) — the region's scratch slot
          const int dt = fl & 3;
          const b200_buffer &b = sbuf[sprog[pc + 1]];
          const int64_t n = sprog[pc + 2];
          const int64_t bytes = n * (dt == 0 || dt == 2 ? 4 : 8);
          unsigned char *q = static_cast<unsigned char *>(b.ptr);
          for (int64_t i = 0; i < bytes; ++i) q[i] = 0;
          pc += 3;
          break;
        }
        default:  // V_NOP (counting only)
          pc += 1;
          break;
      }
    }
  done:;
  }
fault:
  if (COUNT) {
    const unsigned lane = threadIdx.x & 31;
    for (int i = 0; i < kTally; ++i) {
      unsigned long long v = cnt[i];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(&p.tally[i], v);
    }
  }
}

}  // namespace

extern "C" int b200_vm_run(const int32_t *prog, int32_t n_words, const int32_t *init_regs,
                           const int64_t *init_vals, int32_t n_init, int32_t n_regs,
                           const b200_buffer *bufs, int32_t n_bufs, int32_t nd,
                           const int32_t *band_regs, const int64_t *band_lb,
                           const int64_t *band_step, const int64_t *band_trip, int32_t count,
                           unsigned long long *tally, b200_vm_error *err, void *stream) {
  if (nd < 0 || nd > kMaxBand || n_regs > kMaxRegs || n_words <= 0) return B200_EINVAL;
  VmParams p{};
  p.prog = prog;
  p.init_regs = init_regs;
  p.init_vals = init_vals;
  p.bufs = bufs;
  p.tally = tally;
  p.err = err;
  p.n_words = n_words;
  p.n_init = n_init;
  p.n_regs = n_regs;
  p.n_bufs = n_bufs;
  p.nd = nd;
  int64_t total = 1;
  for (int d = 0; d < nd; ++d) {
    p.band_regs[d] = band_regs[d];
    p.band_lb[d] = band_lb[d];
    p.band_step[d] = band_step[d];
    p.band_trip[d] = band_trip[d];
    total *= band_trip[d];
  }
  p.total = total;
  if (total == 0) return B200_OK;
  size_t smem = (size_t)n_bufs * sizeof(b200_buffer) + (size_t)n_init * 12 + (size_t)n_words * 4;
  smem = (smem + 15) & ~(size_t)15;
  int64_t blocks = (total + kThreads - 1) / kThreads;
  const int64_t cap = 148 * 16;  // persistent cap: 16 CTAs per SM
  if (blocks > cap) blocks = cap;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (count) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(vm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    vm_kernel<true><<<(unsigned)blocks, kThreads, smem, s>>>(p);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(vm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    vm_kernel<false><<<(unsigned)blocks, kThreads, smem, s>>>(p);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? B200_OK : B200_ELAUNCH;
}
