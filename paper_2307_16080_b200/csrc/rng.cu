// The tuner's seeded inputs, drawn natively (host code).
//
// The reference tuner fills every float memref argument with
// rng.uniform(-2.0, 2.0) from one random.Random(seed) stream, element by
// element (reference pkg/src/staircase/tuner/search.py:78-102).  CPython's
// random is MT19937 (624-word state, index `pos`); random() is
// genrand_res53: two tempered 32-bit draws a, b ->
// ((a >> 5) * 2^26 + (b >> 6)) / 2^53, and uniform(lo, hi) = lo + (hi - lo) *
// random() in double, stored into an f32 Buffer with round-to-nearest.
// b200_mt_uniform continues a given state (the Python generator's getstate()
// words and index) for n such values and leaves the state where Python's
// would be, so the caller can hand it back (setstate) for the next argument.
// Bit-identical to the Python loop (tests/test_sweep.py), ~5x faster than a
// numpy RandomState round trip on the sweep's 1024^2 operands; it runs on the
// host because the values are host Buffers the reference run reads.
#include <stdint.h>

#include "../../include/b200k.h"

namespace {

constexpr int kN = 624, kM = 397;

inline void twist(uint32_t *mt) {
  int i = 0;
  for (; i < kN - kM; ++i) {
    const uint32_t y = (mt[i] & 0x80000000u) | (mt[i + 1] & 0x7fffffffu);
    mt[i] = mt[i + kM] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
  }
  for (; i < kN - 1; ++i) {
    const uint32_t y = (mt[i] & 0x80000000u) | (mt[i + 1] & 0x7fffffffu);
    mt[i] = mt[i + kM - kN] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
  }
  const uint32_t y = (mt[kN - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
  mt[kN - 1] = mt[kM - 1] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
}

inline uint32_t draw(uint32_t *mt, int &pos) {
  if (pos >= kN) {
    twist(mt);
    pos = 0;
  }
  uint32_t y = mt[pos++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

}  // namespace

extern "C" int b200_mt_uniform(uint32_t *state, int32_t *pos, int64_t n, double lo, double hi,
                               void *out, int32_t dtype) {
  if (!state || !pos || n < 0 || (n > 0 && !out) || *pos < 0 || *pos > kN ||
      (dtype != B200_F32 && dtype != B200_F64))
    return B200_EINVAL;
  int p = *pos;
  // (hi - lo) * r then + lo, two rounded double ops as CPython evaluates
  // them (the build passes -ffp-contract=off to the host compiler)
  const double span = hi - lo;
  auto value = [&](uint32_t a, uint32_t b) {
    const double r = ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) *
                     (1.0 / 9007199254740992.0);
    const double scaled = span * r;
    return lo + scaled;
  };
  auto store = [&](int64_t i, double v) {
    if (dtype == B200_F32)
      static_cast<float *>(out)[i] = (float)v;
    else
      static_cast<double *>(out)[i] = v;
  };
  int64_t i = 0;
  // whole blocks: twist, temper all 624 words at once (a vectorisable loop),
  // then turn word pairs into values; a value whose two draws straddle a
  // block boundary is assembled by the scalar path
  uint32_t tw[kN];
  while (i < n) {
    if (p == kN && n - i >= kN / 2) {
      twist(state);
      for (int k = 0; k < kN; ++k) {
        uint32_t y = state[k];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        tw[k] = y;
      }
      for (int k = 0; k < kN / 2; ++k) store(i + k, value(tw[2 * k], tw[2 * k + 1]));
      i += kN / 2;
      continue;   // p stays kN: the next block twists again
    }
    const uint32_t a = draw(state, p), b = draw(state, p);
    store(i++, value(a, b));
  }
  *pos = p;
  return B200_OK;
}

// Strided host <-> device block copies for the streamed GEMMs (one
// cudaMemcpy2DAsync per block: column panels of B and (row, column) blocks of
// C are not contiguous, and a framework copy of a non-contiguous host view
// would first gather it on the host).  kind 1: host -> device, 2: device ->
// host; pitches and width in bytes; host memory page-locked for overlap.
#include <cuda_runtime.h>

extern "C" int b200_copy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                           int64_t width, int64_t rows, int32_t kind, void *stream) {
  if (!dst || !src || width < 0 || rows < 0 || dpitch < width || spitch < width ||
      (kind != 1 && kind != 2))
    return B200_EINVAL;
  if (width == 0 || rows == 0) return B200_OK;
  const cudaError_t e = cudaMemcpy2DAsync(
      dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)rows,
      kind == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? B200_OK : B200_ELAUNCH;
}
