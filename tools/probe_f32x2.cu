// Dev probe: FP32 pipe throughput of separately rounded multiply + add (the
// bit-exact MAC of the exact kernels), scalar (FMUL + FADD) vs packed
// (FMUL2 + FADD2, sm_100a), with an opaque integer hop between the packed
// multiply and add so ptxas cannot contract them into FFMA2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_f32x2.cu -o /tmp/pf2 && /tmp/pf2
#include <cstdio>
#include <cstdint>

typedef unsigned long long u64;
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
constexpr int CH = 8;  // independent chains per thread

__global__ void scalar_k(float *out, float x, float y, int n) {
  float acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(acc[c], y));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void packed_k(u64 *out, u64 x, u64 y, u64 zero, int n) {
  u64 acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = add2(acc[c], mul2(acc[c], y) ^ zero);
  u64 s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void packed_nobar_k(u64 *out, u64 x, u64 y, int n) {
  u64 acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = add2(acc[c], mul2(acc[c], y));
  u64 s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 148, bs = 256, blocks = sms * 8, n = 4096;
  void *buf;
  cudaMalloc(&buf, (size_t)blocks * bs * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  double macs = (double)blocks * bs * n * CH;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    scalar_k<<<blocks, bs>>>((float *)buf, 1.0001f, 0.9999f, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("scalar FMUL+FADD   : %.1f T MAC/s (%.1f TFLOP/s)\n", macs / ms / 1e9, 2 * macs / ms / 1e9);
    cudaEventRecord(e0);
    packed_k<<<blocks, bs>>>((u64 *)buf, 0x3f8000003f800001ull, 0x3f7fff003f7ffff0ull, 0ull, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("packed FMUL2+FADD2 : %.1f T MAC/s (%.1f TFLOP/s)\n", 2 * macs / ms / 1e9, 4 * macs / ms / 1e9);
    cudaEventRecord(e0);
    packed_nobar_k<<<blocks, bs>>>((u64 *)buf, 0x3f8000003f800001ull, 0x3f7fff003f7ffff0ull, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("packed (FFMA2)     : %.1f T MAC/s (%.1f TFLOP/s)\n", 2 * macs / ms / 1e9, 4 * macs / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
