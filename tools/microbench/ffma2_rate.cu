// Packed FFMA2 vs scalar FFMA issue rate on B200 (12 independent chains per
// thread, register operands).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_rate ffma2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
template <bool PACKED>
__global__ void k(float* out, int iters) {
  constexpr int C = 12;
  if (PACKED) {
    unsigned long long acc[C], a = 0x3f8000003f800001ull, b = 0x3f8000013f800000ull;
    for (int c = 0; c < C; ++c) acc[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int c = 0; c < C; ++c) ffma2(acc[c], a, b);
    float s = 0.f;
    for (int c = 0; c < C; ++c) s += __uint_as_float(static_cast<unsigned>(acc[c]));
    if (s == 1.2345f) out[0] = s;
  } else {
    float acc[2 * C], a = 1.0000001f, b = 0.9999999f;
    for (int c = 0; c < 2 * C; ++c) acc[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int c = 0; c < 2 * C; ++c) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[c]) : "f"(a), "f"(b));
    float s = 0.f;
    for (int c = 0; c < 2 * C; ++c) s += acc[c];
    if (s == 1.2345f) out[0] = s;
  }
}
int main() {
  float* o;
  cudaMalloc(&o, 4);
  const int iters = 20000, blocks = 148 * 4, threads = 256;
  for (int packed = 0; packed < 2; ++packed) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      if (packed) k<true><<<blocks, threads>>>(o, iters); else k<false><<<blocks, threads>>>(o, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fma = double(blocks) * threads * iters * 24;  // scalar FMAs (24 per iteration either way)
    printf("%s: %.3f ms, %.1f TFLOP/s (FMA = 2 flop), %.1f FMA/clk/SM at 1965 MHz\n", packed ? "FFMA2" : "FFMA ",
           ms, 2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
