// Calibration: achievable FFMA rate of the complex 4x4 tile pattern on B200.
//   mode 0: operands from registers (pure FFMA issue)
//   mode 1: operands from smem, all lanes of a warp read the same row (broadcast X, contiguous Y)
//   mode 2: 2x2 tile with smem operands
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_tile ffma_tile.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1404_0424_b200/csrc/cgm_device.cuh"
using namespace cgm;

__global__ void k_reg(float* out, int iters) {
  float2 acc[4][4];
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
  float2 x[4], y[4];
  for (int r = 0; r < 4; ++r) { x[r] = make_float2(threadIdx.x * 1e-3f + r, 0.5f); y[r] = make_float2(0.25f, r * 1e-3f); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) cfma_conj(acc[r][c], x[r], y[c]);
    x[0].x += 1e-7f;
  }
  float s = 0.f;
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) s += acc[r][c].x + acc[r][c].y;
  if (s == 1234.5f) out[0] = s;
}

template <int MODE>
__global__ void k_smem(float* out, int iters, int B) {
  extern __shared__ float2 hs[];
  for (int e = threadIdx.x; e < B * 32; e += blockDim.x) hs[e] = make_float2(e * 1e-4f, 1.f);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float s = 0.f;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1) {
      float2 acc[4][4];
      for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
      const int ib = (warp + it) & 7, jb = lane & 7;
      tile4x4_pipe(acc, hs, 32, ib * 4, hs, 32, jb * 4, 0, B);
      for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) s += acc[r][c].x;
    } else {
      float2 acc[2][2];
      for (int r = 0; r < 2; ++r) for (int c = 0; c < 2; ++c) acc[r][c] = make_float2(0.f, 0.f);
      const int ib = (warp + it) & 15, jb = lane & 15;
      tile2x2<true>(acc, hs, 32, ib * 2, hs, 32, jb * 2, 1 << 30, 0, B);
      for (int r = 0; r < 2; ++r) for (int c = 0; c < 2; ++c) s += acc[r][c].x;
    }
  }
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 20000, nt = 32 * warps, blocks = sms;
    k_reg<<<blocks, nt>>>(out, 100);
    cudaEventRecord(a);
    k_reg<<<blocks, nt>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ffma = double(blocks) * nt * iters * 64;
    printf("reg   warps/SM=%2d  %.1f TFMA/s  = %.1f FMA/clk/SM @%d MHz\n", warps, ffma / ms / 1e9,
           ffma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  const int B = 128;
  cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int warps : {4, 8, 16, 32}) {
    for (int mode : {1, 2}) {
      const int iters = 200, nt = 32 * warps, blocks = sms;
      if (mode == 1) k_smem<1><<<blocks, nt, B * 32 * 8>>>(out, 2, B); else k_smem<2><<<blocks, nt, B * 32 * 8>>>(out, 2, B);
      cudaEventRecord(a);
      if (mode == 1) k_smem<1><<<blocks, nt, B * 32 * 8>>>(out, iters, B); else k_smem<2><<<blocks, nt, B * 32 * 8>>>(out, iters, B);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ffma = double(blocks) * nt * iters * B * (mode == 1 ? 64 : 16);
      printf("smem%d warps/SM=%2d  %.1f TFMA/s  = %.1f FMA/clk/SM\n", mode == 1 ? 4 : 2, warps,
             ffma / ms / 1e9, ffma / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
