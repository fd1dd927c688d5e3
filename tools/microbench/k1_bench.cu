// Channel-kernel variants on the cfg2 shape (B=128, U=32, S=14, 1200
// subcarriers, approx) and raw PCIe copy bandwidth.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o k1_bench k1_bench.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1404_0424_b200/csrc/cgm_split.cuh"
using namespace cgm;

template <int MINB, bool PIPE>
float run(KernelParams p, int nstage, int spl, int grid_per_sm, int reps) {
  K1Smem<32> L; L.plan(p.B, p.S, false, nstage);
  K1Split sp; sp.plan(32, p.B, p.S);
  if (spl > 0) { sp.spl = spl; sp.wpp = (spl * sp.n_tiles + 31) / 32; }
  p.k1_pair = nstage; p.k1_spl = sp.spl; p.k1_wpp = sp.wpp;
  const int nt = 32 * sp.wpp;
  auto k = channel_kernel<32, false, MINB, PIPE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nt, L.total);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int g = std::min<long>(p.n_sc, (long)sms * std::min(occ, grid_per_sm));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<g, nt, L.total>>>(p);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<<<g, nt, L.total>>>(p);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("  MINB=%d PIPE=%d nstage=%d spl=%d nt=%d occ=%d grid=%d smem=%d : %.2f us  %s\n", MINB, PIPE,
         nstage, sp.spl, nt, occ, g, L.total, 1000 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  return ms / reps;
}

template <int MINB, int NSO, bool GREG = false>
void run2(KernelParams p) {
  K2Smem<32> L; L.plan(p.B, p.S, 0, 4, false);
  using GE = K2Geo<32, NSO>;
  const int nw = (p.S + GE::GPW * GE::NS - 1) / (GE::GPW * GE::NS);
  auto k = solve_kernel<32, false, MINB, NSO, GREG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * nw, L.total);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<p.n_sc, 32 * nw, L.total>>>(p);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) k<<<p.n_sc, 32 * nw, L.total>>>(p);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("  K2 MINB=%d NS=%d GREG=%d warps=%d occ=%d : %.2f us %s\n", MINB, GE::NS, GREG, nw, occ, 1000 * ms / 20,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int B = 128, U = 32, S = 14; const long n_sc = 1200;
  float2 *H, *Y, *ws;
  cudaMalloc(&H, n_sc * B * U * 8); cudaMalloc(&Y, n_sc * B * S * 8);
  WsOffsets W; W.plan(32, S, 4, false);
  cudaMalloc(&ws, n_sc * W.stride * 8);
  std::vector<float2> h(n_sc * B * U);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_float2((i * 37 % 101) * 0.01f, (i * 13 % 97) * 0.01f);
  cudaMemcpy(H, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(Y, 0, n_sc * B * S * 8);
  KernelParams p{}; p.H = H; p.Y = Y; p.ws = ws; p.n_sc = n_sc; p.B = B; p.U = U; p.S = S; p.K = 4;
  p.bits = 6; p.use_tma = 1; p.rho_inv_u = 1.f; p.n0 = 1.f; p.es = 1.f;
  printf("channel_kernel cfg2 shape:\n");
  for (int dbg : {4, 8, 12}) { p.debug = dbg; printf("debug=%d\n", dbg); run<2, true>(p, 2, 0, 2, 20); }
  p.debug = 0;
  for (int spl : {0, 2, 3, 4}) {
    run<2, true>(p, 2, spl, 2, 20);
    run<2, false>(p, 2, spl, 2, 20);
  }
  run<3, true>(p, 1, 0, 3, 20);
  run<3, false>(p, 1, 0, 3, 20);
  run<3, true>(p, 1, 3, 3, 20);
  run<2, true>(p, 1, 0, 2, 20);
  run<1, true>(p, 2, 0, 1, 20);
  // ---- solve kernel variants (workspace from one channel-kernel pass)
  p.debug = 0;
  run<2, true>(p, 2, 0, 2, 1);
  float2* xhat; float *mu, *rho, *llr; uint8_t* st;
  cudaMalloc(&xhat, n_sc * S * U * 8); cudaMalloc(&mu, n_sc * S * U * 4); cudaMalloc(&rho, n_sc * S * U * 4);
  cudaMalloc(&llr, n_sc * S * U * 6 * 4); cudaMalloc(&st, n_sc * S);
  p.xhat = xhat; p.mu = mu; p.rho = rho; p.llr = llr; p.status = st; p.K = 4;
  printf("solve_kernel cfg2 shape:\n");
  run2<3, 0>(p);
  run2<1, 1, true>(p);
  run2<2, 1, true>(p);
  p.debug = 32; run2<2, 1, true>(p); p.debug = 0;
  p.S = 7; run2<2, 1, true>(p); run2<3, 0>(p); p.S = 14;
  // PCIe
  const size_t nb = 256ull << 20;
  void *hp, *dp; cudaMallocHost(&hp, nb); cudaMalloc(&dp, nb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int dir = 0; dir < 2; ++dir) {
    cudaMemcpy(dp, hp, nb, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    for (int r = 0; r < 4; ++r) cudaMemcpyAsync(dir ? hp : dp, dir ? dp : hp, nb, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("pcie %s: %.1f GB/s\n", dir ? "D2H" : "H2D", 4.0 * nb / ms / 1e6);
  }
  // bidirectional
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  void *hp2, *dp2; cudaMallocHost(&hp2, nb); cudaMalloc(&dp2, nb);
  cudaEventRecord(a);
  for (int r = 0; r < 4; ++r) { cudaMemcpyAsync(dp, hp, nb, cudaMemcpyHostToDevice, s1); cudaMemcpyAsync(hp2, dp2, nb, cudaMemcpyDeviceToHost, s2); }
  cudaDeviceSynchronize(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("pcie bidir: %.1f GB/s each way\n", 4.0 * nb / ms / 1e6);
  return 0;
}
