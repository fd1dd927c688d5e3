// Tensor-core channel kernel (cgm_tc.cuh) on a BASELINE shape, standalone:
// device time over repeated launches and a per-CTA event timeline
// (clock64 stamps, KernelParams::trace).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tc_bench tc_bench.cu
// Run: ./tc_bench [B U S n_sc exact nstg debug]
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_1404_0424_b200/csrc/cgm_tc.cuh"
using namespace cgm;

template <bool EXACT, int NEP, int NSP, int RING = 2>
void run(KernelParams p, int nstg, const char* tag) {
  tc::Smem L;
  L.plan(p.S, EXACT, nstg, RING);
  p.k1_pair = nstg;
  auto k = channel_tc_kernel<EXACT, NEP, NSP, RING>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * (NEP + NSP + 2), L.total);
  {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("   attrs: regs=%d static_smem=%zu max_threads=%d local=%zu\n", fa.numRegs, fa.sharedSizeBytes,
           fa.maxThreadsPerBlock, fa.localSizeBytes);
    for (int sm : {20000, 60000, 100000, 110000}) {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 32 * (NEP + NSP + 2), sm);
      printf("   occ(smem=%d) = %d\n", sm, o);
    }
  }
  const int g = static_cast<int>(std::min<long>(p.n_sc, (long)sms * (occ > 0 ? occ : 1)));
  const int nt = 32 * (NEP + NSP + 2);
  unsigned long long* tr = p.trace;
  p.trace = nullptr;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<g, nt, L.total>>>(p);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) k<<<g, nt, L.total>>>(p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%s NEP=%d NSP=%d RING=%d nstg=%d smem=%d occ=%d grid=%d: %.2f us  (%s)\n", tag, NEP, NSP, RING, nstg, L.total, occ, g,
         1000 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  {  // correctness of G and MF against FP64 on the host (first 4 subcarriers)
    cudaDeviceSynchronize();
    WsOffsets W;
    W.plan(32, p.S, p.K, EXACT);
    const int ncheck = static_cast<int>(std::min<long>(p.n_sc, 4));
    std::vector<float2> ws(ncheck * W.stride), H(ncheck * p.B * 32), Y(ncheck * p.B * p.S);
    cudaMemcpy(ws.data(), p.ws, ws.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(H.data(), p.H, H.size() * 8, cudaMemcpyDeviceToHost);
    if (p.S) cudaMemcpy(Y.data(), p.Y, Y.size() * 8, cudaMemcpyDeviceToHost);
    double maxe = 0;
    for (int sc = 0; sc < ncheck; ++sc)
      for (int u = 0; u < 32; ++u) {
        for (int j = 0; j < 32; ++j) {
          double re = 0, im = 0, sc_ = 0;
          for (int b = 0; b < p.B; ++b) {
            const float2 x = H[(sc * p.B + b) * 32 + u], z = H[(sc * p.B + b) * 32 + j];
            re += (double)x.x * z.x + (double)x.y * z.y;
            im += (double)x.x * z.y - (double)x.y * z.x;
            sc_ += fabs((double)x.x * z.x) + fabs((double)x.y * z.y) + 1e-30;
          }
          const float2 g = ws[sc * W.stride + W.g + u * 32 + j];
          maxe = fmax(maxe, (fabs(g.x - re) + fabs(g.y - im)) / sc_);
        }
        for (int s_ = 0; s_ < p.S; ++s_) {
          double re = 0, im = 0, sc_ = 1e-30;
          for (int b = 0; b < p.B; ++b) {
            const float2 x = H[(sc * p.B + b) * 32 + u], z = Y[(sc * p.B + b) * p.S + s_];
            re += (double)x.x * z.x + (double)x.y * z.y;
            im += (double)x.x * z.y - (double)x.y * z.x;
            sc_ += fabs((double)x.x * z.x) + fabs((double)x.y * z.y);
          }
          const float2 m = ws[sc * W.stride + W.mf + s_ * 32 + u];
          maxe = fmax(maxe, (fabs(m.x - re) + fabs(m.y - im)) / sc_);
        }
      }
    printf("   check: max |err| / sum|terms| over %d subcarriers = %.3e %s\n", ncheck, maxe, maxe < 1e-5 ? "OK" : "BAD");
  }
  if (!tr) return;
  p.trace = tr;
  if (g > 148) return;
  cudaMemset(tr, 0, sizeof(unsigned long long) * g * 512);
  k<<<g, nt, L.total>>>(p);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(g * 512);
  cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
  const char* names[32] = {"tma0", "tmaL", "stg0", "split0", "stgL", "splitL", "mma0",
                           "mmaL", "mmadone", "accfull", "accfree", "Gcopy", "basis", "pcs0ok",
                           "pcsLok", "-", "ld0", "ld1", "stores", "bar1", "copy", "-", "-", "-",
                           "-", "-", "-", "-", "-", "-", "-", "-"};
  for (int cta : {0, g / 2}) {
    printf(" CTA %d timeline (clk rel. to first TMA issue):\n", cta);
    const unsigned long long t0 = h[(cta * 16) * 32 + 0];
    for (int i = 0; i < 10; ++i) {
      printf("  sc%-2d", i);
      for (int ev = 0; ev < 32; ++ev) {
        const unsigned long long v = h[(cta * 16 + i) * 32 + ev];
        if (v) printf(" %s=%lld", names[ev], static_cast<long long>(v - t0));
      }
      printf("\n");
    }
  }
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 128, U = argc > 2 ? atoi(argv[2]) : 32,
            S = argc > 3 ? atoi(argv[3]) : 14;
  const long n_sc = argc > 4 ? atol(argv[4]) : 1200;
  const int exact = argc > 5 ? atoi(argv[5]) : 0, nstg = argc > 6 ? atoi(argv[6]) : 3;
  const int debug = argc > 7 ? atoi(argv[7]) : 0;
  float2 *H, *Y, *ws;
  cudaMalloc(&H, n_sc * B * U * 8);
  cudaMalloc(&Y, n_sc * B * S * 8);
  WsOffsets W;
  W.plan(32, S, 4, exact);
  cudaMalloc(&ws, n_sc * W.stride * 8);
  std::vector<float2> h(n_sc * B * U);
  for (size_t i = 0; i < h.size(); ++i)
    h[i] = make_float2((i * 37 % 101) * 0.01f - 0.5f, (i * 13 % 97) * 0.01f - 0.5f);
  cudaMemcpy(H, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  {
    std::vector<float2> hy(n_sc * B * S);
    for (size_t i = 0; i < hy.size(); ++i) hy[i] = make_float2((i * 29 % 89) * 0.02f - 0.9f, (i * 17 % 83) * 0.02f - 0.8f);
    cudaMemcpy(Y, hy.data(), hy.size() * 8, cudaMemcpyHostToDevice);
  }
  unsigned long long* tr;
  cudaMalloc(&tr, 148 * 512 * 8);
  KernelParams p{};
  p.H = H; p.Y = Y; p.ws = ws; p.n_sc = n_sc; p.B = B; p.U = U; p.S = S; p.K = 4;
  p.bits = 6; p.use_tma = 1; p.rho_inv_u = 1.f; p.n0 = 1.f; p.es = 1.f; p.debug = debug < 0 ? 0 : debug;
  p.trace = tr;
  printf("channel_tc_kernel B=%d U=%d S=%d n_sc=%ld exact=%d\n", B, U, S, n_sc, exact);
  if (exact) {
    run<true, 4, 8>(p, nstg, "exact");
    p.trace = nullptr;
    run<true, 8, 0>(p, nstg, "exact unified");
    run<true, 16, 0>(p, nstg, "exact unified");
  } else {
    run<false, 8, 8>(p, nstg, "approx");
    p.trace = nullptr;
    run<false, 4, 4, 1>(p, 2, "approx 2cta");
    run<false, 4, 4, 1>(p, 3, "approx 2cta");
    run<false, 4, 2, 1>(p, 2, "approx 2cta");
    run<false, 4, 8>(p, nstg, "approx");
    run<false, 8, 0>(p, nstg, "approx unified");
    run<false, 16, 0>(p, nstg, "approx unified");
    if (debug < 0) return 0;
    const int dbg[][2] = {{1024 | 256 | 512 | 4096, 0}, {1024 | 256 | 4096, 0}, {1024 | 512 | 4096, 0},
                          {1024 | 4096, 0}, {1024, 0}, {4096, 0}, {512, 0}, {256, 0}, {128, 0},
                          {128 | 256 | 512 | 4096, 0}};
    const char* what[] = {"MMA only", "MMA+epi loads", "MMA+split", "MMA+split+epi", "no TMA",
                          "no Gcopy", "no epi loads", "no split", "no MMA", "TMA only"};
    for (int c = 0; c < 10; ++c) {
      p.debug = dbg[c][0];
      printf("%-14s dbg=%5d: ", what[c], p.debug);
      run<false, 4, 8>(p, nstg, "approx");
      printf("%-14s dbg=%5d: ", what[c], p.debug);
      run<false, 8, 8>(p, nstg, "approx");
    }
  }
  return 0;
}
