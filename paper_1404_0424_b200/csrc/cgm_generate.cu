// cgm_generate.cu -- seeded synthetic inputs generated on the device.
//
// Mirrors the reference's counter-based splitmix64 streams (rng.cpp:12-52),
// the Rayleigh channel draw order (channel.cpp:10-17), transmit()'s AWGN
// (channel.cpp:21-30), Gray QAM mapping (constellation.cpp:37-99) and the
// harness's per-purpose forks (sim.cpp:151-154, 164, 178).  Because
// next_u64 is a pure function of (key, counter) and every complex Gaussian
// consumes exactly one Box-Muller pair, entry e of a stream uses counters
// 2e+1 and 2e+2 and every entry can be drawn by its own thread.  Integer
// streams are bit-exact with the reference; Gaussians agree to within the
// last ulp of the libm transcendental (double), i.e. bit-exact after the
// rounding to complex64 in all but rare cases.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/cgmimo_b200.h"

struct cgm_ctx;
extern "C" int cgm_internal_fail(cgm_ctx* ctx, int code, const char* msg);
extern "C" int cgm_internal_device(cgm_ctx* ctx, void** stream, int* sms, long** launches);

#include "cgm_rng.cuh"

namespace {

using namespace cgm_rng;

// Rayleigh entries: matrix [rows][cols] of subcarrier sc from root.fork(2).fork(sc)
__global__ void gen_rayleigh(float2* out, int rows, int cols, long sc0, long n_sc,
                             uint64_t chan_key) {
  const long per = static_cast<long>(rows) * cols;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < per * n_sc;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long sc = idx / per, e = idx - sc * per;
    const uint64_t key = fork_key(chan_key, static_cast<uint64_t>(sc0 + sc));
    const double2 g = gauss_pair(key, static_cast<uint64_t>(e), sqrt(0.5));
    out[idx] = make_float2(static_cast<float>(g.x), static_cast<float>(g.y));
  }
}

// Symbols of instance i = (sc0+sc)*S + s for every user: labels -> points.
__global__ void gen_symbols(float2* out, uint8_t* labels, int U, long sc0, long n_sc, int S,
                            int bits, uint64_t lab_key) {
  const long total = n_sc * S * U;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long inst = idx / U;
    const int u = static_cast<int>(idx - inst * U);
    const uint64_t key = fork_key(lab_key, static_cast<uint64_t>(sc0 * S + inst));
    const unsigned label = draw_label(key, u, bits);
    const double2 x = qam_point(label, bits);
    if (out) out[idx] = make_float2(static_cast<float>(x.x), static_cast<float>(x.y));
    if (labels) labels[idx] = static_cast<uint8_t>(label);
  }
}

// y = H x + n for every instance; one block per instance, thread per antenna.
// x from the label stream, n from root.fork(3).fork(i) (channel.cpp:21-30).
__global__ void gen_received(float2* Y, const float2* H, int B, int U, long sc0, long n_sc,
                             int S, int bits, double n0, uint64_t lab_key, uint64_t noise_key) {
  extern __shared__ double2 xs[];
  for (long inst = blockIdx.x; inst < n_sc * S; inst += gridDim.x) {
    const long sc = inst / S;
    const uint64_t gi = static_cast<uint64_t>(sc0 * S + inst);
    const uint64_t lk = fork_key(lab_key, gi);
    for (int u = threadIdx.x; u < U; u += blockDim.x) xs[u] = qam_point(draw_label(lk, u, bits), bits);
    __syncthreads();
    const uint64_t nk = fork_key(noise_key, gi);
    const float2* h = H + sc * static_cast<long>(B) * U;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      double re = 0.0, im = 0.0;  // matvec(H, x) (linalg.cpp:103-114)
      for (int u = 0; u < U; ++u) {
        const float2 hv = h[b * U + u];
        re += static_cast<double>(hv.x) * xs[u].x - static_cast<double>(hv.y) * xs[u].y;
        im += static_cast<double>(hv.x) * xs[u].y + static_cast<double>(hv.y) * xs[u].x;
      }
      const double2 nz = gauss_pair(nk, static_cast<uint64_t>(b), sqrt(0.5 * n0));
      // antenna-major batch layout: Y[sc][b][s]
      Y[(sc * B + b) * S + (inst - sc * S)] =
          make_float2(static_cast<float>(re + nz.x), static_cast<float>(im + nz.y));
    }
    __syncthreads();
  }
}

// H_u[b][u] = sum_b' conj(H_w[u][b']) R^{1/2}[b'][b]; one block per subcarrier.
__global__ void correlate(float2* Hu, const float2* Hw, const float* rsqrt, int B, int U,
                          long n_sc) {
  extern __shared__ float2 hw[];
  for (long sc = blockIdx.x; sc < n_sc; sc += gridDim.x) {
    const float2* src = Hw + sc * static_cast<long>(U) * B;
    for (int e = threadIdx.x; e < U * B; e += blockDim.x) hw[e] = src[e];
    __syncthreads();
    for (int e = threadIdx.x; e < U * B; e += blockDim.x) {
      const int b = e / U, u = e - b * U;
      double re = 0.0, im = 0.0;
      for (int k = 0; k < B; ++k) {
        const float r = rsqrt[k * B + b];
        re += static_cast<double>(hw[u * B + k].x) * r;
        im -= static_cast<double>(hw[u * B + k].y) * r;
      }
      Hu[sc * static_cast<long>(B) * U + e] = make_float2(static_cast<float>(re), static_cast<float>(im));
    }
    __syncthreads();
  }
}

int grid_for(long work, int sms) {
  long g = (work + 255) / 256;
  const long cap = static_cast<long>(sms) * 16;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int cgm_generate_symbols(cgm_ctx* ctx, int U, long sc0, long n_sc, int S, uint64_t seed,
                         int qam_bits, float* T, uint8_t* labels) {
  void* st = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &st, &sms, &launches)) return CGM_EINVAL;
  if (U < 1 || S < 1 || n_sc < 0 || (qam_bits != 2 && qam_bits != 4 && qam_bits != 6))
    return cgm_internal_fail(ctx, CGM_EINVAL, "generate_symbols: bad arguments");
  if (n_sc == 0) return CGM_OK;
  const uint64_t lab = fork_key(seed, 4);
  gen_symbols<<<grid_for(n_sc * S * U, sms), 256, 0, static_cast<cudaStream_t>(st)>>>(
      reinterpret_cast<float2*>(T), labels, U, sc0, n_sc, S, qam_bits, lab);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? CGM_OK
                                           : cgm_internal_fail(ctx, CGM_ECUDA, "gen_symbols launch");
}

int cgm_generate_downlink(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S,
                          uint64_t seed, int qam_bits, float* Hd, float* T, uint8_t* labels) {
  void* st = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &st, &sms, &launches)) return CGM_EINVAL;
  if (B < 1 || U < 1 || n_sc < 0) return cgm_internal_fail(ctx, CGM_EINVAL, "generate_downlink: bad arguments");
  if (n_sc == 0) return CGM_OK;
  gen_rayleigh<<<grid_for(n_sc * B * U, sms), 256, 0, static_cast<cudaStream_t>(st)>>>(
      reinterpret_cast<float2*>(Hd), U, B, sc0, n_sc, fork_key(seed, 2));
  ++*launches;
  if (cudaGetLastError() != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, "gen_rayleigh launch");
  if (T || labels) return cgm_generate_symbols(ctx, U, sc0, n_sc, S, seed, qam_bits, T, labels);
  return CGM_OK;
}

static int received(cgm_ctx* ctx, void* st, int sms, long* launches, int B, int U, long sc0,
                    long n_sc, int S, uint64_t seed, int qam_bits, double n0, const float* H,
                    float* Y, uint8_t* labels) {
  const long inst = n_sc * S;
  gen_received<<<grid_for(inst * 256, sms), 256, U * sizeof(double2), static_cast<cudaStream_t>(st)>>>(
      reinterpret_cast<float2*>(Y), reinterpret_cast<const float2*>(H), B, U, sc0, n_sc, S,
      qam_bits, n0, fork_key(seed, 1), fork_key(seed, 3));
  ++*launches;
  if (cudaGetLastError() != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, "gen_received launch");
  if (labels) {
    gen_symbols<<<grid_for(inst * U, sms), 256, 0, static_cast<cudaStream_t>(st)>>>(
        nullptr, labels, U, sc0, n_sc, S, qam_bits, fork_key(seed, 1));
    ++*launches;
    if (cudaGetLastError() != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, "gen_symbols launch");
  }
  return CGM_OK;
}

int cgm_generate_uplink(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S, uint64_t seed,
                        int qam_bits, double n0, float* H, float* Y, uint8_t* labels) {
  void* st = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &st, &sms, &launches)) return CGM_EINVAL;
  if (B < 1 || U < 1 || S < 1 || n_sc < 0 || !(n0 >= 0.0) || !H || !Y ||
      (qam_bits != 2 && qam_bits != 4 && qam_bits != 6))
    return cgm_internal_fail(ctx, CGM_EINVAL, "generate_uplink: bad arguments");
  if (n_sc == 0) return CGM_OK;
  gen_rayleigh<<<grid_for(n_sc * B * U, sms), 256, 0, static_cast<cudaStream_t>(st)>>>(
      reinterpret_cast<float2*>(H), B, U, sc0, n_sc, fork_key(seed, 2));
  ++*launches;
  if (cudaGetLastError() != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, "gen_rayleigh launch");
  return received(ctx, st, sms, launches, B, U, sc0, n_sc, S, seed, qam_bits, n0, H, Y, labels);
}

int cgm_generate_uplink_correlated(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S,
                                   uint64_t seed, int qam_bits, double n0, const float* rsqrt,
                                   float* H, float* Y, uint8_t* labels) {
  void* st = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &st, &sms, &launches)) return CGM_EINVAL;
  if (B < 1 || U < 1 || S < 1 || n_sc < 0 || !rsqrt || !H || !Y ||
      (qam_bits != 2 && qam_bits != 4 && qam_bits != 6))
    return cgm_internal_fail(ctx, CGM_EINVAL, "generate_uplink_correlated: bad arguments");
  if (n_sc == 0) return CGM_OK;
  const size_t smem = static_cast<size_t>(U) * B * sizeof(float2);
  if (smem > 200 * 1024) return cgm_internal_fail(ctx, CGM_EINVAL, "correlated channel too large");
  float2* hw = nullptr;
  if (cudaMallocAsync(&hw, static_cast<size_t>(n_sc) * U * B * sizeof(float2),
                      static_cast<cudaStream_t>(st)) != cudaSuccess)
    return cgm_internal_fail(ctx, CGM_ENOMEM, "correlated scratch");
  gen_rayleigh<<<grid_for(n_sc * B * U, sms), 256, 0, static_cast<cudaStream_t>(st)>>>(
      hw, U, B, sc0, n_sc, fork_key(seed, 2));
  cudaFuncSetAttribute(correlate, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  correlate<<<grid_for(n_sc * 256, sms), 256, smem, static_cast<cudaStream_t>(st)>>>(
      reinterpret_cast<float2*>(H), hw, rsqrt, B, U, n_sc);
  *launches += 2;
  cudaFreeAsync(hw, static_cast<cudaStream_t>(st));
  if (cudaGetLastError() != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, "correlate launch");
  return received(ctx, st, sms, launches, B, U, sc0, n_sc, S, seed, qam_bits, n0, H, Y, labels);
}

}  // extern "C"
