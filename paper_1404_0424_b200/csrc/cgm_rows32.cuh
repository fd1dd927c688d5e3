// cgm_rows32.cuh -- K2 for U = 32 with the Gram row in registers.
//
// Same mathematics and outputs as solve_sc (cgm_split.cuh): K CG iterations
// on G + rho^-1 I per system (solvers.cpp:37-72, freeze / breakdown rules),
// the approximate tracker (detect.cpp:397-441) or the exact tracker's
// (alpha, beta) history for k2_exact_tail, LLRs, the precoder tail.
//
// Layout: lane u of a warp owns user row u; the warp keeps row u of G
// (G[u][j] = conj(G[j][u]), 64 registers) for the whole subcarrier and runs
// the systems of that subcarrier two at a time.  The matvec e_u = sum_j
// G[u][j] p_j is then 2 packed FFMA2 per (j, system) with p_j broadcast
// from shared memory (one LDS.128 per two columns) and no G traffic at all:
//   a += (g.x, g.y) * (p.x, p.x),  b += (g.x, g.y) * (p.y, p.y)
//   e = (a.x - b.y, b.x + a.y)
// versus the lane-per-row kernel's 4 FFMA + shared G loads per (j, system).
// Two warps per subcarrier (one CTA), so the per-subcarrier G row load is
// paid by 64 threads and ~16 warps share an SM.
#pragma once

#include <type_traits>

#include "cgm_split.cuh"

namespace cgm {

struct Rows32Smem {
  int k2, ps4, total;  // K2Smem plan first (Vs, hist, tails), then the p broadcast rows
  __host__ __device__ void plan(int B, int S, int St, int K, bool exact) {
    K2Smem<32> L;
    L.plan(B, S, St, K, exact);
    k2 = 0;
    ps4 = L.total;
    total = ps4 + 2 * 8 * 32 * 8;  // two broadcast rows per warp, up to 8 warps
  }
};

__device__ __forceinline__ unsigned long long f2dup_lo(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {lo, lo}; }" : "=l"(r) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long f2dup_hi(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {hi, hi}; }" : "=l"(r) : "l"(v));
  return r;
}

// sum over the 32 lanes of two values at once: 5 + 1 shuffles instead of 10
__device__ __forceinline__ void warp_sum2(float& a, float& b) {
  const int lane = threadIdx.x & 31;
  const bool hi = lane & 16;
  // lanes < 16 keep a's half-sums, lanes >= 16 b's
  const float send = hi ? a : b;
  const float keep = hi ? b : a;
  float v = keep + __shfl_xor_sync(0xffffffffu, send, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const float other = __shfl_xor_sync(0xffffffffu, v, 16);
  a = hi ? other : v;
  b = hi ? v : other;
}

// CG for the systems base, base + 1 of subcarrier sc on one warp (lane =
// user row), with row `lane` of G in `grow`; Ps = this warp's two broadcast
// rows.  Approx uplink systems write their outputs here; exact / downlink
// systems leave v in Vs and (exact) the (alpha, beta) history in hist.
// UPONLY: every system is an uplink vector with the same K (the
// approximate-tracker pairs kernel), so the per-system direction / iteration
// count branches fold away.
template <bool EXACT, bool UPONLY = false, int NS = 2>
__device__ __forceinline__ void rows32_pair(const KernelParams& p, long sc, const float2* mfsrc,
                                            int base, const unsigned long long (&grow)[32],
                                            float gdiag, float2* Ps, float* hist, float2* Vs,
                                            uint8_t* sys_st) {
  constexpr int UP = 32;
  static_assert(NS == 1 || NS % 2 == 0, "one system or systems in pairs");
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = UPONLY ? p.K : (p.K > p.Kt ? p.K : p.Kt);
  const int lane = threadIdx.x & 31;
  int sys[NS];
  bool live[NS], down[NS], broke[NS];
  float reg[NS], rn[NS], rn0[NS];
  int iters[NS];
  float2 v[NS], r[NS], pp[NS];
  // approximate tracker state; ia = 1 / alpha of the previous iterations
  float f0[NS], f1[NS], f2[NS], ia1[NS], ia2[NS], bm1[NS], bm2[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sys[s] = base + s;
    live[s] = sys[s] < nsys;
    down[s] = UPONLY ? false : sys[s] >= S;
    reg[s] = down[s] ? p.rho_inv_d : p.rho_inv_u;
    iters[s] = live[s] ? (down[s] ? p.Kt : p.K) : 0;
    float2 b = make_float2(0.f, 0.f);
    if (live[s] && lane < U)
      b = down[s] ? p.T[(sc * St + (sys[s] - S)) * static_cast<long>(U) + lane]
                  : mfsrc[sys[s] * UP + lane];
    v[s] = make_float2(0.f, 0.f);
    r[s] = b;
    pp[s] = b;
    Ps[s * UP + lane] = b;  // this warp's broadcast row for slot s
    rn[s] = cnorm(b);
    broke[s] = false;
    ia1[s] = ia2[s] = 1.f;
    bm1[s] = bm2[s] = 0.f;
    f0[s] = f1[s] = f2[s] = 0.f;
  }
  if constexpr (NS == 1) {
    rn[0] = group_sum<32>(rn[0]);
  } else {
#pragma unroll
    for (int q = 0; q < NS; q += 2) warp_sum2(rn[q], rn[q + 1 < NS ? q + 1 : q]);
  }
#pragma unroll
  for (int q = 0; q < NS; ++q) rn0[q] = rn[q];
  __syncwarp();
  for (int k = 1; k <= Kmax; ++k) {
    // e = (G + reg I) p on the packed pipe
    unsigned long long a0[NS], b0[NS], a1[NS], b1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a0[s] = b0[s] = a1[s] = b1[s] = 0ull;
#pragma unroll
    for (int j = 0; j < UP; j += 2) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj =
            *reinterpret_cast<const ulonglong2*>(Ps + s * UP + j);
        ffma2(a0[s], grow[j], f2dup_lo(pj.x));
        ffma2(b0[s], grow[j], f2dup_hi(pj.x));
        ffma2(a1[s], grow[j + 1], f2dup_lo(pj.y));
        ffma2(b1[s], grow[j + 1], f2dup_hi(pj.y));
      }
    }
    float2 e[NS];
    float curv[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float2 A0 = f2unpack(a0[s]), B0 = f2unpack(b0[s]);
      const float2 A1 = f2unpack(a1[s]), B1 = f2unpack(b1[s]);
      e[s].x = (A0.x - B0.y) + (A1.x - B1.y);
      e[s].y = (B0.x + A0.y) + (B1.x + A1.y);
      e[s].x = fmaf(reg[s], pp[s].x, e[s].x);
      e[s].y = fmaf(reg[s], pp[s].y, e[s].y);
      curv[s] = pp[s].x * e[s].x + pp[s].y * e[s].y;  // Re p^H e
    }
    if constexpr (NS == 1) {
    curv[0] = group_sum<32>(curv[0]);
  } else {
#pragma unroll
    for (int q = 0; q < NS; q += 2) warp_sum2(curv[q], curv[q + 1 < NS ? q + 1 : q]);
  }
    float alpha[NS], beta[NS], rnx[NS];
    bool upd[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool step = UPONLY ? live[s] : k <= iters[s];
      const bool frozen = !(rn[s] > 1e-28f * rn0[s]);  // solvers.cpp:21,25-27
      const bool go = step && !frozen && !broke[s];
      if (go && curv[s] < 1e-30f) broke[s] = true;  // solvers.cpp:55-57
      upd[s] = go && !broke[s];
      alpha[s] = upd[s] ? __fdividef(rn[s], curv[s]) : 1.f;
      beta[s] = 0.f;
      if (upd[s]) {
        v[s].x = fmaf(alpha[s], pp[s].x, v[s].x);
        v[s].y = fmaf(alpha[s], pp[s].y, v[s].y);
        r[s].x = fmaf(-alpha[s], e[s].x, r[s].x);
        r[s].y = fmaf(-alpha[s], e[s].y, r[s].y);
      }
      rnx[s] = cnorm(r[s]);
    }
    if constexpr (NS == 1) {
    rnx[0] = group_sum<32>(rnx[0]);
  } else {
#pragma unroll
    for (int q = 0; q < NS; q += 2) warp_sum2(rnx[q], rnx[q + 1 < NS ? q + 1 : q]);
  }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      float ia = 1.f;  // 1 / alpha
      if (upd[s]) {
        const float irn = __fdividef(1.f, rn[s]);  // MUFU.RCP: no IEEE slow-path call
        beta[s] = rnx[s] * irn;
        ia = curv[s] * irn;
        rn[s] = rnx[s];
        pp[s].x = fmaf(beta[s], pp[s].x, r[s].x);
        pp[s].y = fmaf(beta[s], pp[s].y, r[s].y);
      }
      if (UPONLY || k <= iters[s]) {
        if (!down[s]) {
          if (EXACT) {
            if (lane == 0) {
              hist[(sys[s] * Kmax + (k - 1)) * 2 + 0] = alpha[s];
              hist[(sys[s] * Kmax + (k - 1)) * 2 + 1] = beta[s];
            }
          } else {
            // Eq. (11) on the diagonal (detect.cpp:409-427)
            // k = 1: L_1 = alpha_1 (a select, not a branch)
            const float c1 = alpha[s] * (1.f + bm1[s]) * ia1[s];
            const float c2 = alpha[s] * bm2[s] * ia2[s];
            const float nk = f0[s] + (c1 - alpha[s] * (gdiag + reg[s])) * (f0[s] - f1[s]) -
                             c2 * (f1[s] - f2[s]);
            const float nf = k == 1 ? alpha[s] : nk;
            f2[s] = f1[s];
            f1[s] = f0[s];
            f0[s] = nf;
          }
        }
        ia2[s] = ia1[s]; ia1[s] = ia;
        bm2[s] = bm1[s]; bm1[s] = beta[s];
      }
    }
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (upd[s]) Ps[s * UP + lane] = pp[s];
    __syncwarp();
  }
  // ------------------------------------------------ per-system epilogue
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (!live[s]) continue;
    if ((EXACT || down[s]) && lane == 0) sys_st[sys[s]] = broke[s] ? 1 : 0;  // read by the tails
    if (EXACT || down[s]) {
      Vs[sys[s] * UP + lane] = v[s];
      continue;
    }
    if constexpr (!EXACT) {
      // approx uplink: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
      if (lane < U) {
        const long o = (sc * S + sys[s]) * static_cast<long>(U) + lane;
        const bool ok = !broke[s];
        const float2 xh = ok ? v[s] : make_float2(0.f, 0.f);
        const float mu_u = ok ? f0[s] * gdiag : 0.f;
        const float rho_u = ok ? gdiag / p.n0 : 0.f;
        if (p.xhat) p.xhat[o] = xh;
        if (p.mu) p.mu[o] = mu_u;
        if (p.rho) p.rho[o] = rho_u;
        if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
        if (p.status && lane == 0) p.status[sc * S + sys[s]] = ok ? 0 : 1;
      }
    }
  }
}

template <bool EXACT>
__global__ void __launch_bounds__(256, 2) solve_rows32_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.S, St = p.St, B = p.B;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  Rows32Smem R;
  R.plan(B, S, St, Kmax, EXACT);
  K2Smem<UP> L;
  L.plan(B, S, St, Kmax, EXACT);
  WsOffsets W;
  W.plan(UP, S, p.K, EXACT, p.fx);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* MUs = reinterpret_cast<float*>(smem + L.mu);
  float* RHOs = reinterpret_cast<float*>(smem + L.rho);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  float* gpart = reinterpret_cast<float*>(smem + L.gpart);
  float2* Ps = reinterpret_cast<float2*>(smem + R.ps4);
  const int nt = blockDim.x, nw = nt >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long lsc = blockIdx.x;
  const long sc = p.sc_base + lsc;
  const float2* ws = p.ws + lsc * W.stride;
  const float2* mfsrc = ws + W.mf;

  // row `lane` of G: G[u][j] = conj(G[j][u]) -- column reads, coalesced
  unsigned long long grow[UP];
#pragma unroll
  for (int j = 0; j < UP; ++j) {
    const float2 g = __ldg(ws + W.g + j * UP + lane);
    grow[j] = f2pack(g.x, -g.y);
  }
  const float gdiag = __ldg(ws + W.g + lane * UP + lane).x;

  for (int base = warp * 2; base < nsys; base += nw * 2)
    rows32_pair<EXACT>(p, sc, mfsrc, base, grow, gdiag, Ps + warp * 2 * UP, hist, Vs, sys_st);
  auto sync = [] { __syncthreads(); };
  if (EXACT && S > 0) {
    sync();
    k2_exact_tail<UP>(p, ws, W, sc, Kmax, hist, coef, MUs, RHOs, Vs, sys_st, nt, sync,
                      reinterpret_cast<float*>(smem + L.xp));
  }
  if (St > 0) {
    sync();
    k2_precode_tail<UP>(p, sc, Vs, Qs, gpart, sys_st, nt, sync);
  }
}


// Approximate-tracker uplink (no CTA-wide tail): one warp per (subcarrier,
// pair of systems) work item, so the grid is many short warps that the
// hardware scheduler balances (a CTA per subcarrier at 16 warps / SM leaves
// a 1.01-wave tail on cfg2's 1200 subcarriers).  Each warp reads its G row
// straight from the L2-resident workspace.
template <int NS>
__global__ void __launch_bounds__(128, NS == 1 ? 5 : NS == 2 ? 4 : 3) solve_rows32_pairs_kernel(const KernelParams p) {
  constexpr int UP = 32;
  __shared__ __align__(16) float2 Ps_all[4][NS * UP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npairs = (p.S + NS - 1) / NS;
  const long item = static_cast<long>(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (item >= p.n_sc * npairs) return;
  const long lsc = item / npairs;
  const int base = static_cast<int>(item - lsc * npairs) * NS;
  WsOffsets W;
  W.plan(UP, p.S, p.K, false, p.fx);
  const float2* ws = p.ws + lsc * W.stride;
  unsigned long long grow[UP];
#pragma unroll
  for (int j = 0; j < UP; ++j) {
    const float2 g = __ldg(ws + W.g + j * UP + lane);
    grow[j] = f2pack(g.x, -g.y);
  }
  const float gdiag = __ldg(ws + W.g + lane * UP + lane).x;
  rows32_pair<false, true, NS>(p, p.sc_base + lsc, ws + W.mf, base, grow, gdiag, Ps_all[warp],
                               nullptr, nullptr, nullptr);
}

// Persistent form of the approximate pairs kernel: warp w walks items w,
// w + (warps in the grid), ... and copies the NEXT item's G (8 KB) and
// matched filters into its shared slot with cp.async while the current
// item's CG runs, so the per-item L2 latency of the G row / b loads (the
// largest stall of the one-shot kernel) leaves the critical path.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(128, 4) solve_rows32_pairs_pf_kernel(const KernelParams p) {
  constexpr int UP = 32, NW = 4;
  extern __shared__ __align__(128) unsigned char smem[];
  // per warp: G [32][32], next-item MF [2][32], current MF [2][32], Ps [2][32]
  constexpr int SLOT = (UP * UP + 6 * UP) * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* Gb = reinterpret_cast<float2*>(smem + warp * SLOT);
  float2* MFn = Gb + UP * UP;
  float2* MFc = MFn + 2 * UP;
  float2* Ps = MFc + 2 * UP;
  const int S = p.S;
  const int npairs = (S + 1) >> 1;
  const long n_items = p.n_sc * npairs;
  const long stride = static_cast<long>(gridDim.x) * NW;
  WsOffsets W;
  W.plan(UP, S, p.K, false, p.fx);
  auto prefetch = [&](long item) {
    const long lsc = item / npairs;
    const int base = static_cast<int>(item - lsc * npairs) * 2;
    const float2* ws = p.ws + lsc * W.stride;
#pragma unroll
    for (int c = 0; c < UP * UP / 2 / 32; ++c)  // 16 B chunks of G, coalesced
      cp_async16(Gb + 2 * (c * 32 + lane), ws + W.g + 2 * (c * 32 + lane));
    // the pair's two matched-filter rows (one row when base + 1 == S)
    if (lane < (base + 1 < S ? 32 : 16)) cp_async16(MFn + 2 * lane, ws + W.mf + base * UP + 2 * lane);
    cp_async_commit();
  };
  long item = static_cast<long>(blockIdx.x) * NW + warp;
  if (item < n_items) prefetch(item);
  for (; item < n_items; item += stride) {
    cp_async_wait_all();
    __syncwarp();
    const long lsc = item / npairs;
    const int base = static_cast<int>(item - lsc * npairs) * 2;
    unsigned long long grow[UP];
#pragma unroll
    for (int j = 0; j < UP; ++j) {
      const float2 g = Gb[j * UP + lane];  // G[j][u]: row u of G = conj of column u
      grow[j] = f2pack(g.x, -g.y);
    }
    const float gdiag = Gb[lane * UP + lane].x;
    MFc[lane] = MFn[lane];
    MFc[UP + lane] = MFn[UP + lane];
    __syncwarp();  // Gb / MFn consumed: the next item may land there
    if (item + stride < n_items) prefetch(item + stride);
    rows32_pair<false, true, 2>(p, p.sc_base + lsc, MFc - base * UP, base, grow, gdiag, Ps,
                                nullptr, nullptr, nullptr);
    __syncwarp();
  }
}

// Exact-tracker uplink (St = 0), same one-warp-per-(subcarrier, system pair)
// grid: CG as above with the (alpha, beta) history kept per warp, then the
// tail of k2_exact_tail done inside the warp -- lanes 0 / 1 run the FP64
// coefficient recursion of system 0 / 1 (detect.cpp:336-368 on the
// Chebyshev basis), lane i extracts row i of B = L_K G and L_K from the
// basis T_1..T_K (coalesced row reads, T Hermitian) and forms mu, nu^2, rho
// (detect.cpp:375-395) and the LLRs.  Replaces the CTA-per-subcarrier tail
// whose extraction serialised on one lane group for S = 1 (cfg4).
__global__ void __launch_bounds__(128, 4) solve_rows32_exact_pairs_kernel(const KernelParams p) {
  constexpr int UP = 32, NW = 4;
  __shared__ __align__(16) float2 Ps_all[NW][2 * UP];
  __shared__ __align__(16) float2 Vs_all[NW][2 * UP];
  __shared__ float hist_all[NW][2 * kMaxK * 2];
  __shared__ float coef_all[NW][2][2 * (kMaxK + 2)];
  __shared__ uint8_t st_all[NW][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.S, U = p.U, K = p.K;
  const int npairs = (S + 1) >> 1;
  const long item = static_cast<long>(blockIdx.x) * NW + warp;
  if (item >= p.n_sc * npairs) return;
  const long lsc = item / npairs;
  const int base = static_cast<int>(item - lsc * npairs) * 2;
  const long sc = p.sc_base + lsc;
  WsOffsets W;
  W.plan(UP, S, K, true, p.fx);
  const float2* ws = p.ws + lsc * W.stride;
  unsigned long long grow[UP];
#pragma unroll
  for (int j = 0; j < UP; ++j) {
    const float2 g = __ldg(ws + W.g + j * UP + lane);
    grow[j] = f2pack(g.x, -g.y);
  }
  const float gdiag = __ldg(ws + W.g + lane * UP + lane).x;
  // per-warp arrays indexed by the subcarrier-wide system number (base, base + 1)
  float* hist = hist_all[warp] - base * K * 2;
  float2* Vs = Vs_all[warp] - base * UP;
  uint8_t* sys_st = st_all[warp] - base;
  rows32_pair<true, true>(p, sc, ws + W.mf, base, grow, gdiag, Ps_all[warp], hist, Vs, sys_st);
  __syncwarp();
  if (p.fx) {  // basis_extract_kernel finishes: x_hat and status now, the history for it
    float2* hw = const_cast<float2*>(ws) + W.t;
    for (int t = 0; t < 2; ++t) {
      const int sy = base + t;
      if (sy >= S) break;
      const bool ok = st_all[warp][t] == 0;
      if (lane < U && p.xhat)
        p.xhat[(sc * S + sy) * static_cast<long>(U) + lane] = ok ? Vs_all[warp][t * UP + lane]
                                                                : make_float2(0.f, 0.f);
      if (lane < K)
        hw[sy * K + lane] = make_float2(hist_all[warp][(t * K + lane) * 2],
                                        hist_all[warp][(t * K + lane) * 2 + 1]);
      if (lane == 0 && p.status) p.status[sc * S + sy] = ok ? 0 : 1;
    }
    return;
  }
  // ---------------- coefficient recursion of both systems, warp-parallel (FP64)
  const float2 cdv = ws[W.cd];
  for (int t = 0; t < 2; ++t)
    if (base + t < S)
      cheb_coef_warp(hist_all[warp] + t * K * 2, K, cdv.x, cdv.y, p.rho_inv_u, coef_all[warp][t],
                     coef_all[warp][t] + (kMaxK + 2));
  __syncwarp();
  // ---------------- extraction, lane i <-> row i of both systems
  const float* cl0 = coef_all[warp][0];
  const float* cb0 = cl0 + (kMaxK + 2);
  const float* cl1 = coef_all[warp][1];
  const float* cb1 = cl1 + (kMaxK + 2);
  const bool has1 = base + 1 < S;
  const float2* Tw = ws + W.t;
  const int i = lane;
  float ib2[2] = {0.f, 0.f}, ibl[2] = {0.f, 0.f}, mu_i[2] = {0.f, 0.f};
  // the K basis entries of a column pair are loaded together (predicated,
  // K rounded up to KM) so the L2 / HBM latency is paid once per batch
  auto extract = [&](auto km_tag) {
    constexpr int KM = decltype(km_tag)::value;
#pragma unroll 1
    for (int j0 = 0; j0 < UP; j0 += 2) {
      float2 t[2][KM];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int m = 1; m <= KM; ++m)
          t[jj][m - 1] = m <= K ? __ldg(Tw + (m - 1) * UP * UP + (j0 + jj) * UP + i)
                                : make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int j = j0 + jj;
        float2 B0 = make_float2(i == j ? cb0[0] : 0.f, 0.f);
        float2 L0 = make_float2(i == j ? cl0[0] : 0.f, 0.f);
        float2 B1 = make_float2(i == j ? cb1[0] : 0.f, 0.f);
        float2 L1 = make_float2(i == j ? cl1[0] : 0.f, 0.f);
#pragma unroll
        for (int m = 1; m <= KM; ++m) {
          if (m > K) break;
          const float2 tv = cconj(t[jj][m - 1]);  // T_m[i][j] = conj(T_m[j][i])
          B0.x = fmaf(cb0[m], tv.x, B0.x); B0.y = fmaf(cb0[m], tv.y, B0.y);
          B1.x = fmaf(cb1[m], tv.x, B1.x); B1.y = fmaf(cb1[m], tv.y, B1.y);
          if (m < K) {
            L0.x = fmaf(cl0[m], tv.x, L0.x); L0.y = fmaf(cl0[m], tv.y, L0.y);
            L1.x = fmaf(cl1[m], tv.x, L1.x); L1.y = fmaf(cl1[m], tv.y, L1.y);
          }
        }
        if (j == i) { mu_i[0] = B0.x; mu_i[1] = B1.x; }
        else { ib2[0] += cnorm(B0); ib2[1] += cnorm(B1); }
        ibl[0] += B0.x * L0.x + B0.y * L0.y;  // Re(B_ij conj(L_ij))
        ibl[1] += B1.x * L1.x + B1.y * L1.y;
      }
    }
  };
  if (K <= 4) extract(std::integral_constant<int, 4>{});
  else if (K <= 8) extract(std::integral_constant<int, 8>{});
  else extract(std::integral_constant<int, kMaxK>{});
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (t == 1 && !has1) break;
    const int sy = base + t;
    const float nu2 = ib2[t] * p.es + ibl[t] * p.n0;
    const bool ok = st_all[warp][t] == 0;
    const float mu = ok ? mu_i[t] : 0.f;
    const float rr = ok ? (nu2 <= 0.f ? 0.f : mu_i[t] * mu_i[t] / nu2) : 0.f;  // safe_rho
    const float2 xh = ok ? Vs_all[warp][t * UP + i] : make_float2(0.f, 0.f);
    if (i < U) {
      const long o = (sc * S + sy) * static_cast<long>(U) + i;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = mu;
      if (p.rho) p.rho[o] = rr;
      if (p.llr) store_llrs_fast(xh, mu, rr, p.bits, p.llr + o * p.bits);
    }
    if (p.status && i == 0) p.status[sc * S + sy] = ok ? 0 : 1;
  }
}

// ---------------------------------------------------------------------------
// Fully fused approximate-tracker uplink for U = 32 (cfg2): ONE warp per
// subcarrier does the Gram, the matched filters and all S systems' CG with
// no workspace round trip and no second kernel.
//   * H [B][32] and Y [B][S] stream through a two-slot ring of CB-antenna
//     chunks (cp.async.bulk + one mbarrier per slot, per warp);
//   * lane u accumulates row u of G = H^H H and its S matched-filter entries
//     in registers on the packed pipe: per antenna b, with hu = H[b][u],
//       acc_j += (h_j.x, h_j.y) * hu.x  +  (h_j.y, h_j.x) * (hu.y, -hu.y)
//     = conj(hu) h_j, H[b][:] and Y[b][:] read as broadcast LDS.128;
//   * the G row then IS the register-resident row rows32_pair uses, so the
//     systems run pair by pair straight out of the Gram.
// The full G row per lane is twice the one-triangle FLOPs, traded for zero
// synchronisation: the split path's tensor-core channel kernel plus solve
// kernel spend their time in per-subcarrier pipeline latency, not FLOPs.
__device__ __forceinline__ unsigned long long f2swap_hl(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {hi, lo}; }" : "=l"(r) : "l"(v));
  return r;
}

struct FusedSmem {
  int bar, ring, slot, hbytes, ybytes, mf, ps, xh, total, cb;
  __host__ __device__ void plan(int B, int S) {
    cb = 16;  // antennas per chunk
    while (cb > 1 && B % cb) cb >>= 1;
    hbytes = cb * 32 * 8;
    ybytes = cb * S * 8;
    slot = (hbytes + ybytes + 15) & ~15;
    bar = 0;
    ring = 16;
    mf = ring + 2 * slot;
    ps = mf + S * 32 * 8;
    xh = ps + 2 * 32 * 8;  // exact: per-pair (alpha, beta) history, v rows, status
    total = xh + (2 * kMaxK * 2 * 4 + 2 * 32 * 8 + 16);
  }
};

// EXACT (one vector per subcarrier, p.fx): the same warp then runs the CG
// with the (alpha, beta) history, writes x_hat / status / history and its G
// row to the workspace, and basis_kernel<32, true> finishes the tracker.
template <int MAXS, bool EXACT = false>
__global__ void __launch_bounds__(32) fused_rows32_approx_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int B = p.B, S = p.S;
  FusedSmem L;
  L.plan(B, S);
  const int CB = L.cb, nch = B / CB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Ms = reinterpret_cast<float2*>(smem + L.mf);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  const int lane = threadIdx.x;
  const long sc = p.sc_base + blockIdx.x;
  const float2* Hg = p.H + sc * static_cast<long>(B) * UP;
  const float2* Yg = p.Y + sc * static_cast<long>(B) * S;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncwarp();
  auto slot_h = [&](int c) { return reinterpret_cast<float2*>(smem + L.ring + (c & 1) * L.slot); };
  auto issue = [&](int c) {
    float2* hs = slot_h(c);
    fence_proxy_async();
    mbar_expect_tx(bar + (c & 1), static_cast<uint32_t>(L.hbytes + L.ybytes));
    bulk_g2s(hs, Hg + static_cast<long>(c) * CB * UP, L.hbytes, bar + (c & 1));
    bulk_g2s(reinterpret_cast<unsigned char*>(hs) + L.hbytes, Yg + static_cast<long>(c) * CB * S,
             L.ybytes, bar + (c & 1));
  };
  if (lane == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }
  unsigned long long acc[UP], mf[MAXS];
#pragma unroll
  for (int j = 0; j < UP; ++j) acc[j] = 0ull;
#pragma unroll
  for (int s = 0; s < MAXS; ++s) mf[s] = 0ull;
  for (int c = 0; c < nch; ++c) {
    mbar_wait(bar + (c & 1), static_cast<uint32_t>((c >> 1) & 1));
    const float2* hs = slot_h(c);
    const float2* ys = reinterpret_cast<const float2*>(reinterpret_cast<const unsigned char*>(hs) + L.hbytes);
#pragma unroll 2
    for (int k = 0; k < CB; ++k) {
      const float2 hu = hs[k * UP + lane];
      const unsigned long long ux = f2pack(hu.x, hu.x), uy = f2pack(hu.y, -hu.y);
      const ulonglong2* row = reinterpret_cast<const ulonglong2*>(hs + k * UP);
#pragma unroll
      for (int j2 = 0; j2 < UP / 2; ++j2) {
        const ulonglong2 h2 = row[j2];
        ffma2(acc[2 * j2], h2.x, ux);
        ffma2(acc[2 * j2], f2swap_hl(h2.x), uy);
        ffma2(acc[2 * j2 + 1], h2.y, ux);
        ffma2(acc[2 * j2 + 1], f2swap_hl(h2.y), uy);
      }
      const unsigned long long* yr = reinterpret_cast<const unsigned long long*>(ys + k * S);
#pragma unroll
      for (int s = 0; s < MAXS; ++s) {
        if (s < S) {
          const unsigned long long y = yr[s];
          ffma2(mf[s], y, ux);
          ffma2(mf[s], f2swap_hl(y), uy);
        }
      }
    }
    __syncwarp();  // every lane done with this slot
    if (lane == 0 && c + 2 < nch) issue(c + 2);
  }
  // matched filters to shared memory ([sys][u], the layout rows32_pair reads)
#pragma unroll
  for (int s = 0; s < MAXS; ++s)
    if (s < S) Ms[s * UP + lane] = f2unpack(mf[s]);
  float gdiag = 0.f;
#pragma unroll
  for (int j = 0; j < UP; ++j)
    if (j == lane) gdiag = f2unpack(acc[j]).x;
  __syncwarp();
  if constexpr (!EXACT) {
    for (int base = 0; base < S; base += 2)
      rows32_pair<false, true>(p, sc, Ms, base, acc, gdiag, Ps, nullptr, nullptr, nullptr);
  } else {
    const int K = p.K;
    WsOffsets W;
    W.plan(UP, S, K, true, p.fx);
    float2* ws = p.ws + static_cast<long>(blockIdx.x) * W.stride;
#pragma unroll
    for (int j = 0; j < UP; ++j) ws[W.g + lane * UP + j] = f2unpack(acc[j]);  // row u of G
    float* histw = reinterpret_cast<float*>(smem + L.xh);
    float2* Vsw = reinterpret_cast<float2*>(histw + 2 * kMaxK * 2);
    uint8_t* stw = reinterpret_cast<uint8_t*>(Vsw + 2 * UP);
    for (int base = 0; base < S; base += 2) {
      rows32_pair<true, true>(p, sc, Ms, base, acc, gdiag, Ps, histw - base * K * 2, Vsw - base * UP,
                              stw - base);
      __syncwarp();
      for (int t = 0; t < 2; ++t) {
        const int sy = base + t;
        if (sy >= S) break;
        const bool ok = stw[t] == 0;
        if (p.xhat)
          p.xhat[(sc * S + sy) * static_cast<long>(UP) + lane] = ok ? Vsw[t * UP + lane]
                                                                    : make_float2(0.f, 0.f);
        if (lane < K) ws[W.t + sy * K + lane] = make_float2(histw[(t * K + lane) * 2],
                                                           histw[(t * K + lane) * 2 + 1]);
        if (lane == 0 && p.status) p.status[sc * S + sy] = ok ? 0 : 1;
      }
      __syncwarp();
    }
  }
}

}  // namespace cgm
