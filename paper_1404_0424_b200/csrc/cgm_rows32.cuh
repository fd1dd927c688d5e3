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
#include "cgm_moments.cuh"

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
  a = __shfl_sync(0xffffffffu, v, 0);   // lanes < 16 hold sum(a)
  b = __shfl_sync(0xffffffffu, v, 16);  // lanes >= 16 hold sum(b)
}

// sum over the 32 lanes of four values at once (10 shuffles): halve the
// value set at xor 16 and xor 8, finish one value per 8-lane group, gather
__device__ __forceinline__ void warp_sum4(float (&v)[4]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8;
  float k0 = b4 ? v[2] : v[0], k1 = b4 ? v[3] : v[1];
  const float s0 = b4 ? v[0] : v[2], s1 = b4 ? v[1] : v[3];
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  float k = b3 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  // lane L now holds the sum of value (L >> 3) & 3: gather all four
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = __shfl_sync(0xffffffffu, k, q << 3);
}

// warp_sum4 without the final gather: lane L returns the sum of value
// (L >> 3) & 3 (5 shuffles + 1 select) -- for per-system scalar work done
// once per system by its 8 owner lanes instead of by all 32 lanes per system
__device__ __forceinline__ float warp_sum4_owned(const float (&v)[4]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8;
  float k0 = b4 ? v[2] : v[0], k1 = b4 ? v[3] : v[1];
  const float s0 = b4 ? v[0] : v[2], s1 = b4 ? v[1] : v[3];
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  float k = b3 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
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

// The approximate-tracker pairs path with ONE reduction phase per CG
// iteration (Chronopoulos-Gear): besides p and r the warp carries w = A r
// and s = A p (s = w + beta s, so the matvec runs on r), and the two inner
// products of an iteration, ||r||^2 and Re r^H w, are reduced together for
// both systems (warp_sum4: one 10-shuffle butterfly where the two-phase
// form needs two).  The curvature p^H A p is the recurrence
// delta - beta gamma / alpha_prev (k = 1: delta).  Same decisions as
// solvers.cpp:21-72 -- freeze (||r||^2 <= 1e-28 ||r_0||^2: alpha = 1,
// beta = 0, no update), breakdown (curvature < 1e-30) -- and once an
// iteration does not update, none after it does, so beta of a non-updating
// iteration is 0 as in the reference.  The approximate tracker consumes
// alpha_k, beta_{k-1}, beta_{k-2} in the same order (detect.cpp:409-427).
__device__ __forceinline__ void rows32_pair_cg1(const KernelParams& p, long sc, const float2* mfsrc,
                                                int base, const unsigned long long (&grow)[32],
                                                float gdiag, float2* Ps) {
  constexpr int UP = 32, NS = 2;
  const int S = p.S, U = p.U, K = p.K;
  const int lane = threadIdx.x & 31;
  const float reg = p.rho_inv_u;
  bool live[NS], broke[NS], updp[NS];
  float gam[NS], gam0[NS], alp[NS];
  float2 v[NS], r[NS], pp[NS], sv[NS], w[NS];
  float f0[NS], f1[NS], f2[NS], ia1[NS], ia2[NS], bm1[NS], bm2[NS];
  // w = (G + reg I) x for the NS broadcast rows in Ps
  auto matvec = [&](const float2 (&x)[NS], float2 (&o)[NS]) {
    unsigned long long a0[NS], b0[NS], a1[NS], b1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a0[s] = b0[s] = a1[s] = b1[s] = 0ull;
#pragma unroll
    for (int j = 0; j < UP; j += 2) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj = *reinterpret_cast<const ulonglong2*>(Ps + s * UP + j);
        ffma2(a0[s], grow[j], f2dup_lo(pj.x));
        ffma2(b0[s], grow[j], f2dup_hi(pj.x));
        ffma2(a1[s], grow[j + 1], f2dup_lo(pj.y));
        ffma2(b1[s], grow[j + 1], f2dup_hi(pj.y));
      }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float2 A0 = f2unpack(a0[s]), B0 = f2unpack(b0[s]);
      const float2 A1 = f2unpack(a1[s]), B1 = f2unpack(b1[s]);
      o[s].x = fmaf(reg, x[s].x, (A0.x - B0.y) + (A1.x - B1.y));
      o[s].y = fmaf(reg, x[s].y, (B0.x + A0.y) + (B1.x + A1.y));
    }
  };
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    live[s] = base + s < S;
    float2 b = make_float2(0.f, 0.f);
    if (live[s] && lane < U) b = mfsrc[(base + s) * UP + lane];
    v[s] = pp[s] = sv[s] = make_float2(0.f, 0.f);
    r[s] = b;
    Ps[s * UP + lane] = b;
    broke[s] = false;
    updp[s] = true;
    alp[s] = 1.f;
    ia1[s] = ia2[s] = 1.f;
    bm1[s] = bm2[s] = 0.f;
    f0[s] = f1[s] = f2[s] = 0.f;
  }
  __syncwarp();
  matvec(r, w);  // w_0 = A r_0
  float red[4] = {cnorm(r[0]), r[0].x * w[0].x + r[0].y * w[0].y, cnorm(r[1]),
                  r[1].x * w[1].x + r[1].y * w[1].y};
  warp_sum4(red);
  float dlt[NS] = {red[1], red[3]};
  gam[0] = gam0[0] = red[0];
  gam[1] = gam0[1] = red[2];
  float gold[NS] = {1.f, 1.f};
  for (int k = 1; k <= K; ++k) {
    float alpha[NS], beta[NS];
    bool upd[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      // beta_{k-1} of the reference (0 when iteration k-1 did not update)
      beta[s] = (k > 1 && updp[s]) ? __fdividef(gam[s], gold[s]) : 0.f;
      const bool frozen = !(gam[s] > 1e-28f * gam0[s]);  // solvers.cpp:21,25-27
      const bool go = live[s] && updp[s] && !frozen && !broke[s];
      const float curv = k == 1 ? dlt[s] : dlt[s] - beta[s] * gam[s] * __fdividef(1.f, alp[s]);
      if (go && curv < 1e-30f) broke[s] = true;  // solvers.cpp:55-57
      upd[s] = go && !broke[s];
      alpha[s] = upd[s] ? __fdividef(gam[s], curv) : 1.f;
      // tracker bookkeeping: the previous iteration's beta, then Eq. (11)
      bm2[s] = bm1[s];
      bm1[s] = k > 1 ? beta[s] : 0.f;
      if (live[s]) {
        const float c1 = alpha[s] * (1.f + bm1[s]) * ia1[s];
        const float c2 = alpha[s] * bm2[s] * ia2[s];
        const float nk = f0[s] + (c1 - alpha[s] * (gdiag + reg)) * (f0[s] - f1[s]) -
                         c2 * (f1[s] - f2[s]);
        const float nf = k == 1 ? alpha[s] : nk;
        f2[s] = f1[s];
        f1[s] = f0[s];
        f0[s] = nf;
      }
      ia2[s] = ia1[s];
      ia1[s] = upd[s] ? __fdividef(1.f, alpha[s]) : 1.f;
      if (upd[s]) {
        pp[s].x = fmaf(beta[s], pp[s].x, r[s].x);
        pp[s].y = fmaf(beta[s], pp[s].y, r[s].y);
        sv[s].x = fmaf(beta[s], sv[s].x, w[s].x);
        sv[s].y = fmaf(beta[s], sv[s].y, w[s].y);
        v[s].x = fmaf(alpha[s], pp[s].x, v[s].x);
        v[s].y = fmaf(alpha[s], pp[s].y, v[s].y);
        r[s].x = fmaf(-alpha[s], sv[s].x, r[s].x);
        r[s].y = fmaf(-alpha[s], sv[s].y, r[s].y);
        alp[s] = alpha[s];
      }
      updp[s] = upd[s];
    }
    if (k == K) break;
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s) Ps[s * UP + lane] = r[s];
    __syncwarp();
    matvec(r, w);
    float rd[4] = {cnorm(r[0]), r[0].x * w[0].x + r[0].y * w[0].y, cnorm(r[1]),
                   r[1].x * w[1].x + r[1].y * w[1].y};
    warp_sum4(rd);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      gold[s] = gam[s];
      gam[s] = rd[2 * s];
      dlt[s] = rd[2 * s + 1];
    }
  }
  // outputs: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (!live[s] || lane >= U) continue;
    const long o = (sc * S + base + s) * static_cast<long>(U) + lane;
    const bool ok = !broke[s];
    const float2 xh = ok ? v[s] : make_float2(0.f, 0.f);
    const float mu_u = ok ? f0[s] * gdiag : 0.f;
    const float rho_u = ok ? gdiag / p.n0 : 0.f;
    if (p.xhat) p.xhat[o] = xh;
    if (p.mu) p.mu[o] = mu_u;
    if (p.rho) p.rho[o] = rho_u;
    if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
    if (p.status && lane == 0) p.status[sc * S + base + s] = ok ? 0 : 1;
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
  W.plan(UP, S, p.K, EXACT, p.fx, p.zs);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
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
    moments_tail<UP>(p, ws, W, sc, Kmax, hist, Vs, sys_st, nt,
                     reinterpret_cast<double*>(smem + L.msh));
  }
  if (St > 0) {
    sync();
    k2_precode_tail<UP>(p, sc, Vs, Qs, gpart, sys_st, nt, sync);
  }
}


// Uplink only (St = 0): one warp per (subcarrier, NS systems) work item, so
// the grid is many short warps that the hardware scheduler balances (a CTA
// per subcarrier at 16 warps / SM leaves a 1.01-wave tail on cfg2's 1200
// subcarriers).  Each warp reads its G row straight from the L2-resident
// workspace.  Approximate tracker: the outputs leave from rows32_pair.
// Exact tracker: the (alpha, beta) history stays in the warp's shared slot
// and the extraction runs in the warp from the subcarrier's row-moment
// table (moments_coefs / moments_row, cgm_moments.cuh: O(K^2 + K) per
// lane), then the LLRs.
template <bool EXACT, int NS>
__global__ void __launch_bounds__(128, NS == 1 ? 5 : 4) solve_rows32_pairs_kernel(const KernelParams p) {
  constexpr int UP = 32, NW = 4;
  __shared__ __align__(16) float2 Ps_all[NW][NS * UP];
  __shared__ __align__(16) float2 Vs_all[EXACT ? NW : 1][NS * UP];
  __shared__ float hist_all[EXACT ? NW : 1][NS * kMaxK * 2];
  __shared__ double msh_all[EXACT ? NW : 1][kMomScratch];
  __shared__ uint8_t st_all[EXACT ? NW : 1][NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.S, U = p.U, K = p.K;
  const int npairs = (S + NS - 1) / NS;
  const long item = static_cast<long>(blockIdx.x) * NW + warp;
  if (item >= p.n_sc * npairs) return;
  const long lsc = item / npairs;
  const int base = static_cast<int>(item - lsc * npairs) * NS;
  const long sc = p.sc_base + lsc;
  WsOffsets W;
  W.plan(UP, S, K, EXACT, p.fx, p.zs);
  const float2* ws = p.ws + lsc * W.stride;
  unsigned long long grow[UP];
#pragma unroll
  for (int j = 0; j < UP; ++j) {
    const float2 g = __ldg(ws + W.g + j * UP + lane);
    grow[j] = f2pack(g.x, -g.y);
  }
  const float gdiag = __ldg(ws + W.g + lane * UP + lane).x;
  if constexpr (!EXACT) {
    if constexpr (NS == 2)
      rows32_pair_cg1(p, sc, ws + W.mf, base, grow, gdiag, Ps_all[warp]);
    else
      rows32_pair<false, true, NS>(p, sc, ws + W.mf, base, grow, gdiag, Ps_all[warp], nullptr,
                                   nullptr, nullptr);
  } else {
    const int w = warp;
    // per-warp arrays indexed by the subcarrier-wide system number
    rows32_pair<true, true, NS>(p, sc, ws + W.mf, base, grow, gdiag, Ps_all[warp],
                                hist_all[w] - base * K * 2, Vs_all[w] - base * UP, st_all[w] - base);
    __syncwarp();
    if (p.fx) {  // S = 1: moments_kernel<..., FX> finishes from the workspace
      fx_handoff<UP>(p, const_cast<float2*>(ws), W, sc, hist_all[w], K, Vs_all[w], st_all[w][0],
                     lane, 32);
      return;
    }
    const float2 cdv = ws[W.cd];
    const double* mom = reinterpret_cast<const double*>(ws + W.t);
#pragma unroll 1
    for (int t = 0; t < NS; ++t) {
      const int sy = base + t;
      if (sy >= S) break;
      const MomCoef c = moments_coefs(hist_all[w] + t * K * 2, K, cdv.x, cdv.y, p.rho_inv_u,
                                      msh_all[w]);
      float mu, rho;
      moments_row(msh_all[w], c, K, mom, UP, lane, p.es, p.n0, mu, rho);
      const bool ok = st_all[w][t] == 0;
      const float2 xh = ok ? Vs_all[w][t * UP + lane] : make_float2(0.f, 0.f);
      if (!ok) mu = rho = 0.f;
      if (lane < U) {
        const long o = (sc * S + sy) * static_cast<long>(U) + lane;
        if (p.xhat) p.xhat[o] = xh;
        if (p.mu) p.mu[o] = mu;
        if (p.rho) p.rho[o] = rho;
        if (p.llr) store_llrs_fast(xh, mu, rho, p.bits, p.llr + o * p.bits);
      }
      if (p.status && lane == 0) p.status[sc * S + sy] = ok ? 0 : 1;
      __syncwarp();  // msh is reused by the next system
    }
  }
}

}  // namespace cgm
