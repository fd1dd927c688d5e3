// cgm_kernels.cuh -- the fused per-subcarrier kernel (sm_100a).
//
// One CTA owns one subcarrier at a time (grid-stride "persistent" loop over
// subcarriers).  Everything that depends only on the channel -- the Gram
// matrix G = H^H H and, for the exact tracker, the Chebyshev basis
// T_m(Ahat) -- is built ONCE per subcarrier in shared memory and reused by
// all S received vectors (uplink) and all S_t transmit vectors (downlink)
// that share the channel.  Replaces, per instance:
//
//   gram_regularized          linalg.cpp:59-101      -> phase 1 (tiles)
//   matvec_adjoint (MF)       linalg.cpp:116-126     -> phase 1 (tiles)
//   cg_solve / cg_core        solvers.cpp:37-72      -> phase 2 (one lane group per system)
//   ApproxSinrTracker         detect.cpp:397-441     -> phase 2 (per lane)
//   ExactSinrTracker + extract detect.cpp:330-395    -> phase 3 (shared basis)
//   compute_llrs              detect.cpp:57-86       -> phase 4
//   precode_cg + normalize    precode.cpp:22-71      -> phases 2 + 5
//
// Exact tracker (Eq. 10): L_k is a real-coefficient polynomial in A, so we run
// the reference's three-term recursion (detect.cpp:350-358) on the polynomial
// COEFFICIENTS (O(K^2) per system) in the Chebyshev basis T_m(Ahat),
// Ahat = (A - cI)/d, and evaluate L_K and B = L_K G from the shared basis.
// The U^3 work is (K-1) Hermitian products per SUBCARRIER instead of K per
// vector; the monomial basis is avoided because it loses ~1e-3 at K = 8 in
// FP32.
#pragma once

#include "cgm_device.cuh"

namespace cgm {

constexpr int kMaxK = 16;        // CG iterations supported by the exact tracker
constexpr int kMaxSys = 64;      // systems (uplink + downlink vectors) per subcarrier

struct KernelParams {
  // inputs
  const float2* H;      // uplink layout [n_sc][B][U] or downlink [n_sc][U][B]
  const float2* Y;      // [n_sc][S][B] (uplink vectors), may be null when S == 0
  const float2* T;      // [n_sc][St][U] (downlink vectors), may be null when St == 0
  // uplink outputs ([n_sc][S][U] ...), each may be null
  float2* xhat;
  float* mu;
  float* rho;
  float* llr;           // [n_sc][S][U][bits]
  uint8_t* status;      // [n_sc][S]
  // downlink outputs
  float2* q;            // [n_sc][St][B]
  float2* s_out;        // [n_sc][St][B]
  float* gain;          // [n_sc][St]
  uint8_t* pstatus;     // [n_sc][St]
  float* tscratch;      // per-CTA Chebyshev basis when it does not fit in smem
  long n_sc;
  int B, U, S, St, K, Kt, bits;
  int hd_layout;        // 1: H is the downlink matrix [U][B] (precode only)
  int exact;            // uplink tracker: 1 exact (Eq. 10), 0 approx (Eq. 11)
  int use_tma;          // 1: bulk-copy staging (U == UP, B even, aligned)
  int t_in_smem;        // Chebyshev basis in shared memory
  float rho_inv_u, rho_inv_d, n0, es;
};

// Per-axis Gray amplitude subsets (constellation.cpp:75-84), filled by the
// host from the same closed form: [bits/2 - 1 index by qam][p][k].
struct AxisTables {
  float a0[3][3][4];  // [qam: 0=qpsk,1=16,2=64][p][k]
  float a1[3][3][4];
};
__constant__ AxisTables c_axis;

// ----------------------------------------------------------------- layout
template <int UP>
struct Smem {
  // byte offsets into dynamic shared memory
  int bar, hs, ys, gs, rhs, ps, vs, hist, sys_st, mu, rho, coef, tb, qs, red, total;
  int ldy;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int St, int K, int exact, int t_in_smem,
                                int red_floats, int nwarps) {
    const int nsys = S + St;
    ldy = B + 2;
    int o = 0;
    bar = o; o = align(o + 16);
    hs = o; o = align(o + B * UP * 8);
    ys = o; o = align(o + S * ldy * 8);
    gs = o; o = align(o + UP * UP * 8);
    rhs = o; o = align(o + nsys * UP * 8);
    ps = o; o = align(o + nsys * UP * 8);
    vs = o; o = align(o + nsys * UP * 8);
    hist = o; o = align(o + nsys * K * 2 * 4);
    sys_st = o; o = align(o + nsys);
    mu = o; o = align(o + S * UP * 4);
    rho = o; o = align(o + S * UP * 4);
    coef = o; o = align(o + (exact ? S * 2 * (K + 2) * 4 : 0) + 64);
    tb = o; o = align(o + ((exact && t_in_smem) ? K * UP * UP * 8 : 0));
    qs = o; o = align(o + (St < nwarps ? St : nwarps) * B * 8);
    red = o; o = align(o + (red_floats + 4) * 4);
    total = o;
  }
};

// Tile schedule of the phase-1 contraction: Gram lower-triangle 4x4 blocks
// followed by matched-filter 4x4 blocks (users x uplink vectors).
template <int UP, int NT>
struct GramPlan {
  int n_gram, n_mf, n_tiles, n_split, klen;
  __host__ __device__ void plan(int B, int S) {
    const int nb = UP / 4;
    n_gram = nb * (nb + 1) / 2;
    n_mf = nb * ((S + 3) / 4);
    n_tiles = n_gram + n_mf;
    n_split = n_tiles >= NT ? 1 : NT / n_tiles;
    int cap = B / 8 > 0 ? B / 8 : 1;
    if (n_split > cap) n_split = cap;
    klen = (B + n_split - 1) / n_split;
  }
  __host__ __device__ int red_floats() const { return (n_split - 1) * n_tiles * 32; }
};

template <int UP, int NT>
struct ChebPlan {
  int n_tiles, n_split, klen;
  __host__ __device__ void plan() {
    const int nb = UP / 4;
    n_tiles = nb * (nb + 1) / 2;
    n_split = n_tiles >= NT ? 1 : NT / n_tiles;
    int cap = UP / 4;
    if (n_split > cap) n_split = cap;
    klen = (UP + n_split - 1) / n_split;
  }
  __host__ __device__ int red_floats() const { return (n_split - 1) * n_tiles * 32; }
};

__device__ __forceinline__ void tri_block(int t, int& ib, int& jb) {
  // t -> (ib, jb) with jb <= ib, row-major over the lower triangle
  ib = static_cast<int>((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
  while ((ib + 1) * (ib + 2) / 2 <= t) ++ib;
  while (ib * (ib + 1) / 2 > t) --ib;
  jb = t - ib * (ib + 1) / 2;
}

// Deterministic split-K reduction: splits 1.. park partial tiles in `red`,
// split 0 adds them in split order.  Returns true on the thread that owns
// the final tile value in acc.
__device__ __forceinline__ bool split_reduce(float2 (&acc)[4][4], float* red, int tile, int split,
                                             int n_split, int n_tiles, bool active) {
  if (n_split == 1) return active;
  float2* r2 = reinterpret_cast<float2*>(red);
  if (active && split > 0) {
    float2* dst = r2 + ((split - 1) * n_tiles + tile) * 16;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[r * 4 + c] = acc[r][c];
  }
  __syncthreads();
  if (active && split == 0) {
    for (int sp = 1; sp < n_split; ++sp) {
      const float2* src = r2 + ((sp - 1) * n_tiles + tile) * 16;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = cadd(acc[r][c], src[r * 4 + c]);
    }
    return true;
  }
  return false;
}

// ------------------------------------------------------------------ LLR
// Max-log LLRs of one user (detect.cpp:68-86), written to out[0..bits).
__device__ __forceinline__ float axis_min_sq(float z, const float* amps, int n) {
  float best = INFINITY;
  for (int k = 0; k < n; ++k) {
    const float d = z - amps[k];
    best = fminf(best, d * d);
  }
  return best;
}

__device__ __forceinline__ void store_llrs(float2 xh, float mu, float rho, int bits, float* out) {
  const int half = bits >> 1, q = half - 1, per = 1 << (half - 1);
  float v[6];
  if (fabsf(mu) < 1e-12f) {
#pragma unroll
    for (int b = 0; b < 6; ++b) v[b] = 0.f;
  } else {
    if (rho < 0.f) rho = 0.f;
    const float inv = 1.0f / mu;
    const float zr = xh.x * inv, zi = xh.y * inv;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      if (p < half) {
        const float d0r = axis_min_sq(zr, c_axis.a0[q][p], per);
        const float d1r = axis_min_sq(zr, c_axis.a1[q][p], per);
        const float d0i = axis_min_sq(zi, c_axis.a0[q][p], per);
        const float d1i = axis_min_sq(zi, c_axis.a1[q][p], per);
        v[p] = fminf(64.f, fmaxf(-64.f, rho * (d0r - d1r)));
        v[half + p] = fminf(64.f, fmaxf(-64.f, rho * (d0i - d1i)));
      }
    }
  }
  for (int b = 0; b < bits; ++b) out[b] = v[b];
}

// ------------------------------------------------------------------ kernel
template <int UP, int NT>
__global__ void __launch_bounds__(NT) subcarrier_kernel(const KernelParams p) {
  constexpr int G = UP < 32 ? UP : 32;  // lanes per CG system
  constexpr int RU = UP / G;            // rows per lane
  constexpr int NGRP = NT / G;          // concurrent systems per CTA
  extern __shared__ __align__(128) unsigned char smem[];

  Smem<UP> L;
  GramPlan<UP, NT> gp;
  gp.plan(p.B, p.S);
  ChebPlan<UP, NT> cp;
  cp.plan();
  const int red_floats = max(gp.red_floats(), cp.red_floats());
  L.plan(p.B, p.S, p.St, p.K > p.Kt ? p.K : p.Kt, p.exact, p.t_in_smem, red_floats, NT / 32);
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Hs = reinterpret_cast<float2*>(smem + L.hs);
  float2* Ys = reinterpret_cast<float2*>(smem + L.ys);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  float2* Rs = reinterpret_cast<float2*>(smem + L.rhs);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* MUs = reinterpret_cast<float*>(smem + L.mu);
  float* RHOs = reinterpret_cast<float*>(smem + L.rho);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  float* red = reinterpret_cast<float*>(smem + L.red);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float2* Tb = p.t_in_smem ? reinterpret_cast<float2*>(smem + L.tb)
                           : reinterpret_cast<float2*>(p.tscratch) +
                                 static_cast<long>(blockIdx.x) * Kmax * UP * UP;

  const int tid = threadIdx.x;
  const int B = p.B, S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;

  if (p.use_tma && tid == 0) mbar_init(bar, 1);
  __syncthreads();

  uint32_t phase = 0;
  for (long sc = blockIdx.x; sc < p.n_sc; sc += gridDim.x, phase ^= 1u) {
    // ------------------------------------------------ phase 0: stage inputs
    if (p.use_tma) {
      if (tid == 0) {
        const uint32_t hbytes = static_cast<uint32_t>(B) * UP * 8u;
        const uint32_t ybytes = static_cast<uint32_t>(B) * 8u;
        fence_proxy_async();
        mbar_expect_tx(bar, hbytes + ybytes * S);
        bulk_g2s(Hs, p.H + sc * static_cast<long>(B) * UP, hbytes, bar);
        for (int s = 0; s < S; ++s)
          bulk_g2s(Ys + s * L.ldy, p.Y + (sc * S + s) * static_cast<long>(B), ybytes, bar);
      }
    } else {
      if (p.hd_layout) {
        // downlink H_d [U][B] -> Hs[b][u] = conj(H_d[u][b]) (= H_u = H_d^H)
        const float2* src = p.H + sc * static_cast<long>(U) * B;
        for (int e = tid; e < UP * B; e += NT) {
          const int u = e / B, b = e - u * B;
          Hs[b * UP + u] = u < U ? cconj(src[u * B + b]) : make_float2(0.f, 0.f);
        }
      } else {
        const float2* src = p.H + sc * static_cast<long>(B) * U;
        for (int e = tid; e < UP * B; e += NT) {
          const int b = e / UP, u = e - b * UP;
          Hs[e] = u < U ? src[b * U + u] : make_float2(0.f, 0.f);
        }
      }
      for (int e = tid; e < S * B; e += NT) {
        const int s = e / B, b = e - s * B;
        Ys[s * L.ldy + b] = p.Y[(sc * S + s) * static_cast<long>(B) + b];
      }
    }
    // downlink right-hand sides t (precode.cpp:64: CG starts from b = t)
    for (int e = tid; e < St * UP; e += NT) {
      const int s = e / UP, u = e - s * UP;
      Rs[(S + s) * UP + u] =
          u < U ? p.T[(sc * St + s) * static_cast<long>(U) + u] : make_float2(0.f, 0.f);
    }
    if (p.use_tma) mbar_wait(bar, phase);
    __syncthreads();

    // ------------------------------------- phase 1: Gram + matched filter
    {
      const int split = tid / gp.n_tiles;
      const int tile = tid - split * gp.n_tiles;
      for (int t0 = 0; t0 < gp.n_tiles; t0 += NT) {
        const int my_tile = gp.n_split == 1 ? t0 + tid : tile;
        const bool active = gp.n_split == 1 ? my_tile < gp.n_tiles : split < gp.n_split;
        float2 acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
        int ib = 0, jb = 0;
        const bool is_gram = my_tile < gp.n_gram;
        if (active) {
          const int k0 = gp.n_split == 1 ? 0 : split * gp.klen;
          const int k1 = min(B, k0 + (gp.n_split == 1 ? B : gp.klen));
          if (is_gram) {
            tri_block(my_tile, ib, jb);
            tile4x4<true>(acc, Hs, UP, ib * 4, Hs, UP, 1, jb * 4, UP, k0, k1);
          } else {
            const int m = my_tile - gp.n_gram;
            const int nsb = (S + 3) / 4;
            ib = m / nsb;
            jb = m - ib * nsb;
            tile4x4<false>(acc, Hs, UP, ib * 4, Ys, 1, L.ldy, jb * 4, S, k0, k1);
          }
        }
        const bool owner = split_reduce(acc, red, my_tile, gp.n_split == 1 ? 0 : split,
                                        gp.n_split, gp.n_tiles, active);
        if (owner) {
          if (is_gram) {
            // one triangle + conjugate mirror: G == G^H exactly (linalg.hpp:42-52)
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int i = ib * 4 + r, j = jb * 4 + c;
                if (j < i) {
                  Gs[i * UP + j] = acc[r][c];
                  Gs[j * UP + i] = cconj(acc[r][c]);
                } else if (j == i) {
                  Gs[i * UP + i] = make_float2(acc[r][c].x, 0.f);
                }
              }
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int s = jb * 4 + c;
                if (s < S) Rs[s * UP + ib * 4 + r] = acc[r][c];
              }
          }
        }
        if (gp.n_split > 1) break;  // all tiles covered in one round
      }
    }
    __syncthreads();

    // --------------------------------------------- phase 2: CG per system
    {
      const int grp = tid / G, gl = tid - grp * G;
      float2 grow[UP <= 32 ? UP : 1];
      if constexpr (RU == 1) {
        // row gl of G (read as column: G[j][gl] = conj(G[gl][j]))
#pragma unroll
        for (int j = 0; j < UP; ++j) grow[j] = cconj(Gs[j * UP + gl]);
      }
      for (int base = 0; base < nsys; base += NGRP) {
        const int sys = base + grp;
        const bool live = sys < nsys;
        const bool down = sys >= S;
        const int iters = down ? p.Kt : p.K;
        const float reg = down ? p.rho_inv_d : p.rho_inv_u;
        float2 b[RU], v[RU], r[RU], pp[RU], e[RU];
        float gdiag[RU];
#pragma unroll
        for (int m = 0; m < RU; ++m) {
          const int u = gl + m * G;
          b[m] = live ? Rs[sys * UP + u] : make_float2(0.f, 0.f);
          v[m] = make_float2(0.f, 0.f);
          r[m] = b[m];
          pp[m] = b[m];
          gdiag[m] = Gs[u * UP + u].x;
          if (live) Ps[sys * UP + u] = pp[m];
        }
        float rn = 0.f;
#pragma unroll
        for (int m = 0; m < RU; ++m) rn += cnorm(r[m]);
        rn = group_sum<G>(rn);
        const float rn0 = rn;
        // approximate tracker state (detect.cpp:400-433), histories alpha=1, beta=0
        float f0[RU], f1[RU], f2[RU];
#pragma unroll
        for (int m = 0; m < RU; ++m) f0[m] = f1[m] = f2[m] = 0.f;
        float am1 = 1.f, am2 = 1.f, bm1 = 0.f, bm2 = 0.f;
        bool broke = false;
        __syncwarp();
        const int kmax = nsys > 0 ? Kmax : 0;
        for (int k = 1; k <= kmax; ++k) {
          const bool step = live && k <= iters;
          const bool frozen = !(rn > 1e-28f * rn0);  // solvers.cpp:21,25-27
          float alpha = 1.f, beta = 0.f;
          // e = (G + reg I) p   (uniform control flow across the warp)
#pragma unroll
          for (int m = 0; m < RU; ++m) e[m] = make_float2(0.f, 0.f);
          if constexpr (RU == 1) {
            const float2* prow = Ps + (live ? sys : 0) * UP;
#pragma unroll
            for (int j = 0; j < UP; j += 2) {
              const float4 pj = *reinterpret_cast<const float4*>(prow + j);
              cfma(e[0], grow[j], make_float2(pj.x, pj.y));
              cfma(e[0], grow[j + 1], make_float2(pj.z, pj.w));
            }
          } else {
            const float2* prow = Ps + (live ? sys : 0) * UP;
            for (int j = 0; j < UP; j += 2) {
              const float4 pj = *reinterpret_cast<const float4*>(prow + j);
#pragma unroll
              for (int m = 0; m < RU; ++m) {
                const int u = gl + m * G;
                cfma(e[m], cconj(Gs[j * UP + u]), make_float2(pj.x, pj.y));
                cfma(e[m], cconj(Gs[(j + 1) * UP + u]), make_float2(pj.z, pj.w));
              }
            }
          }
          float curv = 0.f;
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            e[m].x = fmaf(reg, pp[m].x, e[m].x);
            e[m].y = fmaf(reg, pp[m].y, e[m].y);
            curv += pp[m].x * e[m].x + pp[m].y * e[m].y;  // Re p^H e
          }
          curv = group_sum<G>(curv);
          const bool go = step && !frozen && !broke;
          if (go && curv < 1e-30f) broke = true;  // solvers.cpp:55-57
          const bool upd = go && !broke;
          float rn_next = 0.f;
          if (upd) alpha = rn / curv;
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            if (upd) {
              v[m].x = fmaf(alpha, pp[m].x, v[m].x);
              v[m].y = fmaf(alpha, pp[m].y, v[m].y);
              r[m].x = fmaf(-alpha, e[m].x, r[m].x);
              r[m].y = fmaf(-alpha, e[m].y, r[m].y);
            }
            rn_next += cnorm(r[m]);
          }
          rn_next = group_sum<G>(rn_next);
          if (upd) {
            beta = rn_next / rn;
            rn = rn_next;
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              pp[m].x = fmaf(beta, pp[m].x, r[m].x);
              pp[m].y = fmaf(beta, pp[m].y, r[m].y);
            }
          }
          __syncwarp();
          if (upd) {
#pragma unroll
            for (int m = 0; m < RU; ++m) Ps[sys * UP + gl + m * G] = pp[m];
          }
          __syncwarp();
          if (step) {
            if (gl == 0 && !down && p.exact) {
              hist[(sys * Kmax + (k - 1)) * 2 + 0] = alpha;
              hist[(sys * Kmax + (k - 1)) * 2 + 1] = beta;
            }
            if (!down && !p.exact) {
              // Eq. (11) on the diagonal (detect.cpp:409-427)
#pragma unroll
              for (int m = 0; m < RU; ++m) {
                float nf;
                if (k == 1) {
                  nf = alpha;
                } else {
                  const float c1 = alpha * (1.f + bm1) / am1;
                  const float c2 = alpha * bm2 / am2;
                  const float d1 = f0[m] - f1[m], d2 = f1[m] - f2[m];
                  nf = f0[m] + (c1 - alpha * (gdiag[m] + reg)) * d1 - c2 * d2;
                }
                f2[m] = f1[m];
                f1[m] = f0[m];
                f0[m] = nf;
              }
            }
            am2 = am1; am1 = alpha; bm2 = bm1; bm1 = beta;
          }
        }
        if (live) {
#pragma unroll
          for (int m = 0; m < RU; ++m) Vs[sys * UP + gl + m * G] = v[m];
          if (gl == 0) sys_st[sys] = broke ? 1 : 0;
          if (!down && !p.exact) {
            // detect.cpp:435-441: mu = Ltilde * G_ii, rho = G_ii / N0
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              const int u = gl + m * G;
              MUs[sys * UP + u] = f0[m] * gdiag[m];
              RHOs[sys * UP + u] = gdiag[m] / p.n0;
            }
          }
        }
      }
    }
    __syncthreads();

    // ------------------------------- phase 3: exact tracker, shared basis
    if (p.exact && S > 0) {
      const int K = p.K;
      // centre / half-width of the spectrum of A = G + rho_u^-1 I
      float* cd = red + red_floats;  // 2 floats after the split-K scratch
      if (tid < 32) {
        float tr = 0.f, fr = 0.f;
        for (int i = tid; i < UP; i += 32) tr += Gs[i * UP + i].x + p.rho_inv_u;
        tr = group_sum<32>(tr);
        const float c = tr / UP;
        for (int e = tid; e < UP * UP; e += 32) {
          const int i = e / UP, j = e - i * UP;
          float2 a = Gs[e];
          if (i == j) a.x += p.rho_inv_u - c;
          fr += cnorm(a);
        }
        fr = group_sum<32>(fr);
        float d = 2.f * sqrtf(fr / UP);
        if (!(d > 1e-6f * fmaxf(fabsf(c), 1e-30f))) d = fmaxf(fabsf(c), 1.f);
        if (tid == 0) { cd[0] = c; cd[1] = d; }
      }
      __syncthreads();
      const float cc = cd[0], dd = cd[1];
      // T_1 = (A - cI)/d into Tb[0]
      const float invd = 1.f / dd;
      for (int e = tid; e < UP * UP; e += NT) {
        const int i = e / UP, j = e - i * UP;
        float2 a = Gs[e];
        if (i == j) a.x += p.rho_inv_u - cc;
        Tb[e] = cscale(invd, a);
      }
      // per-system coefficient recursion (thread per system), in FP64
      for (int s = tid; s < S; s += NT) {
        double l0[kMaxK + 2], l1[kMaxK + 2], l2[kMaxK + 2], tmp[kMaxK + 2], d1[kMaxK + 2];
        const int n = K + 2;
        for (int m = 0; m < n; ++m) l0[m] = l1[m] = l2[m] = 0.0;
        double am1 = 1.0, am2 = 1.0, bm1 = 0.0, bm2 = 0.0;
        auto mulA = [&](const double* x, double* out) {  // coefficients of A * poly
          for (int m = 0; m < n; ++m) out[m] = static_cast<double>(cc) * x[m];
          for (int m = 0; m < n; ++m) {
            if (x[m] == 0.0) continue;
            const double h = static_cast<double>(dd) * x[m];
            if (m == 0) {
              out[1] += h;
            } else {
              if (m + 1 < n) out[m + 1] += 0.5 * h;
              out[m - 1] += 0.5 * h;
            }
          }
        };
        for (int k = 1; k <= K; ++k) {
          const double a = hist[(s * Kmax + (k - 1)) * 2 + 0];
          const double bb = hist[(s * Kmax + (k - 1)) * 2 + 1];
          if (k == 1) {
            for (int m = 0; m < n; ++m) { l2[m] = l1[m]; l1[m] = l0[m]; l0[m] = 0.0; }
            l0[0] = a;  // L_1 = alpha_1 I (detect.cpp:342-347)
          } else {
            const double c1 = a * (1.0 + bm1) / am1, c2 = a * bm2 / am2;
            for (int m = 0; m < n; ++m) d1[m] = l0[m] - l1[m];
            mulA(d1, tmp);
            for (int m = 0; m < n; ++m) {
              const double nx = l0[m] + c1 * d1[m] - a * tmp[m] - c2 * (l1[m] - l2[m]);
              l2[m] = l1[m];
              l1[m] = l0[m];
              l0[m] = nx;
            }
          }
          am2 = am1; am1 = a; bm2 = bm1; bm1 = bb;
        }
        // B = L (A - rho^-1 I)  (G = unregularized A, detect.cpp:215)
        mulA(l0, tmp);
        float* cl = coef + s * 2 * (K + 2);
        float* cb = cl + (K + 2);
        for (int m = 0; m < n; ++m) {
          cl[m] = static_cast<float>(l0[m]);
          cb[m] = static_cast<float>(tmp[m] - static_cast<double>(p.rho_inv_u) * l0[m]);
        }
      }
      __syncthreads();
      // T_{m+1} = 2 T_1 T_m - T_{m-1}, m = 1..K-1 (lower tiles + mirror)
      for (int m = 1; m < K; ++m) {
        const float2* T1 = Tb;
        const float2* Tm = Tb + (m - 1) * UP * UP;
        float2* Tn = Tb + m * UP * UP;
        const float2* Tp = m >= 2 ? Tb + (m - 2) * UP * UP : nullptr;  // T_{m-1}; T_0 = I
        const int split = tid / cp.n_tiles;
        const int tile = tid - split * cp.n_tiles;
        for (int t0 = 0; t0 < cp.n_tiles; t0 += NT) {
          const int my_tile = cp.n_split == 1 ? t0 + tid : tile;
          const bool active = cp.n_split == 1 ? my_tile < cp.n_tiles : split < cp.n_split;
          float2 acc[4][4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
          int ib = 0, jb = 0;
          if (active) {
            tri_block(my_tile, ib, jb);
            const int k0 = cp.n_split == 1 ? 0 : split * cp.klen;
            const int k1 = min(UP, k0 + (cp.n_split == 1 ? UP : cp.klen));
            // (T1 Tm)_ij = sum_k conj(T1[k][i]) Tm[k][j]   (T1 Hermitian)
            tile4x4<true>(acc, T1, UP, ib * 4, Tm, UP, 1, jb * 4, UP, k0, k1);
          }
          const bool owner = split_reduce(acc, red, my_tile, cp.n_split == 1 ? 0 : split,
                                          cp.n_split, cp.n_tiles, active);
          if (owner) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int i = ib * 4 + r, j = jb * 4 + c;
                if (j > i) continue;
                float2 prev = Tp ? Tp[i * UP + j] : make_float2(i == j ? 1.f : 0.f, 0.f);
                float2 val = make_float2(2.f * acc[r][c].x - prev.x, 2.f * acc[r][c].y - prev.y);
                if (i == j) {
                  Tn[i * UP + i] = make_float2(val.x, 0.f);
                } else {
                  Tn[i * UP + j] = val;
                  Tn[j * UP + i] = cconj(val);
                }
              }
          }
          if (cp.n_split > 1) break;
        }
        __syncthreads();
      }
      // extraction (detect.cpp:375-395): thread <-> (row i, system subset)
      {
        constexpr int RG = NT / UP;  // row groups
        const int i = tid % UP, g = tid / UP;
        for (int s = g; s < S; s += RG) {
          if (sys_st[s]) continue;
          const float* cl = coef + s * 2 * (K + 2);
          const float* cb = cl + (K + 2);
          float ib2 = 0.f, ibl = 0.f, mu_i = 0.f;
          for (int j = 0; j < UP; ++j) {
            float2 Bij = make_float2(i == j ? cb[0] : 0.f, 0.f);
            float2 Lij = make_float2(i == j ? cl[0] : 0.f, 0.f);
            for (int m = 1; m <= K; ++m) {
              const float2 t = cconj(Tb[(m - 1) * UP * UP + j * UP + i]);  // T_m[i][j]
              Bij.x = fmaf(cb[m], t.x, Bij.x);
              Bij.y = fmaf(cb[m], t.y, Bij.y);
              if (m < K) {
                Lij.x = fmaf(cl[m], t.x, Lij.x);
                Lij.y = fmaf(cl[m], t.y, Lij.y);
              }
            }
            if (j == i) mu_i = Bij.x;
            else ib2 += cnorm(Bij);
            ibl += Bij.x * Lij.x + Bij.y * Lij.y;  // Re(B_ij conj(L_ij))
          }
          const float nu2 = ib2 * p.es + ibl * p.n0;
          MUs[s * UP + i] = mu_i;
          RHOs[s * UP + i] = nu2 <= 0.f ? 0.f : mu_i * mu_i / nu2;  // safe_rho (detect.cpp:26-29)
        }
      }
      __syncthreads();
    }

    // ------------------------------------------- phase 4: LLRs + stores
    for (int e = tid; e < S * U; e += NT) {
      const int s = e / U, u = e - s * U;
      const long o = (sc * S + s) * static_cast<long>(U) + u;
      const bool ok = sys_st[s] == 0;
      const float2 xh = ok ? Vs[s * UP + u] : make_float2(0.f, 0.f);
      const float m = ok ? MUs[s * UP + u] : 0.f;
      const float rr = ok ? RHOs[s * UP + u] : 0.f;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = m;
      if (p.rho) p.rho[o] = rr;
      if (p.llr) {
        float* out = p.llr + o * p.bits;
        if (ok) store_llrs(xh, m, rr, p.bits, out);
        else for (int b = 0; b < p.bits; ++b) out[b] = 0.f;
      }
    }
    if (p.status)
      for (int s = tid; s < S; s += NT) p.status[sc * S + s] = sys_st[s];

    // ------------------------------------- phase 5: precode q = H_d^H v
    // q_b = sum_u H_u[b][u] v_u (precode.cpp:69, linalg.cpp:116-126), then
    // gain = ||q||, s = q / gain, zero_input when ||q|| vanishes (:22-36).
    if (St > 0) {
      constexpr int NW = NT / 32;
      const int w = tid / 32, lane = tid & 31;
      float2* qb = Qs + w * B;
      for (int ts = w; ts < St; ts += NW) {
        const int sys = S + ts;
        const bool ok = sys_st[sys] == 0;
        const float2* vv = Vs + sys * UP;
        float nrm = 0.f;
        for (int b = lane; b < B; b += 32) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll 8
          for (int u0 = 0; u0 < UP; ++u0) {
            const int u = (u0 + lane) & (UP - 1);  // rotated: spreads smem banks
            cfma(acc, Hs[b * UP + u], vv[u]);
          }
          nrm += cnorm(acc);
          qb[b] = acc;
        }
        nrm = group_sum<32>(nrm);
        const float g = sqrtf(nrm);
        const bool zero = ok && !(g > 0.f);
        const float inv = (ok && !zero) ? 1.f / g : 0.f;
        const long ob = (sc * St + ts) * static_cast<long>(B);
        for (int b = lane; b < B; b += 32) {
          const float2 acc = qb[b];
          if (p.q) p.q[ob + b] = ok ? acc : make_float2(0.f, 0.f);
          if (p.s_out) p.s_out[ob + b] = cscale(inv, acc);
        }
        if (lane == 0) {
          if (p.gain) p.gain[sc * St + ts] = (ok && !zero) ? g : 0.f;
          if (p.pstatus) p.pstatus[sc * St + ts] = ok ? (zero ? 2 : 0) : 1;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

}  // namespace cgm
