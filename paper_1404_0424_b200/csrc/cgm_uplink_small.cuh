// cgm_uplink_small.cuh -- fused CG detector for small U (U <= 16): one warp
// per subcarrier does the whole of detect_cg (detect.cpp:182-237) for the S
// vectors sharing the channel, with no workspace and no second kernel.
//
//   0. H [B][U] and Y [B][S] staged by cp.async.bulk (read from HBM once);
//   1. G = H^H H (gram_regularized, linalg.cpp:59-101 without the rho^-1 I,
//      added in the CG): lower 4 x 4 tiles x antenna ranges on the packed
//      FFMA2 pipe, fixed-order partial sums, exact Hermitian mirror;
//   2. matched filters y_MF = H^H y (linalg.cpp:116-126), one lane per
//      (vector, user);
//   3. exact tracker only: the Chebyshev basis T_1..T_K of
//      Ahat = (A - cI)/d in shared memory (cheb_interval, then K - 1 U x U
//      products on the lanes);
//   4. K CG iterations per vector on UP-lane groups (solvers.cpp:37-72,
//      freeze / breakdown rules), the approximate tracker's Eq. (11)
//      recursion (detect.cpp:409-427) or the (alpha, beta) history;
//   5. exact: FP64 coefficient recursion on the basis (warp-parallel)
//      and the extraction of mu, nu^2, rho (detect.cpp:330-395); LLRs.
// The split path spends two launches and their per-subcarrier pipeline
// latency on a few kFLOP per subcarrier (cfg1: 1024 subcarriers, U = 8).
#pragma once

#include "cgm_rows32.cuh"  // f2dup_lo / f2dup_hi

namespace cgm {

template <int UP>
struct UpSmallGeo {
  static constexpr int NB = UP / 4;
  static constexpr int NTILE = NB * (NB + 1) / 2;
  static constexpr int KP = 32 / NTILE;  // antenna parts per tile (10 / 3)
  // Gram / matched-filter partials [part][tile entry | user], odd row stride:
  // the lanes of the fixed-order sums read consecutive words
  static constexpr int PSTR = (NTILE * 16 + UP) | 1;
  static constexpr int GL = UP;          // lanes per CG system
  static constexpr int GPW = 32 / GL;
};

struct UpSmallSmem {
  int bar, hs, ys, part, gs, tb, xs, ps, mfs, vs, hist, coef, st, total;
  __host__ __device__ static int align(int x) { return (x + 15) & ~15; }
  __host__ __device__ void plan(int UP, int B, int U, int S, int K, bool exact) {
    const int nb = UP / 4, ntile = nb * (nb + 1) / 2, kp = 32 / ntile;
    int o = 0;
    bar = o; o = align(o + 8);
    hs = o; o = align(o + B * U * 8);
    ys = o; o = align(o + B * S * 8);
    // the Gram partials are dead once G is summed, before the Chebyshev
    // basis is formed: the two share one region (more warps per SM)
    // (+ the matched-filter partials of the one-vector case: UP users x kp parts)
    const int part_b = ((ntile * 16 + UP) | 1) * kp * 8, tb_b = exact ? K * UP * UP * 8 : 0;
    const int pt_b = part_b > tb_b ? part_b : tb_b;
    // one vector per subcarrier: the matched filter rides on the Gram loop, so
    // H is dead too once the loop ends -- the partials and the basis then sit
    // on top of the H staging buffer (cfg1: 14.1 -> 10.3 KB per warp)
    if (S == 1 && pt_b <= B * U * 8) {
      part = hs; tb = hs;
    } else {
      part = o; tb = o; o = align(o + pt_b);
    }
    gs = o; o = align(o + UP * UP * 8);
    xs = o; o = align(o + UP * 8);
    ps = o; o = align(o + 32 * 8);
    mfs = o; o = align(o + S * UP * 8);
    vs = o; o = align(o + S * UP * 8);
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    coef = o; o = align(o + (exact ? S * 2 * (K + 2) * 4 : 0));
    st = o; o = align(o + S);
    total = o;
  }
};

// U <= 8 with one vector per subcarrier needs ~10 KB of shared memory per warp
// (cfg1), so registers bound the warps per SM.  Measured on 64 frames of cfg1:
// 128 registers (16 warps per SM) 0.305 ms, 120 (still 16 warps: warp
// allocation granularity) 0.322 ms, 104 (19 warps, spills in the Gram loop)
// 0.461 ms; the Gram loop unrolled by 2 at 128 registers 0.312 ms.
#ifndef CGM_US_UNR
#define CGM_US_UNR 1
#endif
constexpr int kUsUnroll = CGM_US_UNR;
#ifndef CGM_US_MAXR8
#define CGM_US_MAXR8 128
#endif

template <int UP, bool EXACT>
__global__ void __maxnreg__(UP == 8 ? CGM_US_MAXR8 : 128) uplink_small_kernel(const KernelParams p) {
  using UG = UpSmallGeo<UP>;
  constexpr int GL = UG::GL, GPW = UG::GPW, KP = UG::KP, PSTR = UG::PSTR;
  extern __shared__ __align__(128) unsigned char smem[];
  const int B = p.B, U = p.U, S = p.S, K = p.K;
  UpSmallSmem L;
  L.plan(UP, B, U, S, K, EXACT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Hs = reinterpret_cast<float2*>(smem + L.hs);
  float2* Ys = reinterpret_cast<float2*>(smem + L.ys);
  float2* P = reinterpret_cast<float2*>(smem + L.part);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  float2* Tb = reinterpret_cast<float2*>(smem + L.tb);
  float2* xs = reinterpret_cast<float2*>(smem + L.xs);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* MFs = reinterpret_cast<float2*>(smem + L.mfs);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.st);
  const int lane = threadIdx.x;
  const bool tma = p.use_tma != 0;
  if (tma && lane == 0) mbar_init(bar, 1);
  __syncwarp();

  // Gram work item: lower tile (rb, cb) x antenna range
  const int item_part = lane / UG::NTILE, item_tile = lane - item_part * UG::NTILE;
  const bool gram_busy = item_part < KP;
  int rb = 0;
  while ((rb + 1) * (rb + 2) / 2 <= item_tile) ++rb;
  const int cb = item_tile - rb * (rb + 1) / 2;
  // part p takes antennas p, p + KP, ...: at every step the parts read KP
  // consecutive rows of H, and each takes its 4 users in the order
  // (0 1 2 3) or (2 3 0 1) (rot2) -- for U = 8 (64-byte rows: two row phases
  // x two orders) and U = 16 (one phase) the 16-byte loads of a quarter
  // warp then fall in distinct banks, where contiguous antenna ranges with
  // the same user order were 3- to 4-way conflicts on every load of the
  // loop.  The accumulators hold the rotated order; the partials are stored
  // un-rotated.
  // (calls with U < UP keep the plain order: their row stride is not the
  // one the rotation is made for)
  const int rot2 = p.U != UP ? 0 : UP == 8 ? (item_part >> 1) & 1 : item_part & 1;
  const int unrot = rot2 * 10;  // (r, c) -> (r ^ 2, c ^ 2) on the index 4 r + c

  uint32_t phase = 0;
  for (long sc = blockIdx.x; sc < p.n_sc; sc += gridDim.x) {
    // ------------------------------------------------------------ 0. stage
    const float2* Hg = p.H + sc * static_cast<long>(B) * U;
    const float2* Yg = p.Y + sc * static_cast<long>(B) * S;
    if (tma) {
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(bar, static_cast<uint32_t>(B) * (U + S) * 8u);
        bulk_g2s(Hs, Hg, B * U * 8u, bar);
        bulk_g2s(Ys, Yg, B * S * 8u, bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      for (int e = lane; e < B * U; e += 32) Hs[e] = Hg[e];
      for (int e = lane; e < B * S; e += 32) Ys[e] = Yg[e];
      __syncwarp();
    }
    // ----------------------------------------------- 1. Gram partials (FFMA2)
    // acc[r][c] = sum_b conj(H[b][u]) H[b][v], u = 4rb + r, v = 4cb + c:
    // a += (y.x, y.y) * x.x, b += (y.x, y.y) * x.y; conj(x) y = (a.x + b.y, a.y - b.x)
    unsigned long long a[4][4], bb[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) a[r][c] = bb[r][c] = 0ull;
    // one vector per subcarrier: the matched filter of the tile's row users
    // rides on the same loads, conj(x) y = x.x (y.x, y.y) + x.y (y.y, -y.x)
    // (the diagonal tiles' lanes keep it; the separate pass below is skipped)
    unsigned long long mfa[4] = {0ull, 0ull, 0ull, 0ull};
    // one antenna row into the accumulators
    auto gram_mac = [&](const unsigned long long (&x)[4], const unsigned long long (&y)[4],
                        const float2 yb) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          ffma2(a[r][c], y[c], f2dup_lo(x[r]));
          ffma2(bb[r][c], y[c], f2dup_hi(x[r]));
        }
      if (S == 1) {
        const unsigned long long y1 = f2pack(yb.x, yb.y), y2 = f2pack(yb.y, -yb.x);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          ffma2(mfa[r], y1, f2dup_lo(x[r]));
          ffma2(mfa[r], y2, f2dup_hi(x[r]));
        }
      }
    };
    if (gram_busy && U == UP) {
      // full user count: constant row stride, the users in pairs by 16-byte
      // loads at [lane pointer + immediate], no bounds selects
      constexpr int RS = KP * UP / 2;  // ulonglong2 per step
      const ulonglong2* hx0 = reinterpret_cast<const ulonglong2*>(Hs + item_part * UP + rb * 4) + rot2;
      const ulonglong2* hx1 = hx0 + 1 - 2 * rot2;
      const ulonglong2* hy0 = reinterpret_cast<const ulonglong2*>(Hs + item_part * UP + cb * 4) + rot2;
      const ulonglong2* hy1 = hy0 + 1 - 2 * rot2;
      const float2* yp = Ys + item_part * S;
      const int nst = (B - item_part + KP - 1) / KP;
#pragma unroll(kUsUnroll)
      for (int t = 0; t < nst; ++t) {
        const ulonglong2 X0 = *hx0, X1 = *hx1, Y0 = *hy0, Y1 = *hy1;
        const unsigned long long x[4] = {X0.x, X0.y, X1.x, X1.y};
        const unsigned long long y[4] = {Y0.x, Y0.y, Y1.x, Y1.y};
        gram_mac(x, y, S == 1 ? *yp : make_float2(0.f, 0.f));
        hx0 += RS; hx1 += RS; hy0 += RS; hy1 += RS;
        yp += KP * S;
      }
    } else if (gram_busy) {
      for (int b = item_part; b < B; b += KP) {
        unsigned long long x[4], y[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int u = rb * 4 + r, v = cb * 4 + r;
          const float2 xu = u < U ? Hs[b * U + u] : make_float2(0.f, 0.f);
          const float2 yv = v < U ? Hs[b * U + v] : make_float2(0.f, 0.f);
          x[r] = f2pack(xu.x, xu.y);
          y[r] = f2pack(yv.x, yv.y);
        }
        gram_mac(x, y, S == 1 ? Ys[b] : make_float2(0.f, 0.f));
      }
    }
    __syncwarp();  // every lane's reads of H are done (the partials may overlay it)
    if (gram_busy) {
      if (S == 1 && rb == cb) {
        float2* Pm = P + item_part * PSTR + UG::NTILE * 16;  // [part][user]
#pragma unroll
        for (int r = 0; r < 4; ++r) Pm[rb * 4 + (r ^ (2 * rot2))] = f2unpack(mfa[r]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 A2 = f2unpack(a[r][c]), B2 = f2unpack(bb[r][c]);
          P[item_part * PSTR + (item_tile * 16) + ((r * 4 + c) ^ unrot)] =
              make_float2(A2.x + B2.y, A2.y - B2.x);
        }
    }
    __syncwarp();
    for (int e = lane; e < UP * UP; e += 32) {  // fixed-order part sums, lower entries
      const int u = e / UP, v = e - u * UP;
      if (v > u) continue;
      const int t = (u / 4) * (u / 4 + 1) / 2 + v / 4;
      const float2* pp = P + (t * 16 + (u % 4) * 4 + (v % 4));
      float2 g = pp[0];
#pragma unroll
      for (int k = 1; k < KP; ++k) g = cadd(g, pp[k * PSTR]);
      if (u == v) {
        Gs[u * UP + u] = make_float2(g.x, 0.f);
      } else {
        Gs[u * UP + v] = g;
        Gs[v * UP + u] = cconj(g);
      }
    }
    // --------------------------------------------- 2. matched filters H^H y
    if (S == 1) {  // fixed-order sums of the Gram loop's partials
      if (lane < UP) {
        const float2* pm = P + UG::NTILE * 16 + lane;
        float2 m = pm[0];
#pragma unroll
        for (int k = 1; k < KP; ++k) m = cadd(m, pm[k * PSTR]);
        MFs[lane] = m;
      }
    } else {
      // (vector, user) pairs x antenna parts: 4 parts when the pairs fit in 8
      // lanes, 2 in 16, else 1; the parts are summed by xor shuffles
      const int nq = S * UP;
      const int parts = nq <= 8 ? 4 : nq <= 16 ? 2 : 1;
      const int stride = 32 / parts;  // lanes per part
      const int part = lane / stride, q = lane - part * stride;
      for (int e0 = 0; e0 < nq; e0 += stride) {
        const int e = e0 + q;
        const int s = e / UP, u = e - s * UP;
        float2 m0 = make_float2(0.f, 0.f), m1 = make_float2(0.f, 0.f);
        if (e < nq && u < U) {
          int b = part;
          for (; b + parts < B; b += 2 * parts) {
            cfma_conj(m0, Hs[b * U + u], Ys[b * S + s]);
            cfma_conj(m1, Hs[(b + parts) * U + u], Ys[(b + parts) * S + s]);
          }
          if (b < B) cfma_conj(m0, Hs[b * U + u], Ys[b * S + s]);
        }
        float2 m = cadd(m0, m1);
        for (int o = stride; o < 32; o <<= 1) {
          m.x += __shfl_xor_sync(0xffffffffu, m.x, o);
          m.y += __shfl_xor_sync(0xffffffffu, m.y, o);
        }
        if (part == 0 && e < nq) MFs[s * UP + u] = m;
      }
    }
    __syncwarp();
    // ------------------------------------------- 3. exact: Chebyshev basis
    float cc = 0.f, dd = 1.f;
    if (EXACT) {
      const float2 cd = cheb_interval<UP>(Gs, p.rho_inv_u, xs, lane);
      cc = cd.x;
      dd = cd.y;
      const float invd = 1.f / dd;
      for (int e = lane; e < UP * UP; e += 32) {  // T_1 = (A - cI)/d
        const int i = e / UP, j = e - i * UP;
        float2 v = Gs[e];
        if (i == j) v.x += p.rho_inv_u - cc;
        Tb[e] = cscale(invd, v);
      }
      __syncwarp();
      for (int m = 1; m < K; ++m) {  // T_{m+1} = 2 T_1 T_m - T_{m-1}
        const float2* T1 = Tb;
        const float2* Tm = Tb + (m - 1) * UP * UP;
        float2* Tn = Tb + m * UP * UP;
        for (int e = lane; e < UP * UP; e += 32) {
          const int i = e / UP, j = e - i * UP;
          float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < UP; k += 2) {
            cfma(acc, T1[i * UP + k], Tm[k * UP + j]);
            cfma(acc2, T1[i * UP + k + 1], Tm[(k + 1) * UP + j]);
          }
          acc = cadd(acc, acc2);
          const float2 prev = m == 1 ? make_float2(i == j ? 1.f : 0.f, 0.f)
                                     : Tb[(m - 2) * UP * UP + e];
          float2 val = make_float2(2.f * acc.x - prev.x, 2.f * acc.y - prev.y);
          if (i == j) val.y = 0.f;
          Tn[e] = val;
        }
        __syncwarp();
      }
    }
    // ------------------------------------------------------ 4. CG per vector
    {
      const int grp = lane / GL, gl = lane - grp * GL;
      float2* Pw = Ps + grp * UP;
      const float gdiag = Gs[gl * UP + gl].x;
      for (int base = 0; base < S; base += GPW) {
        const int sys = base + grp;
        const bool live = sys < S;
        const float2 b = live && gl < U ? MFs[sys * UP + gl] : make_float2(0.f, 0.f);
        float2 v = make_float2(0.f, 0.f), r = b, pp = b;
        Pw[gl] = b;
        float rn = cnorm(b);
        for (int o = GL / 2; o > 0; o >>= 1) rn += __shfl_xor_sync(0xffffffffu, rn, o);
        const float rn0 = rn;
        bool broke = false;
        float f0 = 0.f, f1 = 0.f, f2 = 0.f, am1 = 1.f, am2 = 1.f, bm1 = 0.f, bm2 = 0.f;
        __syncwarp();
        for (int k = 1; k <= K; ++k) {
          float2 e = make_float2(0.f, 0.f), e2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < UP; j += 2) {
            cfma_conj(e, Gs[j * UP + gl], Pw[j]);  // G[gl][j] = conj(G[j][gl])
            cfma_conj(e2, Gs[(j + 1) * UP + gl], Pw[j + 1]);
          }
          e = cadd(e, e2);
          e.x = fmaf(p.rho_inv_u, pp.x, e.x);
          e.y = fmaf(p.rho_inv_u, pp.y, e.y);
          float curv = pp.x * e.x + pp.y * e.y;
          for (int o = GL / 2; o > 0; o >>= 1) curv += __shfl_xor_sync(0xffffffffu, curv, o);
          const bool frozen = !(rn > 1e-28f * rn0);  // solvers.cpp:21,25-27
          const bool go = live && !frozen && !broke;
          if (go && curv < 1e-30f) broke = true;     // solvers.cpp:55-57
          const bool upd = go && !broke;
          const float alpha = upd ? __fdividef(rn, curv) : 1.f;
          float beta = 0.f;
          if (upd) {
            v.x = fmaf(alpha, pp.x, v.x);
            v.y = fmaf(alpha, pp.y, v.y);
            r.x = fmaf(-alpha, e.x, r.x);
            r.y = fmaf(-alpha, e.y, r.y);
          }
          float rnx = cnorm(r);
          for (int o = GL / 2; o > 0; o >>= 1) rnx += __shfl_xor_sync(0xffffffffu, rnx, o);
          __syncwarp();
          if (upd) {
            beta = __fdividef(rnx, rn);
            rn = rnx;
            pp.x = fmaf(beta, pp.x, r.x);
            pp.y = fmaf(beta, pp.y, r.y);
            Pw[gl] = pp;
          }
          if (EXACT) {
            if (live && gl == 0) {
              hist[(sys * K + (k - 1)) * 2 + 0] = alpha;
              hist[(sys * K + (k - 1)) * 2 + 1] = beta;
            }
          } else {
            // Eq. (11) on the diagonal (detect.cpp:409-427)
            float nf;
            if (k == 1) {
              nf = alpha;
            } else {
              const float c1 = __fdividef(alpha * (1.f + bm1), am1);
              const float c2 = __fdividef(alpha * bm2, am2);
              nf = f0 + (c1 - alpha * (gdiag + p.rho_inv_u)) * (f0 - f1) - c2 * (f1 - f2);
            }
            f2 = f1;
            f1 = f0;
            f0 = nf;
          }
          am2 = am1; am1 = alpha;
          bm2 = bm1; bm1 = beta;
          __syncwarp();
        }
        if (!live) continue;
        if (EXACT) {
          Vs[sys * UP + gl] = v;
          if (gl == 0) sys_st[sys] = broke ? 1 : 0;
        } else if (gl < U) {
          // approx: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
          const long o = (sc * S + sys) * static_cast<long>(U) + gl;
          const bool ok = !broke;
          const float2 xh = ok ? v : make_float2(0.f, 0.f);
          const float mu_u = ok ? f0 * gdiag : 0.f;
          const float rho_u = ok ? gdiag / p.n0 : 0.f;
          if (p.xhat) p.xhat[o] = xh;
          if (p.mu) p.mu[o] = mu_u;
          if (p.rho) p.rho[o] = rho_u;
          if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
          if (p.status && gl == 0) p.status[sc * S + sys] = ok ? 0 : 1;
        }
      }
    }
    // ------------------------------------- 5. exact: coefficients + extraction
    if (EXACT) {
      __syncwarp();
      for (int s = 0; s < S; ++s) {  // FP64 coefficient recursion, warp-parallel
        float* cl = coef + s * 2 * (K + 2);
        cheb_coef_warp(hist + s * K * 2, K, cc, dd, p.rho_inv_u, cl, cl + (K + 2));
      }
      __syncwarp();
      // one vector per subcarrier: the 32 / UP lane groups split the columns
      // of row i = lane mod UP (xor-shuffle sums, every group ends with the
      // same bits); otherwise a (vector, row) per lane walks all UP columns
      const int xparts = S == 1 ? GPW : 1, xnc = UP / xparts;
      for (int e = lane; e < S * UP * xparts; e += 32) {
        const int xpart = S == 1 ? e / UP : 0;
        const int s = S == 1 ? 0 : e / UP, i = e - (S == 1 ? xpart : s) * UP;
        const float* cl = coef + s * 2 * (K + 2);
        const float* cbq = cl + (K + 2);
        float ib2 = 0.f, ibl = 0.f, mu_i = 0.f;
        for (int j = xpart * xnc; j < (xpart + 1) * xnc; ++j) {
          float2 Bv = make_float2(i == j ? cbq[0] : 0.f, 0.f);
          float2 Lv = make_float2(i == j ? cl[0] : 0.f, 0.f);
          for (int m = 1; m <= K; ++m) {
            const float2 t = Tb[(m - 1) * UP * UP + i * UP + j];  // T_m[i][j]
            Bv.x = fmaf(cbq[m], t.x, Bv.x); Bv.y = fmaf(cbq[m], t.y, Bv.y);
            if (m < K) { Lv.x = fmaf(cl[m], t.x, Lv.x); Lv.y = fmaf(cl[m], t.y, Lv.y); }
          }
          if (j == i) mu_i = Bv.x;
          else ib2 += cnorm(Bv);
          ibl += Bv.x * Lv.x + Bv.y * Lv.y;  // Re(B_ij conj(L_ij))
        }
        if (S == 1) {  // all 32 lanes are here (UP * GPW = 32)
#pragma unroll
          for (int o = UP; o < 32; o <<= 1) {
            ib2 += __shfl_xor_sync(0xffffffffu, ib2, o);
            ibl += __shfl_xor_sync(0xffffffffu, ibl, o);
            mu_i += __shfl_xor_sync(0xffffffffu, mu_i, o);
          }
          if (xpart != 0) continue;
        }
        if (i >= U) continue;
        const float nu2 = ib2 * p.es + ibl * p.n0;
        const bool ok = sys_st[s] == 0;
        const float mu = ok ? mu_i : 0.f;
        const float rr = ok ? (nu2 <= 0.f ? 0.f : mu_i * mu_i / nu2) : 0.f;  // safe_rho
        const float2 xh = ok ? Vs[s * UP + i] : make_float2(0.f, 0.f);
        const long o = (sc * S + s) * static_cast<long>(U) + i;
        if (p.xhat) p.xhat[o] = xh;
        if (p.mu) p.mu[o] = mu;
        if (p.rho) p.rho[o] = rr;
        if (p.llr) store_llrs_fast(xh, mu, rr, p.bits, p.llr + o * p.bits);
        if (p.status && i == 0) p.status[sc * S + s] = ok ? 0 : 1;
      }
    }
    // generic-proxy writes over the staging buffer (overlaid partials / basis)
    // are ordered before the next subcarrier's bulk copy into it
    if (tma) fence_proxy_async();
    __syncwarp();  // shared buffers reused by the next subcarrier
  }
}

}  // namespace cgm
