// cgm_kernels.cuh -- the fused per-subcarrier kernel (sm_100a).
//
// One CTA owns one subcarrier at a time (grid-stride persistent loop).
// Everything that depends only on the channel -- the Gram matrix G = H^H H
// and, for the exact tracker, the Chebyshev basis T_m(Ahat) -- is built ONCE
// per subcarrier in shared memory and reused by all S received vectors
// (uplink) and all St transmit vectors (downlink) sharing the channel.
// Replaces, per instance:
//
//   gram_regularized           linalg.cpp:59-101   -> phase 1 (4x4 register tiles)
//   matvec_adjoint (MF)        linalg.cpp:116-126  -> phase 1 (same tiles)
//   cg_solve / cg_core         solvers.cpp:37-72   -> phase 2 (lane group per system)
//   ApproxSinrTracker          detect.cpp:397-441  -> phase 2 (per lane)
//   ExactSinrTracker + extract detect.cpp:330-395  -> phase 3 (shared basis)
//   compute_llrs               detect.cpp:57-86    -> phase 2 (approx) / 4 (exact)
//   precode_cg + normalize     precode.cpp:22-71   -> phases 2 + 5
//
// Exact tracker (Eq. 10): L_k is a real-coefficient polynomial in A, so the
// reference's three-term recursion (detect.cpp:350-358) is run on the
// polynomial COEFFICIENTS (O(K^2) per system, FP64) in the Chebyshev basis
// T_m(Ahat), Ahat = (A - cI)/d, and L_K, B = L_K G are evaluated from the
// basis shared by the subcarrier's systems.  The U^3 work is (K-1) Hermitian
// products per SUBCARRIER instead of K per vector.  (The monomial basis
// loses ~1e-3 at K = 8 in FP32; the Chebyshev one stays ~1e-5.)
//
// Barrier discipline: split-K partial sums are reduced with warp shuffles
// (the split lanes of a tile live in one warp); the CG runs per warp with
// no CTA barrier; __syncthreads only separates the phases.
#pragma once

#include "cgm_device.cuh"

namespace cgm {

constexpr int kMaxK = 16;    // CG iterations supported by the exact tracker
constexpr int kMaxSys = 64;  // systems (uplink + downlink vectors) per subcarrier

struct KernelParams {
  const float2* H;  // uplink layout [n_sc][B][U] or downlink [n_sc][U][B]
  const float2* Y;  // [n_sc][B][S] (antenna-major: the B x S matrix of a subcarrier)
  const float2* T;  // [n_sc][St][U]
  float2* xhat;     // [n_sc][S][U]   (each output may be null)
  float* mu;
  float* rho;
  float* llr;       // [n_sc][S][U][bits]
  uint8_t* status;  // [n_sc][S]
  float2* q;        // [n_sc][St][B]
  float2* s_out;    // [n_sc][St][B]
  float* gain;      // [n_sc][St]
  uint8_t* pstatus; // [n_sc][St]
  float* tscratch;  // per-CTA Chebyshev basis when it does not fit in smem
  long n_sc;
  int B, U, S, St, K, Kt, bits;
  int hd_layout;  // 1: H is the downlink matrix [U][B] (precode only)
  int use_tma;    // bulk-copy staging (U == UP, B even, 16B aligned)
  int t_in_smem;  // Chebyshev basis in shared memory
  float rho_inv_u, rho_inv_d, n0, es;
  int debug;      // profiling knobs (0 in production)
  float2* ws;     // split path: per-subcarrier workspace (G, MF, basis)
  long sc_base;   // split path: first subcarrier of this chunk
  int k1_pair, k1_spl, k1_wpp;  // channel kernel: subcarriers per CTA, k-parts, warps per part
  unsigned long long* trace;    // microbenchmarks only: per-CTA event clocks (null in production)
  int method;                   // sim::Method order: 0 Cholesky, 1 CG, 2 CGLS, 3 Neumann (cgm_alt.cuh)
  int basis_ext;                // exact tracker: the Chebyshev basis comes from basis_kernel (cgm_basis.cuh)
  int fx;                       // exact tracker, one vector per subcarrier: basis + extraction fused (basis_extract_kernel); the workspace holds the CG history instead of T_1..T_K
};

// Per-axis Gray amplitude subsets (constellation.cpp:75-84), [qam][p][k],
// qam 0/1/2 = QPSK/16/64.
struct AxisTables {
  float a0[3][3][4];
  float a1[3][3][4];
  float lv[3][8];  // per-axis amplitudes in ascending order (level k <-> Gray label k^(k>>1))
};
__constant__ AxisTables c_axis;

template <int UP>
struct Geo {
  static constexpr int G = UP < 32 ? UP : 32;  // lanes per CG system
  static constexpr int RU = UP / G;            // rows per lane
  static constexpr int GPW = 32 / G;           // groups per warp
  static constexpr int NS = (4 * G / 32) / RU > 0 ? (4 * G / 32) / RU : 1;  // systems per group
};

// ----------------------------------------------------------------- layout
template <int UP>
struct Smem {
  int bar, hs, scr, gs, vs, ps, hist, sys_st, mu, rho, coef, misc, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int St, int K, bool exact, int t_in_smem) {
    const int nsys = S + St;
    // scratch region, phase-aliased: Ys [B][S] (phase 0-1; +64 B so the
    // last row's 4-wide tile reads stay in bounds), T basis (phase 3),
    // q staging (phase 5)
    int scr_bytes = B * S * 8 + 64;
    if (exact && t_in_smem) scr_bytes = scr_bytes > K * UP * UP * 8 ? scr_bytes : K * UP * UP * 8;
    if (St > 0) scr_bytes = scr_bytes > St * B * 8 ? scr_bytes : St * B * 8;
    int o = 0;
    bar = o; o = align(o + 16);
    hs = o; o = align(o + B * UP * 8);
    scr = o; o = align(o + scr_bytes);
    gs = o; o = align(o + UP * UP * 8);
    vs = o; o = align(o + nsys * UP * 8);
    ps = o; o = align(o + nsys * UP * 8);
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    sys_st = o; o = align(o + nsys);
    mu = o; o = align(o + (exact ? S * UP * 4 : 0));
    rho = o; o = align(o + (exact ? S * UP * 4 : 0));
    coef = o; o = align(o + (exact ? S * 2 * (K + 2) * 4 : 0));
    misc = o; o = align(o + 16);
    total = o;
  }
};

__device__ __forceinline__ void tri_block(int t, int& ib, int& jb) {
  // t -> (ib, jb), jb <= ib, row-major over the lower triangle
  ib = static_cast<int>((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
  while ((ib + 1) * (ib + 2) / 2 <= t) ++ib;
  while (ib * (ib + 1) / 2 > t) --ib;
  jb = t - ib * (ib + 1) / 2;
}

// ------------------------------------------------------- split-K tile pass
// Tiles 0..n_lower-1 are 4x4 blocks of the lower triangle of
// C = conj(X)^T Y (k over [0, klen)); tiles n_lower.. are 4x4 blocks of
// C2 = conj(X)^T Z with Z(k, j) = Zs[k*ldz + j] (the matched filter; its
// tiles are ordered so that neighbouring lanes share the Z block).  SPL
// lanes of one warp share a tile and split k; their partial sums are
// combined with butterflies, no CTA barrier.  Epilogue fn(tile, ib, jb, acc)
// runs on the split-0 lane.
template <int SPL, class Epi>
__device__ __forceinline__ void tile_pass_spl(int nwarps, int n_lower, int n_other, int nsb,
                                             const float2* __restrict__ X, int ldx,
                                             const float2* __restrict__ Yl, int ldyl,
                                             const float2* __restrict__ Zs, int ldz, int zcols,
                                             int klen, Epi&& fn) {
  const int n_tiles = n_lower + n_other;
  constexpr int TPW = 32 / SPL;  // tiles per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int part = lane % SPL;
  const int kchunk = (klen + SPL - 1) / SPL;
  const int k0 = part * kchunk, k1 = min(klen, k0 + kchunk);
  for (int base = warp * TPW; base < n_tiles; base += nwarps * TPW) {
    const int tile = base + lane / SPL;
    const bool active = tile < n_tiles;
    float2 acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
    int ib = 0, jb = 0;
    if (active) {
      if (tile < n_lower) {
        tri_block(tile, ib, jb);
        tile4x4<true>(acc, X, ldx, ib * 4, Yl, ldyl, 1, jb * 4, 1 << 30, k0, k1);
      } else {
        const int m = tile - n_lower;
        const int nbi = n_other / nsb;
        jb = m / nbi;
        ib = m - jb * nbi;
        if ((ldz & 1) == 0)
          tile4x4<true>(acc, X, ldx, ib * 4, Zs, ldz, 1, jb * 4, 1 << 30, k0, k1);
        else
          tile4x4<false>(acc, X, ldx, ib * 4, Zs, ldz, 1, jb * 4, zcols, k0, k1);
      }
    }
#pragma unroll
    for (int o = 1; o < SPL; o <<= 1)
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[r][c].x += __shfl_xor_sync(0xffffffffu, acc[r][c].x, o);
          acc[r][c].y += __shfl_xor_sync(0xffffffffu, acc[r][c].y, o);
        }
    if (active && part == 0) fn(tile, ib, jb, acc);
  }
}

template <class Epi>
__device__ __forceinline__ void tile_pass_nw(int NW, int n_lower, int n_other, int nsb,
                                             const float2* X, int ldx, const float2* Yl, int ldyl,
                                             const float2* Zs, int ldz, int zcols, int klen,
                                             Epi&& fn) {
  const int n_tiles = n_lower + n_other;
  // widest split whose tiles fit in one pass over the warps
  if (n_tiles <= NW * 2 && klen >= 64)
    tile_pass_spl<16>(NW, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
  else if (n_tiles <= NW * 4 && klen >= 32)
    tile_pass_spl<8>(NW, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
  else if (n_tiles <= NW * 8 && klen >= 16)
    tile_pass_spl<4>(NW, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
  else if (n_tiles <= NW * 16 && klen >= 8)
    tile_pass_spl<2>(NW, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
  else
    tile_pass_spl<1>(NW, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
}

template <int NT, class Epi>
__device__ __forceinline__ void tile_pass(int n_lower, int n_other, int nsb, const float2* X,
                                          int ldx, const float2* Yl, int ldyl, const float2* Zs,
                                          int ldz, int zcols, int klen, Epi&& fn) {
  tile_pass_nw(NT / 32, n_lower, n_other, nsb, X, ldx, Yl, ldyl, Zs, ldz, zcols, klen, fn);
}

// ------------------------------------------------ Chebyshev interval
// Interval [lo, hi] containing the spectrum of A = G + reg I for the exact
// tracker's basis T_m((A - cI)/d), c = (lo + hi)/2, d = (hi - lo)/2:
// lo = reg (G >= 0), hi = 1.1 x a 6-step power-iteration estimate of
// lambda_max.  A positive interval keeps the Chebyshev coefficients of
// L_K ~ A^-1 small; the round-1 choice c = tr(A)/U, d = 2 ||A - cI||_F /
// sqrt(U) reached below 0 at weak regularisation and lost up to 1.5e-3 in
// rho at K = 16 (tools/fp32_tracker_study.py "weak": 1.5e-6 with this one).
// One warp; G Hermitian in smem (read by columns); xs: UP float2 scratch.
// Exact tracker's three-term recursion (detect.cpp:336-368) on the
// Chebyshev coefficients of L_k, WARP-PARALLEL: lane m holds coefficient m
// of L_k, L_{k-1}, L_{k-2} (FP64), the multiplication by A = c + d Ahat
// couples neighbouring coefficients through shuffles:
//   A T_0 = c T_0 + d T_1,  A T_m = c T_m + d/2 (T_{m+1} + T_{m-1}).
// hist: the K (alpha, beta) pairs of one system.  Writes the coefficients of
// L_K (cl) and of B = L_K (A - rho^-1 I) (cb), K + 2 floats each.  Same
// values as the per-thread loops of k2_exact_tail (FP64; only the order of
// two or three additions per coefficient differs).  All 32 lanes must call.
__device__ __forceinline__ void cheb_coef_warp(const float* hist, int K, double cc, double dd,
                                               double rho_inv, float* cl, float* cb) {
  const int m = threadIdx.x & 31;
  const int n = K + 2;
  auto mulA = [&](double x) {
    const double up = __shfl_down_sync(0xffffffffu, x, 1);  // x[m + 1]
    const double dn = __shfl_up_sync(0xffffffffu, x, 1);    // x[m - 1]
    double out = cc * x;
    if (m + 1 < n) out += 0.5 * dd * up;
    if (m == 1) out += dd * dn;
    else if (m >= 2 && m < n) out += 0.5 * dd * dn;
    return m < n ? out : 0.0;
  };
  double l0 = 0.0, l1 = 0.0, l2 = 0.0;
  double a_m1 = 1.0, a_m2 = 1.0, b_m1 = 0.0, b_m2 = 0.0;
  for (int k = 1; k <= K; ++k) {
    const double a = hist[(k - 1) * 2 + 0];
    const double bb = hist[(k - 1) * 2 + 1];
    if (k == 1) {
      l2 = l1;
      l1 = l0;
      l0 = m == 0 ? a : 0.0;  // L_1 = alpha_1 I
    } else {
      const double c1 = a * (1.0 + b_m1) / a_m1, c2 = a * b_m2 / a_m2;
      const double d1 = l0 - l1;
      const double t = mulA(d1);
      const double nx = l0 + c1 * d1 - a * t - c2 * (l1 - l2);
      l2 = l1;
      l1 = l0;
      l0 = m < n ? nx : 0.0;
    }
    a_m2 = a_m1; a_m1 = a; b_m2 = b_m1; b_m1 = bb;
  }
  const double t = mulA(l0);  // B = L (A - rho^-1 I)
  if (m < n) {
    cl[m] = static_cast<float>(l0);
    cb[m] = static_cast<float>(t - rho_inv * l0);
  }
}

template <int UP, int LDG = UP>
__device__ __forceinline__ float2 cheb_interval(const float2* Gs, float reg, float2* xs, int lane) {
  constexpr int RU = UP < 32 ? 1 : UP / 32;
  float2 xr[RU];
#pragma unroll
  for (int m = 0; m < RU; ++m) {
    const int i = lane + 32 * m;
    xr[m] = make_float2(i < UP ? 1.f : 0.f, 0.f);
    if (i < UP) xs[i] = xr[m];
  }
  __syncwarp();
  float lam = reg;
  for (int it = 0; it <= 6; ++it) {
    float2 y[RU];
    float nrm = 0.f, ray = 0.f;
#pragma unroll
    for (int m = 0; m < RU; ++m) {
      const int i = lane + 32 * m;
      y[m] = make_float2(0.f, 0.f);
      if (i < UP) {
        // (A x)_i = sum_j conj(G[j][i]) x_j + reg x_i  (G Hermitian; column reads)
        for (int j = 0; j < UP; ++j) cfma_conj(y[m], Gs[j * LDG + i], xs[j]);
        y[m].x = fmaf(reg, xr[m].x, y[m].x);
        y[m].y = fmaf(reg, xr[m].y, y[m].y);
      }
      nrm += cnorm(y[m]);
      ray += xr[m].x * y[m].x + xr[m].y * y[m].y;
    }
    nrm = group_sum<32>(nrm);
    ray = group_sum<32>(ray);
    if (it > 0) lam = ray;  // Rayleigh quotient x^H A x, ||x|| = 1
    const float inv = nrm > 0.f ? rsqrtf(nrm) : 0.f;
    __syncwarp();
#pragma unroll
    for (int m = 0; m < RU; ++m) {
      const int i = lane + 32 * m;
      xr[m] = cscale(inv, y[m]);
      if (i < UP) xs[i] = xr[m];
    }
    __syncwarp();
  }
  const float lo = reg;
  const float hi = fmaxf(1.1f * lam, 1.0001f * lo);
  const float c = 0.5f * (lo + hi);
  float d = 0.5f * (hi - lo);
  if (!(d > 1e-6f * fmaxf(fabsf(c), 1e-30f))) d = fmaxf(fabsf(c), 1.f);
  return make_float2(c, d);
}

// ------------------------------------------------------------------ LLR
__device__ __forceinline__ float axis_min_sq(float z, const float* amps, int n) {
  float best = INFINITY;
  for (int k = 0; k < n; ++k) {
    const float d = z - amps[k];
    best = fminf(best, __fmul_rn(d, d));
  }
  return best;
}

// Max-log LLRs of one user (detect.cpp:68-86) into out[0..bits): erasure
// below the gain floor, rho < 0 -> 0, z = xhat/mu, I bits then Q bits,
// positive favours bit 1, clip +-64.
__device__ __forceinline__ void store_llrs(float2 xh, float mu, float rho, int bits, float* out) {
  const int half = bits >> 1, q = half - 1, per = 1 << (half - 1);
  float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (!(fabsf(mu) < 1e-12f)) {
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
        const float lr = fminf(64.f, fmaxf(-64.f, rho * (d0r - d1r)));
        const float li = fminf(64.f, fmaxf(-64.f, rho * (d0i - d1i)));
        if (p == 0) { v[0] = lr; v[half] = li; }
        if (p == 1) { v[1] = lr; v[half + 1] = li; }
        if (p == 2) { v[2] = lr; v[half + 2] = li; }
      }
    }
  }
  if (bits == 4) {
    *reinterpret_cast<float4*>(out) = make_float4(v[0], v[1], v[2], v[3]);
  } else if (bits == 6) {
    reinterpret_cast<float2*>(out)[0] = make_float2(v[0], v[1]);
    reinterpret_cast<float2*>(out)[1] = make_float2(v[2], v[3]);
    reinterpret_cast<float2*>(out)[2] = make_float2(v[4], v[5]);
  } else {
    *reinterpret_cast<float2*>(out) = make_float2(v[0], v[1]);
  }
}

// Closed-form max-log LLRs of one user: the squared distances to the L
// sorted axis levels are formed once and the two per-bit minima taken over
// fixed index sets.  Level k carries the Gray axis label k ^ (k >> 1)
// (constellation.cpp:58-84), so for 64-QAM bit 0 = [k >= 4], bit 1 =
// [k in 2..5], bit 2 = [k in {1,2,5,6}]; for 16-QAM bit 0 = [k >= 2],
// bit 1 = [k in {1,2}].  Same values as the min loops of detect.cpp:57-86.
template <int BITS>
__device__ __forceinline__ void llr_axis(float z, float rho, float* o) {
  constexpr int q = BITS / 2 - 1;
  if (BITS == 6) {
    float d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float t = z - c_axis.lv[q][k];
      d[k] = __fmul_rn(t, t);  // rounded alone (no FMA contraction): exact ties stay 0
    }
    const float b0 = fminf(fminf(d[0], d[1]), fminf(d[2], d[3])) -
                     fminf(fminf(d[4], d[5]), fminf(d[6], d[7]));
    const float b1 = fminf(fminf(d[0], d[1]), fminf(d[6], d[7])) -
                     fminf(fminf(d[2], d[3]), fminf(d[4], d[5]));
    const float b2 = fminf(fminf(d[0], d[3]), fminf(d[4], d[7])) -
                     fminf(fminf(d[1], d[2]), fminf(d[5], d[6]));
    o[0] = fminf(64.f, fmaxf(-64.f, rho * b0));
    o[1] = fminf(64.f, fmaxf(-64.f, rho * b1));
    o[2] = fminf(64.f, fmaxf(-64.f, rho * b2));
  } else if (BITS == 4) {
    float d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float t = z - c_axis.lv[q][k];
      d[k] = __fmul_rn(t, t);
    }
    o[0] = fminf(64.f, fmaxf(-64.f, rho * (fminf(d[0], d[1]) - fminf(d[2], d[3]))));
    o[1] = fminf(64.f, fmaxf(-64.f, rho * (fminf(d[0], d[3]) - fminf(d[1], d[2]))));
  } else {
    const float t0 = z - c_axis.lv[q][0], t1 = z - c_axis.lv[q][1];
    o[0] = fminf(64.f, fmaxf(-64.f, rho * (__fmul_rn(t0, t0) - __fmul_rn(t1, t1))));
  }
}

template <int BITS>
__device__ __forceinline__ void llr_user(float2 xh, float mu, float rho, float* out) {
  constexpr int H = BITS / 2;
  float v[BITS];
#pragma unroll
  for (int b = 0; b < BITS; ++b) v[b] = 0.f;
  if (!(fabsf(mu) < 1e-12f)) {  // erasure below the gain floor (detect.cpp:71)
    if (rho < 0.f) rho = 0.f;
    const float inv = 1.0f / mu;
    llr_axis<BITS>(xh.x * inv, rho, v);
    llr_axis<BITS>(xh.y * inv, rho, v + H);
  }
  if (BITS == 4) {
    *reinterpret_cast<float4*>(out) = make_float4(v[0], v[1], v[2], v[3]);
  } else if (BITS == 6) {
    reinterpret_cast<float2*>(out)[0] = make_float2(v[0], v[1]);
    reinterpret_cast<float2*>(out)[1] = make_float2(v[2], v[3]);
    reinterpret_cast<float2*>(out)[2] = make_float2(v[4], v[5]);
  } else {
    *reinterpret_cast<float2*>(out) = make_float2(v[0], v[1]);
  }
}

__device__ __forceinline__ void store_llrs_fast(float2 xh, float mu, float rho, int bits,
                                                float* out) {
  if (bits == 6) llr_user<6>(xh, mu, rho, out);
  else if (bits == 4) llr_user<4>(xh, mu, rho, out);
  else llr_user<2>(xh, mu, rho, out);
}

// sum over the aligned group of G lanes of NS values at once (ILP across systems)
template <int G, int NS>
__device__ __forceinline__ void group_sum_n(float (&v)[NS]) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
    for (int s = 0; s < NS; ++s) v[s] += __shfl_xor_sync(0xffffffffu, v[s], o);
}

// ------------------------------------------------------------------ kernel
template <int UP, int NT, bool EXACT>
__global__ void __launch_bounds__(NT, 2) subcarrier_kernel(const KernelParams p) {
  using GE = Geo<UP>;
  constexpr int G = GE::G, RU = GE::RU, GPW = GE::GPW, NS = GE::NS;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smem[];

  const int B = p.B, S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  Smem<UP> L;
  L.plan(B, S, St, Kmax, EXACT, p.t_in_smem);

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Hs = reinterpret_cast<float2*>(smem + L.hs);
  float2* Ys = reinterpret_cast<float2*>(smem + L.scr);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);  // b on entry, v on exit
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* MUs = reinterpret_cast<float*>(smem + L.mu);
  float* RHOs = reinterpret_cast<float*>(smem + L.rho);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  float* misc = reinterpret_cast<float*>(smem + L.misc);
  float2* Tb = p.t_in_smem ? reinterpret_cast<float2*>(smem + L.scr)
                           : reinterpret_cast<float2*>(p.tscratch) +
                                 static_cast<long>(blockIdx.x) * Kmax * UP * UP;
  float2* Qs = reinterpret_cast<float2*>(smem + L.scr);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (p.use_tma && tid == 0) mbar_init(bar, 1);
  __syncthreads();

  const int nb = UP / 4;
  const int n_gram = nb * (nb + 1) / 2;
  const int nsb = (S + 3) / 4;

  uint32_t phase = 0;
  for (long sc = blockIdx.x; sc < p.n_sc; sc += gridDim.x, phase ^= 1u) {
    // ------------------------------------------------ phase 0: stage inputs
    if (p.use_tma) {
      if (tid == 0) {
        const uint32_t hbytes = static_cast<uint32_t>(B) * UP * 8u;
        const uint32_t ybytes = static_cast<uint32_t>(B) * S * 8u;
        fence_proxy_async();
        mbar_expect_tx(bar, hbytes + ybytes);
        bulk_g2s(Hs, p.H + sc * static_cast<long>(B) * UP, hbytes, bar);
        if (S > 0) bulk_g2s(Ys, p.Y + sc * static_cast<long>(B) * S, ybytes, bar);
      }
    } else {
      if (p.hd_layout) {
        // downlink H_d [U][B] -> Hs[b][u] = conj(H_d[u][b])  (= H_u = H_d^H)
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
      for (int e = tid; e < S * B; e += NT) Ys[e] = p.Y[sc * static_cast<long>(B) * S + e];
    }
    // downlink right-hand sides t (precode.cpp:64: CG on b = t)
    for (int e = tid; e < St * UP; e += NT) {
      const int s = e / UP, u = e - s * UP;
      Vs[(S + s) * UP + u] =
          u < U ? p.T[(sc * St + s) * static_cast<long>(U) + u] : make_float2(0.f, 0.f);
    }
    if (p.use_tma) mbar_wait(bar, phase);
    __syncthreads();

    // ------------------------------------- phase 1: Gram + matched filter
    tile_pass<NT>(n_gram, nb * nsb, nsb, Hs, UP, Hs, UP, Ys, S, S, B,
                  [&](int tile, int ib, int jb, float2 (&acc)[4][4]) {
                    if (tile < n_gram) {
                      // one triangle + conjugate mirror: G == G^H exactly
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
                          if (s < S) Vs[s * UP + ib * 4 + r] = acc[r][c];
                        }
                    }
                  });
    __syncthreads();

    // --------------------------------------------- phase 2: CG per system
    // group g of G lanes runs NS systems at once; lane gl owns rows gl + G*m
    {
      const int grp_in_warp = lane / G, gl = lane - grp_in_warp * G;
      const int n_groups = NW * GPW;
      float gdiag[RU];
#pragma unroll
      for (int m = 0; m < RU; ++m) gdiag[m] = Gs[(gl + m * G) * UP + gl + m * G].x;
      // warp-uniform trip count (shuffles below use the full mask)
      for (int wbase = warp * GPW * NS; wbase < nsys; wbase += n_groups * NS) {
        const int base = wbase + grp_in_warp * NS;
        int sys[NS];
        bool live[NS], down[NS];
        float reg[NS];
        int iters[NS];
        float2 v[NS][RU], r[NS][RU], pp[NS][RU];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          sys[s] = base + s;
          live[s] = sys[s] < nsys;
          down[s] = sys[s] >= S;
          reg[s] = down[s] ? p.rho_inv_d : p.rho_inv_u;
          iters[s] = live[s] ? (down[s] ? p.Kt : p.K) : 0;
          const int row = live[s] ? sys[s] : 0;
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            const float2 b = live[s] ? Vs[row * UP + gl + m * G] : make_float2(0.f, 0.f);
            v[s][m] = make_float2(0.f, 0.f);
            r[s][m] = b;
            pp[s][m] = b;
          }
        }
        float rn[NS], rn0[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          rn[s] = 0.f;
#pragma unroll
          for (int m = 0; m < RU; ++m) rn[s] += cnorm(r[s][m]);
        }
        group_sum_n<G, NS>(rn);
        bool broke[NS];
        // approximate tracker state (detect.cpp:400-433); histories alpha=1, beta=0
        float f0[NS][RU], f1[NS][RU], f2[NS][RU];
        float am1[NS], am2[NS], bm1[NS], bm2[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          rn0[s] = rn[s];
          broke[s] = false;
          am1[s] = am2[s] = 1.f;
          bm1[s] = bm2[s] = 0.f;
#pragma unroll
          for (int m = 0; m < RU; ++m) f0[s][m] = f1[s][m] = f2[s][m] = 0.f;
          if (live[s]) {
#pragma unroll
            for (int m = 0; m < RU; ++m) Ps[sys[s] * UP + gl + m * G] = pp[s][m];
          }
        }
        __syncwarp();
        for (int k = 1; k <= Kmax; ++k) {
          // e = (G + reg I) p for every system of the group (G loaded once)
          float2 e[NS][RU];
#pragma unroll
          for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int m = 0; m < RU; ++m) e[s][m] = make_float2(0.f, 0.f);
#pragma unroll 4
          for (int j = 0; j < UP; j += 2) {
            float2 g0[RU], g1[RU];
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              g0[m] = cconj(Gs[j * UP + gl + m * G]);        // G[u][j]
              g1[m] = cconj(Gs[(j + 1) * UP + gl + m * G]);  // G[u][j+1]
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) {
              const int row = live[s] ? sys[s] : 0;
              const float4 pj = *reinterpret_cast<const float4*>(Ps + row * UP + j);
#pragma unroll
              for (int m = 0; m < RU; ++m) {
                cfma(e[s][m], g0[m], make_float2(pj.x, pj.y));
                cfma(e[s][m], g1[m], make_float2(pj.z, pj.w));
              }
            }
          }
          float curv[NS];
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            curv[s] = 0.f;
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              e[s][m].x = fmaf(reg[s], pp[s][m].x, e[s][m].x);
              e[s][m].y = fmaf(reg[s], pp[s][m].y, e[s][m].y);
              curv[s] += pp[s][m].x * e[s][m].x + pp[s][m].y * e[s][m].y;  // Re p^H e
            }
          }
          group_sum_n<G, NS>(curv);
          float alpha[NS], beta[NS], rnx[NS];
          bool upd[NS];
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const bool step = k <= iters[s];
            const bool frozen = !(rn[s] > 1e-28f * rn0[s]);  // solvers.cpp:21,25-27
            const bool go = step && !frozen && !broke[s];
            if (go && curv[s] < 1e-30f) broke[s] = true;    // solvers.cpp:55-57
            upd[s] = go && !broke[s];
            alpha[s] = upd[s] ? rn[s] / curv[s] : 1.f;
            beta[s] = 0.f;
            rnx[s] = 0.f;
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              if (upd[s]) {
                v[s][m].x = fmaf(alpha[s], pp[s][m].x, v[s][m].x);
                v[s][m].y = fmaf(alpha[s], pp[s][m].y, v[s][m].y);
                r[s][m].x = fmaf(-alpha[s], e[s][m].x, r[s][m].x);
                r[s][m].y = fmaf(-alpha[s], e[s][m].y, r[s][m].y);
              }
              rnx[s] += cnorm(r[s][m]);
            }
          }
          group_sum_n<G, NS>(rnx);
          __syncwarp();
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            if (upd[s]) {
              beta[s] = rnx[s] / rn[s];
              rn[s] = rnx[s];
#pragma unroll
              for (int m = 0; m < RU; ++m) {
                pp[s][m].x = fmaf(beta[s], pp[s][m].x, r[s][m].x);
                pp[s][m].y = fmaf(beta[s], pp[s][m].y, r[s][m].y);
                Ps[sys[s] * UP + gl + m * G] = pp[s][m];
              }
            }
            if (k <= iters[s] && !down[s]) {
              if (EXACT) {
                if (gl == 0) {
                  hist[(sys[s] * Kmax + (k - 1)) * 2 + 0] = alpha[s];
                  hist[(sys[s] * Kmax + (k - 1)) * 2 + 1] = beta[s];
                }
              } else {
                // Eq. (11) on the diagonal (detect.cpp:409-427)
#pragma unroll
                for (int m = 0; m < RU; ++m) {
                  float nf;
                  if (k == 1) {
                    nf = alpha[s];
                  } else {
                    const float c1 = alpha[s] * (1.f + bm1[s]) / am1[s];
                    const float c2 = alpha[s] * bm2[s] / am2[s];
                    const float d1 = f0[s][m] - f1[s][m], d2 = f1[s][m] - f2[s][m];
                    nf = f0[s][m] + (c1 - alpha[s] * (gdiag[m] + reg[s])) * d1 - c2 * d2;
                  }
                  f2[s][m] = f1[s][m];
                  f1[s][m] = f0[s][m];
                  f0[s][m] = nf;
                }
              }
            }
            if (k <= iters[s]) {
              am2[s] = am1[s]; am1[s] = alpha[s];
              bm2[s] = bm1[s]; bm1[s] = beta[s];
            }
          }
          __syncwarp();
        }
        // ------------------------------------------ per-system epilogue
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (!live[s]) continue;
          if (gl == 0) sys_st[sys[s]] = broke[s] ? 1 : 0;
          if (EXACT || down[s]) {
#pragma unroll
            for (int m = 0; m < RU; ++m) Vs[sys[s] * UP + gl + m * G] = v[s][m];
            continue;
          }
          // approx uplink: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
          // then the LLR epilogue and stores straight from the lane
          if constexpr (!EXACT)
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            const int u = gl + m * G;
            if (u >= U) continue;
            const long o = (sc * S + sys[s]) * static_cast<long>(U) + u;
            const bool ok = !broke[s];
            const float2 xh = ok ? v[s][m] : make_float2(0.f, 0.f);
            const float mu_u = ok ? f0[s][m] * gdiag[m] : 0.f;
            const float rho_u = ok ? gdiag[m] / p.n0 : 0.f;
            if (p.xhat) p.xhat[o] = xh;
            if (p.mu) p.mu[o] = mu_u;
            if (p.rho) p.rho[o] = rho_u;
            if (p.llr) store_llrs(xh, ok ? mu_u : 0.f, rho_u, p.bits, p.llr + o * p.bits);
          }
        }
      }
    }
    if (!EXACT && p.status && S > 0) {
      __syncthreads();
      for (int s = tid; s < S; s += NT) p.status[sc * S + s] = sys_st[s];
    }

    // ------------------------------- phase 3: exact tracker, shared basis
    if (EXACT && S > 0) {
      __syncthreads();
      const int K = p.K;
      if (warp == 0) {
        const float2 cd = cheb_interval<UP>(Gs, p.rho_inv_u, Tb, lane);  // Tb: scratch here
        if (lane == 0) { misc[0] = cd.x; misc[1] = cd.y; }
      }
      __syncthreads();
      const float cc = misc[0], dd = misc[1];
      const float invd = 1.f / dd;
      for (int e = tid; e < UP * UP; e += NT) {  // T_1 = (A - cI)/d
        const int i = e / UP, j = e - i * UP;
        float2 a = Gs[e];
        if (i == j) a.x += p.rho_inv_u - cc;
        Tb[e] = cscale(invd, a);
      }
      // per-system coefficient recursion in FP64 (detect.cpp:336-368 on
      // coefficients), then B = L (A - rho^-1 I) (detect.cpp:215, :379)
      for (int s = tid; s < S; s += NT) {
        double l0[kMaxK + 2], l1[kMaxK + 2], l2[kMaxK + 2], tmp[kMaxK + 2], d1[kMaxK + 2];
        const int n = K + 2;
        for (int m = 0; m < n; ++m) l0[m] = l1[m] = l2[m] = 0.0;
        double a_m1 = 1.0, a_m2 = 1.0, b_m1 = 0.0, b_m2 = 0.0;
        auto mulA = [&](const double* x, double* out) {
          // A T_0 = c T_0 + d T_1;  A T_m = c T_m + d/2 (T_{m+1} + T_{m-1})
          for (int m = 0; m < n; ++m) out[m] = static_cast<double>(cc) * x[m];
          for (int m = 0; m < n; ++m) {
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
            l0[0] = a;  // L_1 = alpha_1 I
          } else {
            const double c1 = a * (1.0 + b_m1) / a_m1, c2 = a * b_m2 / a_m2;
            for (int m = 0; m < n; ++m) d1[m] = l0[m] - l1[m];
            mulA(d1, tmp);
            for (int m = 0; m < n; ++m) {
              const double nx = l0[m] + c1 * d1[m] - a * tmp[m] - c2 * (l1[m] - l2[m]);
              l2[m] = l1[m];
              l1[m] = l0[m];
              l0[m] = nx;
            }
          }
          a_m2 = a_m1; a_m1 = a; b_m2 = b_m1; b_m1 = bb;
        }
        mulA(l0, tmp);
        float* cl = coef + s * 2 * (K + 2);
        float* cb = cl + (K + 2);
        for (int m = 0; m < n; ++m) {
          cl[m] = static_cast<float>(l0[m]);
          cb[m] = static_cast<float>(tmp[m] - static_cast<double>(p.rho_inv_u) * l0[m]);
        }
      }
      __syncthreads();
      // T_{m+1} = 2 T_1 T_m - T_{m-1}, lower tiles + mirror (T_m Hermitian)
      for (int m = 1; m < K; ++m) {
        const float2* T1 = Tb;
        const float2* Tm = Tb + (m - 1) * UP * UP;
        float2* Tn = Tb + m * UP * UP;
        const float2* Tp = m >= 2 ? Tb + (m - 2) * UP * UP : nullptr;
        tile_pass<NT>(n_gram, 0, 1, T1, UP, Tm, UP, T1, 1, 1, UP,
                      [&](int, int ib, int jb, float2 (&acc)[4][4]) {
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                          for (int c = 0; c < 4; ++c) {
                            const int i = ib * 4 + r, j = jb * 4 + c;
                            if (j > i) continue;
                            const float2 prev =
                                Tp ? Tp[i * UP + j] : make_float2(i == j ? 1.f : 0.f, 0.f);
                            const float2 val = make_float2(2.f * acc[r][c].x - prev.x,
                                                           2.f * acc[r][c].y - prev.y);
                            if (i == j) {
                              Tn[i * UP + i] = make_float2(val.x, 0.f);
                            } else {
                              Tn[i * UP + j] = val;
                              Tn[j * UP + i] = cconj(val);
                            }
                          }
                      });
        __syncthreads();
      }
      // extraction (detect.cpp:375-395): thread <-> (row i, system subset);
      // the T_m entries of (i, j) are loaded once and reused by the subset
      {
        constexpr int RG = NT / UP > 0 ? NT / UP : 1;
        const int i = tid % UP, g = tid / UP;
        if (g < RG) {
          constexpr int SMAX = (kMaxSys + RG - 1) / RG;
          float ib2[SMAX], ibl[SMAX], mu_i[SMAX];
          int ns = 0;
          for (int s = g; s < S; s += RG) ++ns;
#pragma unroll
          for (int t = 0; t < SMAX; ++t) ib2[t] = ibl[t] = mu_i[t] = 0.f;
          for (int j = 0; j < UP; ++j) {
            float2 tv[kMaxK];
            for (int m = 1; m <= K; ++m) tv[m - 1] = cconj(Tb[(m - 1) * UP * UP + j * UP + i]);
#pragma unroll
            for (int t = 0; t < SMAX; ++t) {
              if (t >= ns) break;
              const int s = g + t * RG;
              const float* cl = coef + s * 2 * (K + 2);
              const float* cb = cl + (K + 2);
              float2 Bij = make_float2(i == j ? cb[0] : 0.f, 0.f);
              float2 Lij = make_float2(i == j ? cl[0] : 0.f, 0.f);
              for (int m = 1; m <= K; ++m) {
                Bij.x = fmaf(cb[m], tv[m - 1].x, Bij.x);
                Bij.y = fmaf(cb[m], tv[m - 1].y, Bij.y);
                if (m < K) {
                  Lij.x = fmaf(cl[m], tv[m - 1].x, Lij.x);
                  Lij.y = fmaf(cl[m], tv[m - 1].y, Lij.y);
                }
              }
              if (j == i) mu_i[t] = Bij.x;
              else ib2[t] += cnorm(Bij);
              ibl[t] += Bij.x * Lij.x + Bij.y * Lij.y;  // Re(B_ij conj(L_ij))
            }
          }
#pragma unroll
          for (int t = 0; t < SMAX; ++t) {
            if (t >= ns) break;
            const int s = g + t * RG;
            const float nu2 = ib2[t] * p.es + ibl[t] * p.n0;
            MUs[s * UP + i] = mu_i[t];
            RHOs[s * UP + i] = nu2 <= 0.f ? 0.f : mu_i[t] * mu_i[t] / nu2;  // safe_rho
          }
        }
      }
      __syncthreads();
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
        if (p.llr) store_llrs(xh, m, rr, p.bits, p.llr + o * p.bits);
      }
      if (p.status)
        for (int s = tid; s < S; s += NT) p.status[sc * S + s] = sys_st[s];
    }

    // ------------------------------------- phase 5: precode q = H_d^H v
    // q_b = sum_u H_u[b][u] v_u (precode.cpp:69, linalg.cpp:116-126): 4 rows
    // b x 4 systems register tiles, u rotated per lane to spread banks;
    // then gain = ||q||, s = q / gain, zero_input when ||q|| vanishes (:22-36)
    if (St > 0) {
      __syncthreads();
      const int nbb = (B + 3) / 4, nss = (St + 3) / 4;
      for (int t = tid; t < nbb * nss; t += NT) {
        const int bb = t % nbb, sb = t / nbb;
        float2 acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
        int brow[4], srow[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) brow[r] = min(bb * 4 + r, B - 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) srow[c] = S + min(sb * 4 + c, St - 1);
#pragma unroll 4
        for (int u0 = 0; u0 < UP; ++u0) {
          const int u = (u0 + lane) & (UP - 1);
          float2 h[4], vv[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) h[r] = Hs[brow[r] * UP + u];
#pragma unroll
          for (int c = 0; c < 4; ++c) vv[c] = Vs[srow[c] * UP + u];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) cfma(acc[r][c], h[r], vv[c]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int b = bb * 4 + r, s = sb * 4 + c;
            if (b < B && s < St) Qs[s * B + b] = acc[r][c];
          }
      }
      __syncthreads();
      for (int ts = warp; ts < St; ts += NW) {
        const int sys = S + ts;
        const bool ok = sys_st[sys] == 0;
        float nrm = 0.f;
        for (int b = lane; b < B; b += 32) nrm += cnorm(Qs[ts * B + b]);
        nrm = group_sum<32>(nrm);
        const float g = sqrtf(nrm);
        const bool zero = ok && !(g > 0.f);
        const float inv = (ok && !zero) ? 1.f / g : 0.f;
        const long ob = (sc * St + ts) * static_cast<long>(B);
        for (int b = lane; b < B; b += 32) {
          const float2 q = Qs[ts * B + b];
          if (p.q) p.q[ob + b] = ok ? q : make_float2(0.f, 0.f);
          if (p.s_out) p.s_out[ob + b] = cscale(inv, q);
        }
        if (lane == 0) {
          if (p.gain) p.gain[sc * St + ts] = (ok && !zero) ? g : 0.f;
          if (p.pstatus) p.pstatus[sc * St + ts] = ok ? (zero ? 2 : 0) : 1;
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace cgm
