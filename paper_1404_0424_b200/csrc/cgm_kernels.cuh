// cgm_kernels.cuh -- shared device code of the sm_100a kernels: the kernel
// parameter block, the Gray-QAM axis tables, the max-log LLR demapper
// (compute_llrs, detect.cpp:57-86), the Chebyshev interval of the exact
// tracker (power iteration on A = G + rho^-1 I), the FP64 coefficient form
// of its three-term recursion (detect.cpp:336-368), and the 4 x 4 register
// tile passes of the Gram / matched-filter kernels.
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
  long n_sc;
  int B, U, S, St, K, Kt, bits;
  int hd_layout;  // 1: H is the downlink matrix [U][B] (precode only)
  int use_tma;    // bulk-copy staging (U == UP, B even, 16B aligned)
  int exact;      // uplink systems use the exact tracker (the workspace carries the row moments)
  int fx;         // exact, one vector per subcarrier: the CG runs before moments_kernel<..., FX>
  int zs;         // transmit-vector slots in the workspace (separate precoder kernel), else 0
  float rho_inv_u, rho_inv_d, n0, es;
  float2* ws;     // split path: per-subcarrier workspace (G, MF, (c, d), row moments)
  long sc_base;   // split path: first subcarrier of this chunk
  int k1_pair, k1_spl, k1_wpp;  // channel kernel: staging depth, k-parts, warps
  int method;                   // sim::Method order: 0 Cholesky, 1 CG, 2 CGLS, 3 Neumann (cgm_alt.cuh)
};

// Per-axis Gray amplitude subsets (constellation.cpp:75-84), [qam][p][k],
// qam 0/1/2 = QPSK/16/64.
struct AxisTables {
  float a0[3][3][4];
  float a1[3][3][4];
  float lv[3][8];  // per-axis amplitudes in ascending order (level k <-> Gray label k^(k>>1))
};
__constant__ AxisTables c_axis;

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
      // ratios of the CG's FP32 step lengths, in FP32: an FP64 division is a
      // long dependent sequence on this recursion's critical path
      const double c1 = static_cast<double>(__fdividef(static_cast<float>(a * (1.0 + b_m1)),
                                                       static_cast<float>(a_m1)));
      const double c2 = static_cast<double>(__fdividef(static_cast<float>(a * b_m2),
                                                       static_cast<float>(a_m2)));
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

// Power iteration for lambda_max(A), A = G + reg I: x_0 = 1, x_{t+1} = A x_t
// / tr(A) (tr(A) >= lambda_max, so the iterates neither overflow nor, in six
// steps of at most a factor U, underflow), lambda = the Rayleigh quotient
// x_6^H A x_6 / x_6^H x_6; one warp reduction for the trace and one for the
// quotient, none inside the chain.  Interval [reg, 1.1 lambda] -> (c, d).
template <int UP, int LDG = UP>
__device__ __forceinline__ float2 cheb_interval(const float2* Gs, float reg, float2* xs, int lane) {
  float lam = reg;
  if constexpr (UP < 32) {
    // U <= 16: the 32 / UP lane groups each take UP / (32 / UP) columns of
    // the matvec for row i = lane mod UP and the partial sums are combined by
    // xor shuffles (every group ends with the same bits), instead of UP lanes
    // walking all UP columns while the rest of the warp idles
    constexpr int GPW = 32 / UP, NC = UP / GPW;
    const int part = lane / UP, i = lane - part * UP;
    float2 xr = make_float2(1.f, 0.f);
    if (part == 0) xs[i] = xr;
    const float tr = group_sum<UP>(Gs[i * LDG + i].x + reg);
    const float itr = tr > 0.f ? 1.f / tr : 1.f;
    __syncwarp();
    for (int it = 0; it <= 6; ++it) {
      float2 y = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) {
        const int j = part * NC + jj;
        cfma_conj(y, Gs[j * LDG + i], xs[j]);  // (A x)_i = sum_j conj(G[j][i]) x_j
      }
#pragma unroll
      for (int o = UP; o < 32; o <<= 1) {
        y.x += __shfl_xor_sync(0xffffffffu, y.x, o);
        y.y += __shfl_xor_sync(0xffffffffu, y.y, o);
      }
      y.x = fmaf(reg, xr.x, y.x);
      y.y = fmaf(reg, xr.y, y.y);
      if (it == 6) {
        const float nx = group_sum<UP>(cnorm(xr));
        const float ray = group_sum<UP>(xr.x * y.x + xr.y * y.y);
        if (nx > 0.f) lam = ray / nx;
        break;
      }
      __syncwarp();
      xr = cscale(itr, y);
      if (part == 0) xs[i] = xr;
      __syncwarp();
    }
  } else {
  constexpr int RU = UP < 32 ? 1 : UP / 32;
  float2 xr[RU];
  float tr = 0.f;
#pragma unroll
  for (int m = 0; m < RU; ++m) {
    const int i = lane + 32 * m;
    xr[m] = make_float2(i < UP ? 1.f : 0.f, 0.f);
    if (i < UP) {
      xs[i] = xr[m];
      tr += Gs[i * LDG + i].x + reg;
    }
  }
  tr = group_sum<32>(tr);
  const float itr = tr > 0.f ? 1.f / tr : 1.f;
  __syncwarp();
  for (int it = 0; it <= 6; ++it) {
    float2 y[RU];
    float nx = 0.f, ray = 0.f;
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
      nx += cnorm(xr[m]);
      ray += xr[m].x * y[m].x + xr[m].y * y[m].y;
    }
    if (it == 6) {
      nx = group_sum<32>(nx);
      ray = group_sum<32>(ray);
      if (nx > 0.f) lam = ray / nx;
      break;
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < RU; ++m) {
      const int i = lane + 32 * m;
      xr[m] = cscale(itr, y[m]);
      if (i < UP) xs[i] = xr[m];
    }
    __syncwarp();
  }
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

}  // namespace cgm
