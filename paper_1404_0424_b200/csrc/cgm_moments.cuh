// cgm_moments.cuh -- the exact SINR tracker through row moments of a
// shared Chebyshev basis.
//
// The reference's exact tracker (ExactSinrTracker, detect.cpp:330-368) runs
// a three-term matrix recursion per received vector and extracts
// (tracker_exact_extract, detect.cpp:370-395), with G = A - rho^-1 I,
//   B     = L_K G
//   mu_i  = Re B_ii
//   nu2_i = Es sum_{j != i} |B_ij|^2 + N0 Re sum_j B_ij conj(L_ij)
// L_k is a real-coefficient polynomial in A (the recursion only ever
// multiplies by A and adds scaled identities), so L_K and B are too.  In
// the Chebyshev basis T_m = T_m(Ahat), Ahat = (A - cI)/d:
//   L = sum_n l_n T_n  (degree K-1),   B = sum_m g_m T_m  (degree K)
// with the coefficients l, g per vector (cheb_coef_warp: the reference's
// recursion run on coefficients, FP64).  Write E = B - g_0 I, F = L - l_0 I.
// The T_m commute and are Hermitian, so every quantity above is a diagonal
// entry of a polynomial in Ahat:
//   mu_i  = g_0 + e_i,                         e_i = sum_{m>=1} g_m D_m[i]
//   L_ii  = l_0 + f_i,                         f_i = sum_{n>=1} l_n D_n[i]
//   sum_{j!=i} |B_ij|^2          = (E E)_ii - e_i^2
//   Re sum_j B_ij conj(L_ij)     = mu_i L_ii + (E F)_ii - e_i f_i
// where D_k[i] = (T_k)_ii and (E E)_ii = sum_k ee_k D_k[i], (E F)_ii =
// sum_k ef_k D_k[i] with ee, ef the Chebyshev products of the coefficient
// vectors (T_a T_b = (T_{a+b} + T_{|a-b|}) / 2).  So everything a vector
// needs from the channel is D_k[i], k = 0..2K, per row i -- a (2K+1) x U
// table per SUBCARRIER -- and the per-vector extraction costs O(K^2 + K U)
// instead of the reference's O(K U^3) recursion and U^3 extraction.
//
// The table comes from the row products of the basis matrices: with the
// window T_{a-1}, T_a of the recursion T_{a+1} = 2 Ahat T_a - T_{a-1},
//   D_{2a}   = 2 sum_j |T_a[i][j]|^2 - 1
//   D_{2a-1} = 2 Re sum_j T_a[i][j] conj(T_{a-1}[i][j]) - D_1
// for a = 1..K: K - 1 Hermitian products per subcarrier (lower tiles +
// mirror), only three matrices resident.  The identity part g_0 I (the
// O(1) part of B) never enters the interference sum, so the subtraction
// (E E)_ii - e_i^2 works on small numbers.  FP32 products hold the 1e-3
// contract with margin up to K = 8 (tools/moments_study.py: rho within
// 4e-5 of the FP64 reference on every BASELINE shape, incl. the correlated
// cfg5 channel); for K > 8 the products run in FP64 (K = 16 at 28 dB:
// 1.6e-6, FP32 would give 2e-3).
#pragma once

#include <type_traits>

#include "cgm_kernels.cuh"

namespace cgm {

// split-path workspace layout per subcarrier (float2 units): G (UP x UP,
// full Hermitian), the S matched filters, (c, d) of the Chebyshev interval,
// and for the exact tracker the row-moment table D_k[i] (double, k = 0..2K)
// fx (exact, one vector per subcarrier): instead of the moment table, the
// CG's (alpha, beta) history (K float2), v_K (UP float2) and the breakdown
// flag (1 float2) for moments_kernel<..., FX>.  zs (St > 0 and a separate
// precoder kernel, precode_q_kernel): each transmit vector's v_K (UP float2)
// and its breakdown flag (one float2 per vector after the St rows).  The
// span [g, z) is contiguous for one bulk copy.
struct WsOffsets {
  int g, mf, cd, t, z, stride;
  __host__ __device__ void plan(int UP, int S, int K, bool exact, bool fx = false, int zs = 0) {
    g = 0;
    mf = UP * UP;
    cd = mf + S * UP;
    t = cd + 2;
    z = t + (exact ? (fx ? K + UP + 1 : (2 * K + 1) * UP) : 0);
    z = (z + 1) & ~1;
    stride = z + zs * (UP + 1);
    stride = (stride + 1) & ~1;
  }
};

// per subcarrier in the workspace: (c, d) at W.cd, D_k[i] (double) at W.t:
// mom[k * UP + i], k = 0..2K
__host__ __device__ inline int moments_words(int UP, int K) { return (2 * K + 1) * UP; }

template <int UP>
struct MomGeo {
  static constexpr int NB = UP / 4;                 // tile rows
  static constexpr int NTILE = NB * (NB + 1) / 2;   // lower-triangle tiles
  static constexpr int SPC = UP == 8 ? 32 : UP == 16 ? 8 : UP == 32 ? 2 : 1;  // subcarriers per CTA
  static constexpr int NT = ((SPC * NTILE + 31) / 32) * 32 < 64 ? 64 : ((SPC * NTILE + 31) / 32) * 32;
  static constexpr int LD = UP + 2;                 // padded row (bank spread, 16 B aligned)
  static constexpr int MAT = UP * LD;               // complex entries per matrix
  static constexpr int PART = 4 * UP * NB;          // row / column partial slots (in R), 2 sums each
  // per subcarrier: Ahat and the current T_a (the previous T_{a-1} stays in
  // the tile threads' registers), plus the partial slots
  template <class R>
  __host__ __device__ static constexpr int slot_bytes() {
    return 2 * MAT * 2 * static_cast<int>(sizeof(R)) + PART * static_cast<int>(sizeof(R));
  }
  template <class R>
  __host__ __device__ static constexpr int smem() { return SPC * slot_bytes<R>(); }
};

template <class R>
struct Cx;
template <>
struct Cx<float> { using T = float2; };
template <>
struct Cx<double> { using T = double2; };

// acc[r][c] = sum_k Ahat[i0 + r][k] T[k][j0 + c] for one 4 x 4 tile (Ahat
// Hermitian: row i0 + r of Ahat is the conjugate of column i0 + r, read
// along rows k of the padded smem matrix).  FP32: one packed accumulator per
// entry, conj(a) t = t * a.x + swap(t) * (a.y, -a.y) (swap / negation are
// FFMA2 operand modifiers); FP64: plain DFMA.
template <int UP>
__device__ __forceinline__ void tile_prod(const float2* A, const float2* T, int i0, int j0,
                                          float2 (&out)[4][4]) {
  constexpr int LD = MomGeo<UP>::LD;
  unsigned long long acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0ull;
  auto ld = [&](int k, ulonglong2 (&av)[2], ulonglong2 (&tv)[2]) {
    av[0] = *reinterpret_cast<const ulonglong2*>(A + k * LD + i0);
    av[1] = *reinterpret_cast<const ulonglong2*>(A + k * LD + i0 + 2);
    tv[0] = *reinterpret_cast<const ulonglong2*>(T + k * LD + j0);
    tv[1] = *reinterpret_cast<const ulonglong2*>(T + k * LD + j0 + 2);
  };
  ulonglong2 av[2], tv[2];
  ld(0, av, tv);
#pragma unroll 2
  for (int k = 0; k < UP; ++k) {
    const unsigned long long ah[4] = {av[0].x, av[0].y, av[1].x, av[1].y};
    const unsigned long long t[4] = {tv[0].x, tv[0].y, tv[1].x, tv[1].y};
    if (k + 1 < UP) ld(k + 1, av, tv);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2 a2 = f2unpack(ah[r]);
      const unsigned long long ax = f2pack(a2.x, a2.x), ay = f2pack(a2.y, -a2.y);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ffma2(acc[r][c], t[c], ax);
        ffma2(acc[r][c], f2swap_hl(t[c]), ay);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) out[r][c] = f2unpack(acc[r][c]);
}

template <int UP>
__device__ __forceinline__ void tile_prod(const double2* A, const double2* T, int i0, int j0,
                                          double2 (&out)[4][4]) {
  constexpr int LD = MomGeo<UP>::LD;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) out[r][c] = make_double2(0.0, 0.0);
#pragma unroll 2
  for (int k = 0; k < UP; ++k) {
    double2 a[4], t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = A[k * LD + i0 + q];
      t[q] = T[k * LD + j0 + q];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // conj(a) t
        out[r][c].x = fma(a[r].x, t[c].x, fma(a[r].y, t[c].y, out[r][c].x));
        out[r][c].y = fma(a[r].x, t[c].y, fma(-a[r].y, t[c].x, out[r][c].y));
      }
  }
}

// moments_kernel: per subcarrier (SPC per CTA), from G in the workspace:
// (c, d) by power iteration (cheb_interval), Ahat, the K - 1 products of the
// Chebyshev recursion, and
//   FX = false: D_k[i], k = 0..2K, into the workspace (any S);
//   FX = true (one vector per subcarrier, S = 1): the CG kernel ran first and
//     left its (alpha, beta) history, v_K and status in the workspace; the
//     coefficients of L_K and B are formed here and every tile thread
//     accumulates its entries of B = sum g_m T_m and L = sum l_m T_m while the
//     products produce T_2..T_K, then the extraction (detect.cpp:375-395) and
//     the LLRs finish in this kernel.  With a single vector the per-vector
//     U^3 work is unavoidable, and the entrywise sums keep FP32 accurate to
//     K = 16 (the moment table's quadratic forms need FP64 products from
//     K = 7 on).
// Only Ahat and the current T_a live in shared memory: each tile thread
// keeps its own entries of T_{a-1} in registers (the recursion's "prev"
// term only needs the thread's own tile), and the row sums behind D_k come
// from the tiles too -- per lower entry, |T_{a+1}|^2 and Re T_{a+1} conj(T_a)
// count for row i and (mirror, i != j) for row j -- through fixed slots
// summed in a fixed order, so no separate row pass serialises the CTA.
template <int UP, class R, bool FX = false>
__global__ void __launch_bounds__(MomGeo<UP>::NT, UP == 32 ? 4 : 2) moments_kernel(const KernelParams p) {
  using MG = MomGeo<UP>;
  using C = typename Cx<R>::T;
  static_assert(!FX || std::is_same<R, float>::value, "FX runs in FP32");
  constexpr int MAT = MG::MAT, SPC = MG::SPC, LD = MG::LD, NT = MG::NT, NB = MG::NB;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = p.K;
  WsOffsets W;
  W.plan(UP, p.S, K, true, FX, p.zs);
  const long sc0 = static_cast<long>(blockIdx.x) * SPC;
  const int nsc = static_cast<int>(p.n_sc - sc0 < SPC ? p.n_sc - sc0 : SPC);
  auto slotp = [&](int s) { return smem + s * MG::template slot_bytes<R>(); };
  auto Abuf = [&](int s) { return reinterpret_cast<C*>(slotp(s)); };            // Ahat
  auto Tbuf = [&](int s) { return reinterpret_cast<C*>(slotp(s)) + MAT; };      // T_a
  // partial row sums in R: FP64 products need FP64 sums (K > 6)
  auto Part = [&](int s) { return reinterpret_cast<R*>(slotp(s) + 2 * MAT * sizeof(C)); };
  // G -> the T buffer as padded float2 rows (16-byte cp.async chunks,
  // coalesced reads); the power iteration reads it there
  for (int s = 0; s < nsc; ++s) {
    const float2* src = p.ws + (sc0 + s) * W.stride + W.g;
    float2* dst = reinterpret_cast<float2*>(Tbuf(s));
    for (int e = tid; e < UP * UP / 2; e += NT) {
      const int r = e / (UP / 2), c2 = e - r * (UP / 2);
      cp_async16(dst + r * LD + 2 * c2, src + 2 * e);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  __shared__ float2 cds[SPC];
  // FX: the Chebyshev coefficients of L_K and B per subcarrier (cl, cb)
  __shared__ float coefs[FX ? SPC : 1][2][kMaxK + 2];
  if constexpr (SPC == 1) {
    // one subcarrier per CTA (U = 64): the power iteration of cheb_interval
    // on 2 U threads (row i, half of the columns each), so the other warps
    // do not idle behind one warp's 7 sequential U x U products
    if (nsc > 0) {
      const float2* Gs = reinterpret_cast<const float2*>(Tbuf(0));
      float2* xs = reinterpret_cast<float2*>(Abuf(0));  // scratch: x, then the two half products
      float2* yp = xs + UP;
      float* rd = reinterpret_cast<float*>(yp + 2 * UP);  // [warps][2]
      const float reg = p.rho_inv_u;
      // iterates scaled by 1 / tr(A) (>= lambda_max) instead of normalised:
      // one CTA reduction for the trace, one for the final Rayleigh quotient
      float itr;
      {
        float t = tid < UP ? Gs[tid * LD + tid].x + reg : 0.f;
        t = group_sum<32>(t);
        if (lane == 0 && warp < UP / 32) rd[warp * 2] = t;
        __syncthreads();
        t = 0.f;
        for (int w = 0; w < UP / 32; ++w) t += rd[w * 2];  // fixed order
        itr = t > 0.f ? 1.f / t : 1.f;
      }
      float2 xr = make_float2(tid < UP ? 1.f : 0.f, 0.f);
      if (tid < UP) xs[tid] = xr;
      __syncthreads();
      float lam = reg;
      for (int it = 0; it <= 6; ++it) {
        if (tid < 2 * UP) {
          const int i = tid % UP, h = tid / UP;
          float2 y4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};  // four independent chains
#pragma unroll
          for (int j = h * (UP / 2); j < (h + 1) * (UP / 2); j += 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) cfma_conj(y4[q], Gs[(j + q) * LD + i], xs[j + q]);
          }
          yp[h * UP + i] = cadd(cadd(y4[0], y4[1]), cadd(y4[2], y4[3]));
        }
        __syncthreads();
        float2 y = make_float2(0.f, 0.f);
        if (tid < UP) {
          y = cadd(yp[tid], yp[UP + tid]);
          y.x = fmaf(reg, xr.x, y.x);
          y.y = fmaf(reg, xr.y, y.y);
        }
        if (it == 6) {
          float nx = tid < UP ? cnorm(xr) : 0.f, ray = tid < UP ? xr.x * y.x + xr.y * y.y : 0.f;
          nx = group_sum<32>(nx);
          ray = group_sum<32>(ray);
          if (lane == 0 && warp < UP / 32) {
            rd[warp * 2] = nx;
            rd[warp * 2 + 1] = ray;
          }
          __syncthreads();
          nx = 0.f;
          ray = 0.f;
          for (int w = 0; w < UP / 32; ++w) {  // fixed order
            nx += rd[w * 2];
            ray += rd[w * 2 + 1];
          }
          if (nx > 0.f) lam = ray / nx;
          break;
        }
        if (tid < UP) {
          xr = cscale(itr, y);
          xs[tid] = xr;
        }
        __syncthreads();
      }
      if (warp == 0) {
        const float lo = reg;
        const float hi = fmaxf(1.1f * lam, 1.0001f * lo);
        const float c = 0.5f * (lo + hi);
        float d = 0.5f * (hi - lo);
        if (!(d > 1e-6f * fmaxf(fabsf(c), 1e-30f))) d = fmaxf(fabsf(c), 1.f);
        const float2 cd = make_float2(c, d);
        if (lane == 0) {
          cds[0] = cd;
          p.ws[sc0 * W.stride + W.cd] = cd;
        }
        if constexpr (FX) {
          const float2* hw = p.ws + sc0 * W.stride + W.t;  // K (alpha, beta) pairs
          cheb_coef_warp(reinterpret_cast<const float*>(hw), K, cd.x, cd.y, p.rho_inv_u,
                         coefs[0][0], coefs[0][1]);
        }
      }
    }
  } else
  for (int s = warp; s < nsc; s += NT / 32) {
    // power-iteration scratch: the A buffer (as float2)
    const float2 cd = cheb_interval<UP, LD>(reinterpret_cast<const float2*>(Tbuf(s)),
                                            p.rho_inv_u, reinterpret_cast<float2*>(Abuf(s)), lane);
    if (lane == 0) {
      cds[s] = cd;
      p.ws[(sc0 + s) * W.stride + W.cd] = cd;
    }
    if constexpr (FX) {
      const float2* hw = p.ws + (sc0 + s) * W.stride + W.t;  // K (alpha, beta) pairs
      cheb_coef_warp(reinterpret_cast<const float*>(hw), K, cd.x, cd.y, p.rho_inv_u,
                     coefs[s][0], coefs[s][1]);
    }
  }
  __syncthreads();
  // Ahat = (A - cI)/d = (G + (rho^-1 - c) I) / d -> A buffer (in R)
  for (int e = tid; e < nsc * UP * UP; e += NT) {
    const int s = e / (UP * UP), r = (e / UP) % UP, c = e % UP;
    const float2 g = reinterpret_cast<const float2*>(Tbuf(s))[r * LD + c];
    const R cc = cds[s].x, invd = R(1) / static_cast<R>(cds[s].y);
    R x = g.x, y = g.y;
    if (r == c) {
      x += static_cast<R>(p.rho_inv_u) - cc;
      y = R(0);
    }
    C v;
    v.x = x * invd;
    v.y = y * invd;
    Abuf(s)[r * LD + c] = v;
  }
  __syncthreads();
  // thread <-> (subcarrier slot, lower tile)
  const int slot = tid / MG::NTILE;
  const int tile = tid - slot * MG::NTILE;
  int rb = 0;
  while ((rb + 1) * (rb + 2) / 2 <= tile) ++rb;
  const int cb = tile - rb * (rb + 1) / 2;
  const bool busy = slot < nsc;
  const int i0 = rb * 4, j0 = cb * 4;
  const int ss = busy ? slot : 0;
  // this tile's entries of T_{a-1} (prv) stay in registers; T_0 = I
  C prv[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      prv[r][c].x = (i0 + r == j0 + c) ? R(1) : R(0);
      prv[r][c].y = R(0);
    }
  auto load_tile = [&](const C* M, C (&t)[4][4]) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) t[r][c] = M[(i0 + r) * LD + j0 + c];
  };
  double* mom = reinterpret_cast<double*>(p.ws + (sc0 + ss) * W.stride + W.t);
  // row / column partials of the tile's lower entries: [row][NB][2]
  auto partials = [&](const C (&nw)[4][4], const C (&ol)[4][4], bool cross) {
    R* Rp = Part(ss);
    R* Cp = Rp + 2 * UP * NB;
    R rn[4] = {0, 0, 0, 0}, rx[4] = {0, 0, 0, 0};
    R cn[4] = {0, 0, 0, 0}, cx[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + r, j = j0 + c;
        if (j > i) continue;
        const R n2 = nw[r][c].x * nw[r][c].x + nw[r][c].y * nw[r][c].y;
        const R x2 = cross ? nw[r][c].x * ol[r][c].x + nw[r][c].y * ol[r][c].y : R(0);
        rn[r] += n2; rx[r] += x2;
        if (i != j) { cn[c] += n2; cx[c] += x2; }
      }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      Rp[((i0 + r) * NB + cb) * 2 + 0] = rn[r];
      Rp[((i0 + r) * NB + cb) * 2 + 1] = rx[r];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      Cp[((j0 + c) * NB + rb) * 2 + 0] = cn[c];
      Cp[((j0 + c) * NB + rb) * 2 + 1] = cx[c];
    }
  };
  // fixed-order row sums of the partials -> D_{2a-1}, D_{2a} (thread = row)
  auto row_sums = [&](int a) {
    for (int e = tid; e < nsc * UP; e += NT) {
      const int s = e / UP, i = e - s * UP;
      const R* Rp = Part(s);
      const R* Cp = Rp + 2 * UP * NB;
      const int rbi = i / 4;
      double n2 = 0.0, x2 = 0.0;
      for (int q = 0; q <= rbi; ++q) { n2 += Rp[(i * NB + q) * 2]; x2 += Rp[(i * NB + q) * 2 + 1]; }
      for (int q = rbi; q < NB; ++q) { n2 += Cp[(i * NB + q) * 2]; x2 += Cp[(i * NB + q) * 2 + 1]; }
      double* m = reinterpret_cast<double*>(p.ws + (sc0 + s) * W.stride + W.t);
      const double d1 = static_cast<double>(Abuf(s)[i * LD + i].x);
      if (a == 1) {
        m[i] = 1.0;
        m[UP + i] = d1;
      } else {
        m[(2 * a - 1) * UP + i] = 2.0 * x2 - d1;
      }
      m[2 * a * UP + i] = 2.0 * n2 - 1.0;
    }
  };
  (void)mom;
  // FX: this tile's entries of B = sum_m cb_m T_m and L = sum_{m<K} cl_m T_m
  float2 Bacc[FX ? 4 : 1][FX ? 4 : 1], Lacc[FX ? 4 : 1][FX ? 4 : 1];
  if constexpr (FX) {
    const float* cl = coefs[ss][0];
    const float* cbq = coefs[ss][1];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const C a1 = Abuf(ss)[(i0 + r) * LD + j0 + c];
        const float2 t1 = make_float2(a1.x, a1.y);  // T_1
        const float d0 = (i0 + r == j0 + c) ? 1.f : 0.f;           // T_0 = I
        Bacc[r][c] = make_float2(cbq[0] * d0 + cbq[1] * t1.x, cbq[1] * t1.y);
        Lacc[r][c] = K > 1 ? make_float2(cl[0] * d0 + cl[1] * t1.x, cl[1] * t1.y)
                           : make_float2(cl[0] * d0, 0.f);
      }
  } else {
    if (busy) {  // D_2 from T_1 = Ahat
      C t1[4][4];
      load_tile(Abuf(ss), t1);
      partials(t1, prv, false);
    }
    __syncthreads();
    row_sums(1);
  }
  for (int a = 1; a < K; ++a) {
    // T_{a+1} = 2 Ahat T_a - T_{a-1}; T_a is Ahat itself for a = 1
    C nx[4][4];
    if (busy) {
      C acc[4][4];
      tile_prod<UP>(Abuf(slot), a == 1 ? Abuf(slot) : Tbuf(slot), i0, j0, acc);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = i0 + r, j = j0 + c;
          nx[r][c].x = R(2) * acc[r][c].x - prv[r][c].x;
          nx[r][c].y = i == j ? R(0) : R(2) * acc[r][c].y - prv[r][c].y;
        }
    }
    __syncthreads();  // every thread's reads of T_a are done: overwrite it with T_{a+1}
    if (busy) {
      C* Tn = Tbuf(slot);
      C cur[4][4];  // this tile's T_a, the next step's T_{a-1}
      load_tile(a == 1 ? Abuf(slot) : Tn, cur);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = i0 + r, j = j0 + c;
          if (j > i) continue;
          Tn[i * LD + j] = nx[r][c];
          if (i != j) {
            C cv;
            cv.x = nx[r][c].x;
            cv.y = -nx[r][c].y;
            Tn[j * LD + i] = cv;
          }
          if constexpr (FX) {  // T_{a+1} into this tile's B and L
            const float cbm = coefs[slot][1][a + 1];
            Bacc[r][c].x = fmaf(cbm, nx[r][c].x, Bacc[r][c].x);
            Bacc[r][c].y = fmaf(cbm, nx[r][c].y, Bacc[r][c].y);
            if (a + 1 < K) {
              const float clm = coefs[slot][0][a + 1];
              Lacc[r][c].x = fmaf(clm, nx[r][c].x, Lacc[r][c].x);
              Lacc[r][c].y = fmaf(clm, nx[r][c].y, Lacc[r][c].y);
            }
          }
        }
      if (!FX) partials(nx, cur, true);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) prv[r][c] = cur[r][c];
    }
    __syncthreads();  // T_{a+1} complete (and the partials)
    if (!FX) {
      row_sums(a + 1);
      __syncthreads();  // the partial slots are reused by the next step
    }
  }
  if constexpr (FX) {
    // ---------------- extraction (detect.cpp:375-395) from the tile sums:
    // per lower entry (i, j): |B_ij|^2 and Re(B_ij conj(L_ij)) count for row
    // i and (i != j, Hermitian) for row j; mu_i = Re B_ii.  Row parts go to
    // Rb[i][cb], column parts to Cb[j][rb] (each slot written by one tile),
    // summed in a fixed order.
    float* Rb = reinterpret_cast<float*>(Part(ss));  // [UP][NB][2]
    float* Cb = Rb + 2 * UP * NB;                    // [UP][NB][2]
    float* Mb = reinterpret_cast<float*>(Tbuf(ss));  // [UP] (T is dead now)
    if (busy) {
      float rr2[4] = {0.f, 0.f, 0.f, 0.f}, rrl[4] = {0.f, 0.f, 0.f, 0.f};
      float cc2[4] = {0.f, 0.f, 0.f, 0.f}, ccl[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = i0 + r, j = j0 + c;
          if (j > i) continue;
          const float2 b = Bacc[r][c], l = Lacc[r][c];
          const float wl = b.x * l.x + b.y * l.y;
          if (i == j) {
            Mb[i] = b.x;
            rrl[r] += wl;
          } else {
            const float w2 = cnorm(b);
            rr2[r] += w2; rrl[r] += wl;
            cc2[c] += w2; ccl[c] += wl;
          }
        }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        Rb[((i0 + r) * NB + cb) * 2 + 0] = rr2[r];
        Rb[((i0 + r) * NB + cb) * 2 + 1] = rrl[r];
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        Cb[((j0 + c) * NB + rb) * 2 + 0] = cc2[c];
        Cb[((j0 + c) * NB + rb) * 2 + 1] = ccl[c];
      }
    }
    __syncthreads();
    for (int e = tid; e < nsc * UP; e += NT) {
      const int s = e / UP, i = e - s * UP;
      if (i >= p.U) continue;
      const float* Rr = reinterpret_cast<const float*>(Part(s));
      const float* Cc = Rr + 2 * UP * NB;
      const float* M = reinterpret_cast<const float*>(Tbuf(s));
      const int rbi = i / 4;
      float ib2 = 0.f, ibl = 0.f;
      for (int q = 0; q <= rbi; ++q) { ib2 += Rr[(i * NB + q) * 2]; ibl += Rr[(i * NB + q) * 2 + 1]; }
      for (int q = rbi; q < NB; ++q) { ib2 += Cc[(i * NB + q) * 2]; ibl += Cc[(i * NB + q) * 2 + 1]; }
      const float2* wsx = p.ws + (sc0 + s) * W.stride;
      const bool ok = wsx[W.t + K + UP].x == 0.f;  // the CG's breakdown flag
      const long sc = p.sc_base + sc0 + s;           // S = 1: vector index == subcarrier
      const long o = sc * static_cast<long>(p.U) + i;
      const float mu_i = M[i];
      const float nu2 = ib2 * p.es + ibl * p.n0;
      const float mu = ok ? mu_i : 0.f;
      const float rho = ok ? (nu2 <= 0.f ? 0.f : mu_i * mu_i / nu2) : 0.f;  // safe_rho
      const float2 xh = ok ? wsx[W.t + K + i] : make_float2(0.f, 0.f);
      if (p.mu) p.mu[o] = mu;
      if (p.rho) p.rho[o] = rho;
      if (p.llr) store_llrs_fast(xh, mu, rho, p.bits, p.llr + o * p.bits);
    }
  }
}

// ------------------------------------------------- moments, warp per subcarrier
// U = 32, FP32 moment table (K <= 6), several vectors per subcarrier (not
// FX): the same (c, d) and D_k[i] as moments_kernel<32, float>, but one warp
// owns a subcarrier end to end with no block barriers: lane i keeps row i
// of G (then Ahat) in registers (conflict-free LDS.128 reads of the padded
// rows), runs the power iteration of cheb_interval on its row, and forms its
// part of every product T_{a+1} = 2 Ahat T_a - T_{a-1}: (Ahat T_a)[i][j] =
// sum_k Ahat[i][k] T_a[k][j], Ahat[i][k] from registers, two lanes per
// 16-byte chunk of row k of T_a (one LDS.128 per two j), 2 packed FFMA2 per
// complex MAC, a Hermitian band of 18 of the 32 columns per row (see below)
// -- every lane busy, no tile bookkeeping, no barriers; row i's moments |T_{a+1}[i][:]|^2 and
// Re T_{a+1}[i][:] . conj(T_a[i][:]) are summed by the lane in column
// order.  T_{a+1} overwrites T_{a-1}, so two padded U x U buffers per warp.
constexpr int kMrW = 4;  // warps (subcarriers) per CTA
struct MomRowsSmem {
  static constexpr int LD = 34;                  // padded row (float2): conflict-free LDS.128 per lane
  static constexpr int MAT = 32 * LD * 8;        // bytes
  static constexpr int PER_WARP = 2 * MAT + 32 * 8;  // T_a, T_{a-1/a+1}, power-iteration vector
  static constexpr int TOTAL = kMrW * PER_WARP;
};

__global__ void __launch_bounds__(32 * kMrW, 3) moments_rows32_kernel(const KernelParams p) {
  constexpr int UP = 32, LD = MomRowsSmem::LD;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, i = threadIdx.x & 31;
  const long lsc = static_cast<long>(blockIdx.x) * kMrW + warp;
  if (lsc >= p.n_sc) return;
  const int K = p.K;
  WsOffsets W;
  W.plan(UP, p.S, K, true, false, p.zs);
  unsigned char* base = smem + warp * MomRowsSmem::PER_WARP;
  float2* buf0 = reinterpret_cast<float2*>(base);
  float2* buf1 = reinterpret_cast<float2*>(base + MomRowsSmem::MAT);
  float2* xs = reinterpret_cast<float2*>(base + 2 * MomRowsSmem::MAT);
  float2* ws = p.ws + lsc * W.stride;
  // G row i -> registers (the workspace G is the full Hermitian matrix)
  ulonglong2 g[UP / 2];
  {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(ws + W.g + i * UP);
#pragma unroll
    for (int c = 0; c < UP / 2; ++c) g[c] = src[c];
  }
  // power iteration on A = G + reg I (cheb_interval: x_0 = 1, 7 products,
  // the Rayleigh quotient of x_6).  The iterates are scaled by 1 / tr(A)
  // (>= lambda_max, so no overflow; >= lambda_max / 32 per step, so no
  // underflow in 6 steps) instead of normalised, so only the last step
  // reduces over the warp: the per-step butterfly and rsqrt leave the chain.
  const float reg = p.rho_inv_u;
  float itr;
  {
    float dg = 0.f;
#pragma unroll
    for (int c = 0; c < UP / 2; ++c) {
      if (2 * c == i) dg = f2unpack(g[c].x).x;
      if (2 * c + 1 == i) dg = f2unpack(g[c].y).x;
    }
    float t = dg + reg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    itr = t > 0.f ? 1.f / t : 1.f;
  }
  float2 xr = make_float2(1.f, 0.f);
  xs[i] = xr;
  __syncwarp();
  float lam = reg;
  for (int it = 0; it <= 6; ++it) {
    // (Ax)_i = sum_j G[i][j] x_j: a += g x.x, b += g x.y, even / odd columns
    // in separate accumulators (half the dependent chain)
    unsigned long long a0 = 0ull, b0 = 0ull, a1 = 0ull, b1 = 0ull;
#pragma unroll
    for (int c = 0; c < UP / 2; ++c) {
      const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(xs + 2 * c);
      ffma2(a0, g[c].x, f2dup_lo(xv.x));
      ffma2(b0, g[c].x, f2dup_hi(xv.x));
      ffma2(a1, g[c].y, f2dup_lo(xv.y));
      ffma2(b1, g[c].y, f2dup_hi(xv.y));
    }
    const float2 A0 = f2unpack(a0), B0 = f2unpack(b0), A1 = f2unpack(a1), B1 = f2unpack(b1);
    float2 y = make_float2((A0.x - B0.y) + (A1.x - B1.y), (A0.y + B0.x) + (A1.y + B1.x));
    y.x = fmaf(reg, xr.x, y.x);
    y.y = fmaf(reg, xr.y, y.y);
    if (it == 6) {
      // ||x||^2 and Re x^H A x over the warp in one butterfly: lanes 0-15
      // carry the first sum, 16-31 the second after the xor-16 exchange
      const float v0 = cnorm(xr), v1 = xr.x * y.x + xr.y * y.y;
      const bool up = i & 16;
      float k = up ? v1 : v0;
      k += __shfl_xor_sync(0xffffffffu, up ? v0 : v1, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
      const float nx = __shfl_sync(0xffffffffu, k, 0), ray = __shfl_sync(0xffffffffu, k, 16);
      if (nx > 0.f) lam = ray / nx;
      break;
    }
    __syncwarp();
    xr = cscale(itr, y);
    xs[i] = xr;
    __syncwarp();
  }
  float2 cd;
  {
    const float lo = reg;
    const float hi = fmaxf(1.1f * lam, 1.0001f * lo);
    const float c = 0.5f * (lo + hi);
    float d = 0.5f * (hi - lo);
    if (!(d > 1e-6f * fmaxf(fabsf(c), 1e-30f))) d = fmaxf(fabsf(c), 1.f);
    cd = make_float2(c, d);
  }
  if (i == 0) ws[W.cd] = cd;
  // Ahat = (G + (reg - c) I) / d, row i in registers and as T_1 in buf0
  const float invd = 1.f / cd.y, shift = reg - cd.x;
  float dii = 0.f;  // Ahat[i][i]
#pragma unroll
  for (int c = 0; c < UP / 2; ++c) {
    float2 e0 = f2unpack(g[c].x), e1 = f2unpack(g[c].y);
    if (2 * c == i) { e0.x += shift; e0.y = 0.f; }
    if (2 * c + 1 == i) { e1.x += shift; e1.y = 0.f; }
    e0 = make_float2(e0.x * invd, e0.y * invd);
    e1 = make_float2(e1.x * invd, e1.y * invd);
    if (2 * c == i) dii = e0.x;
    if (2 * c + 1 == i) dii = e1.x;
    g[c].x = f2pack(e0.x, e0.y);
    g[c].y = f2pack(e1.x, e1.y);
    *reinterpret_cast<ulonglong2*>(buf0 + i * LD + 2 * c) = g[c];
  }
  double* mom = reinterpret_cast<double*>(ws + W.t);
  const double d1 = static_cast<double>(dii);
  {
    float n2 = 0.f;
#pragma unroll
    for (int c = 0; c < UP / 2; ++c) {
      const float2 e0 = f2unpack(g[c].x), e1 = f2unpack(g[c].y);
      n2 += cnorm(e0);
      n2 += cnorm(e1);
    }
    mom[i] = 1.0;
    mom[UP + i] = d1;
    mom[2 * UP + i] = 2.0 * static_cast<double>(n2) - 1.0;  // D_2 = 2 diag(T_1^2) - 1
  }
  __syncwarp();
  float2* cur = buf0;  // T_a
  float2* prv = buf1;  // T_{a-1} (a = 1: T_0 = I, implicit)
  // T_{a+1} is Hermitian: lane i forms only the band of columns
  // j = (i0 + q) mod 32, q = 0..17 (i0 = i rounded down to even, so the
  // reads are aligned LDS.128 pairs), which covers every pair (i, j) with
  // cyclic distance <= 16 from one side; the owner of a pair (distance
  // d = j - i mod 32 in 0..15, or 16 for i < 16) writes it and its
  // conjugate mirror -- 56% of the full-row products, exactly Hermitian
  constexpr int NQ = 18;
  const int i0 = i & ~1;
  for (int a = 1; a < K; ++a) {
    unsigned long long acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0ull;
#pragma unroll
    for (int k = 0; k < UP; ++k) {
      const float2 ak = f2unpack((k & 1) ? g[k >> 1].y : g[k >> 1].x);
      const unsigned long long ax = f2pack(ak.x, ak.x), ay = f2pack(-ak.y, ak.y);
      const float2* trow = cur + k * LD;
#pragma unroll
      for (int c = 0; c < NQ / 2; ++c) {
        const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(trow + ((i0 + 2 * c) & (UP - 1)));
        ffma2(acc[2 * c], t.x, ax);
        ffma2(acc[2 * c], f2swap_hl(t.x), ay);
        ffma2(acc[2 * c + 1], t.y, ax);
        ffma2(acc[2 * c + 1], f2swap_hl(t.y), ay);
      }
    }
    float2 nx[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = (i0 + q) & (UP - 1);
      const float2 pr = a == 1 ? make_float2(j == i ? 1.f : 0.f, 0.f) : prv[i * LD + j];
      const float2 v = f2unpack(acc[q]);
      nx[q] = make_float2(2.f * v.x - pr.x, 2.f * v.y - pr.y);
      if (j == i) nx[q].y = 0.f;
    }
    __syncwarp();  // every lane's reads of T_{a-1} are done before it is overwritten
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = (i0 + q) & (UP - 1), d = (j - i) & (UP - 1);
      if (d <= 15 || (d == 16 && i < 16)) {
        prv[i * LD + j] = nx[q];
        if (d != 0) prv[j * LD + i] = make_float2(nx[q].x, -nx[q].y);
      }
    }
    __syncwarp();  // T_{a+1} complete
    // row i's moments: |T_{a+1}[i][:]|^2 and Re T_{a+1}[i][:] . conj(T_a[i][:]), column order
    float n2 = 0.f, x2 = 0.f;
#pragma unroll
    for (int c = 0; c < UP / 2; ++c) {
      const float4 nv = *reinterpret_cast<const float4*>(prv + i * LD + 2 * c);
      const float4 cu = *reinterpret_cast<const float4*>(cur + i * LD + 2 * c);
      n2 += nv.x * nv.x + nv.y * nv.y;
      n2 += nv.z * nv.z + nv.w * nv.w;
      x2 += nv.x * cu.x + nv.y * cu.y;
      x2 += nv.z * cu.z + nv.w * cu.w;
    }
    mom[(2 * a + 1) * UP + i] = 2.0 * static_cast<double>(x2) - d1;  // D_{2a+1}
    mom[(2 * a + 2) * UP + i] = 2.0 * static_cast<double>(n2) - 1.0;  // D_{2a+2}
    float2* t = cur;
    cur = prv;
    prv = t;
  }
}

// ------------------------------------------------------------ extraction
// Chebyshev coefficients (FP64) of L_K and B = L_K (A - rho^-1 I) for one
// system, warp-parallel (cheb_coef_warp's recursion, kept in double), then
// the products ee = E*E and ef = E*F into `sh` (per-warp shared scratch of
// at least 2 * (2 * kMaxK + 1) + 2 * (kMaxK + 2) doubles).  All 32 lanes call.
struct MomCoef {
  double g0, l0;
};
__device__ __forceinline__ MomCoef moments_coefs(const float* hist, int K, double cc, double dd,
                                                 double rho_inv, double* sh) {
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
  // detect.cpp:336-368 on the coefficients: L_1 = alpha_1 I, then the
  // three-term update with c1 = a_k (1 + b_{k-1}) / a_{k-1}, c2 = a_k b_{k-2} / a_{k-2}
  // (a_0 = 1, b_0 = 0).  Lane k forms c1_k, c2_k (the FP64 divisions run in
  // parallel, off the recursion's dependency chain), shuffled in below.
  double c1v = 0.0, c2v = 0.0;
  if (m >= 2 && m <= K) {
    const double a = hist[(m - 1) * 2], am1 = hist[(m - 2) * 2], bm1 = hist[(m - 2) * 2 + 1];
    const double am2 = m >= 3 ? static_cast<double>(hist[(m - 3) * 2]) : 1.0;
    const double bm2 = m >= 3 ? static_cast<double>(hist[(m - 3) * 2 + 1]) : 0.0;
    c1v = a * (1.0 + bm1) / am1;
    c2v = a * bm2 / am2;
  }
  double l0 = m == 0 ? static_cast<double>(hist[0]) : 0.0, l1 = 0.0, l2 = 0.0;  // L_1 = alpha_1 I
  for (int k = 2; k <= K; ++k) {
    const double a = hist[(k - 1) * 2];
    const double c1 = __shfl_sync(0xffffffffu, c1v, k), c2 = __shfl_sync(0xffffffffu, c2v, k);
    const double d1 = l0 - l1;
    const double t = mulA(d1);
    const double nx = l0 + c1 * d1 - a * t - c2 * (l1 - l2);
    l2 = l1;
    l1 = l0;
    l0 = m < n ? nx : 0.0;
  }
  const double gm = mulA(l0) - rho_inv * l0;  // B = L (A - rho^-1 I)
  double* gs = sh;           // [kMaxK + 2]
  double* ls = sh + kMaxK + 2;
  double* ee = ls + kMaxK + 2;      // [2 kMaxK + 1]
  double* ef = ee + 2 * kMaxK + 1;  // [2 kMaxK + 1]
  if (m < n) {
    gs[m] = m == 0 ? 0.0 : gm;  // E = B - g_0 I
    ls[m] = m == 0 ? 0.0 : l0;  // F = L - l_0 I
  }
  const double g0 = __shfl_sync(0xffffffffu, gm, 0);
  const double l00 = __shfl_sync(0xffffffffu, l0, 0);
  __syncwarp();
  // Chebyshev products: (x*y)_k = 1/2 sum_{a+b=k} x_a y_b + 1/2 sum_{|a-b|=k} x_a y_b
  for (int k = m; k <= 2 * K; k += 32) {
    double se = 0.0, sf = 0.0;
    for (int a = 1; a <= K; ++a) {
      const double ga = gs[a];
      const int b1 = k - a;
      if (b1 >= 1 && b1 <= K) {
        se = fma(ga, gs[b1], se);
        sf = fma(ga, ls[b1], sf);
      }
      const int b2 = a - k, b3 = a + k;
      if (b2 >= 1) {
        se = fma(ga, gs[b2], se);
        sf = fma(ga, ls[b2], sf);
      }
      if (k > 0 && b3 <= K) {
        se = fma(ga, gs[b3], se);
        sf = fma(ga, ls[b3], sf);
      }
    }
    ee[k] = 0.5 * se;
    ef[k] = 0.5 * sf;
  }
  __syncwarp();
  return {g0, l00};
}

// Row i's mu and rho from the coefficient products in `sh` and the
// subcarrier's moment table (detect.cpp:375-395 + safe_rho :26-29).
__device__ __forceinline__ void moments_row(const double* sh, MomCoef c, int K, const double* mom,
                                            int UP, int i, double es, double n0, float& mu,
                                            float& rho, int km = kMaxK) {
  const double* gs = sh;  // scratch layout sized for K <= km
  const double* ls = sh + km + 2;
  const double* ee = ls + km + 2;
  const double* ef = ee + 2 * km + 1;
  double e = 0.0, f = 0.0, e2 = ee[0], efd = ef[0];
  for (int k = 1; k <= 2 * K; ++k) {
    const double d = mom[k * UP + i];
    if (k <= K) {
      e = fma(gs[k], d, e);
      f = fma(ls[k], d, f);
    }
    e2 = fma(ee[k], d, e2);
    efd = fma(ef[k], d, efd);
  }
  const double m = c.g0 + e;
  const double lii = c.l0 + f;
  const double interf = e2 - e * e;
  const double cross = m * lii + efd - e * f;
  const double nu2 = interf * es + cross * n0;
  mu = static_cast<float>(m);
  // safe_rho (detect.cpp:26-29); the quotient in FP32 (FP64 division is a
  // long dependent sequence) unless nu2 leaves FP32's normal range
  const double mm = m * m;
  rho = nu2 < 1e-300 ? 0.f
        : (nu2 > 1e-30 && mm < 1e30) ? __fdividef(static_cast<float>(mm), static_cast<float>(nu2))
                                     : static_cast<float>(mm / nu2);
}

// FX mode, one vector per subcarrier (S = 1): after the CG, x_hat and the
// status leave now; the (alpha, beta) history, v_K and the breakdown flag go
// to the workspace for moments_kernel<..., FX>, which finishes mu / rho /
// LLRs.  Threads [t0, t0 + nt) of the caller take part.
template <int UP>
__device__ __forceinline__ void fx_handoff(const KernelParams& p, float2* ws, const WsOffsets& W,
                                           long sc, const float* hist, int hstride,
                                           const float2* v, uint8_t broke, int t, int nt) {
  const int K = p.K;
  const bool ok = broke == 0;
  for (int e = t; e < UP + K + 1; e += nt) {
    if (e < K) {
      ws[W.t + e] = make_float2(hist[e * 2], hist[e * 2 + 1]);
    } else if (e < K + UP) {
      const int u = e - K;
      ws[W.t + e] = v[u];
      if (u < p.U && p.xhat) p.xhat[sc * static_cast<long>(p.U) + u] = ok ? v[u] : make_float2(0.f, 0.f);
    } else {
      ws[W.t + e] = make_float2(ok ? 0.f : 1.f, 0.f);
      if (p.status) p.status[sc] = ok ? 0 : 1;
    }
  }
  (void)hstride;
}

// per-warp shared scratch (doubles) for moments_coefs / moments_row
constexpr int kMomScratch = 2 * (kMaxK + 2) + 2 * (2 * kMaxK + 1);

// Lane-per-system form of moments_coefs for K <= kLaneK (compile-time K):
// the same FP64 recursion and Chebyshev products with the K + 2
// coefficients of L, B in registers, so the S systems of a subcarrier run in
// parallel on S lanes (moments_coefs spends a whole warp, 6 to 9 of its lanes
// busy and two shuffles per step, on each system).  Writes gs, ls, ee, ef in
// moments_row's layout for km = kLaneK, then g_0 and l_0.
constexpr int kLaneK = 6;
constexpr int kLaneScratch = 2 * (kLaneK + 2) + 2 * (2 * kLaneK + 1) + 2;
template <int K>
__device__ __forceinline__ void moments_coefs_lane(const float* hist, double cc, double dd,
                                                   double rho_inv, double* out) {
  constexpr int n = K + 2;
  double al[K + 1], be[K + 1];  // alpha_k, beta_k; alpha_0 = 1, beta_0 = 0
  al[0] = 1.0;
  be[0] = 0.0;
#pragma unroll
  for (int k = 1; k <= K; ++k) {
    al[k] = hist[(k - 1) * 2];
    be[k] = hist[(k - 1) * 2 + 1];
  }
  auto mulA = [&](const double (&x)[n], double (&o)[n]) {
#pragma unroll
    for (int m = 0; m < n; ++m) {
      double v = cc * x[m];
      if (m + 1 < n) v += 0.5 * dd * x[m + 1];
      if (m == 1) v += dd * x[0];
      else if (m >= 2) v += 0.5 * dd * x[m - 1];
      o[m] = v;
    }
  };
  double l0[n], l1[n], l2[n];
#pragma unroll
  for (int m = 0; m < n; ++m) l0[m] = l1[m] = l2[m] = 0.0;
  l0[0] = al[1];  // L_1 = alpha_1 I
#pragma unroll
  for (int k = 2; k <= K; ++k) {  // detect.cpp:336-368 on the coefficients
    // the ratios of the CG's FP32 step lengths in FP32 (off the FP64 chain)
    const double c1 = static_cast<double>(__fdividef(static_cast<float>(al[k] * (1.0 + be[k - 1])),
                                                     static_cast<float>(al[k - 1])));
    const double c2 = static_cast<double>(__fdividef(static_cast<float>(al[k] * be[k - 2]),
                                                     static_cast<float>(al[k - 2])));
    double d1[n], t[n];
#pragma unroll
    for (int m = 0; m < n; ++m) d1[m] = l0[m] - l1[m];
    mulA(d1, t);
#pragma unroll
    for (int m = 0; m < n; ++m) {
      const double nx = l0[m] + c1 * d1[m] - al[k] * t[m] - c2 * (l1[m] - l2[m]);
      l2[m] = l1[m];
      l1[m] = l0[m];
      l0[m] = nx;
    }
  }
  double gm[n];
  mulA(l0, gm);
#pragma unroll
  for (int m = 0; m < n; ++m) gm[m] -= rho_inv * l0[m];  // B = L (A - rho^-1 I)
  double* gs = out;
  double* ls = out + kLaneK + 2;
  double* ee = ls + kLaneK + 2;
  double* ef = ee + 2 * kLaneK + 1;
#pragma unroll
  for (int m = 0; m < n; ++m) {
    gs[m] = m == 0 ? 0.0 : gm[m];  // E = B - g_0 I
    ls[m] = m == 0 ? 0.0 : l0[m];  // F = L - l_0 I
  }
  // (x*y)_k = 1/2 sum_{a+b=k} x_a y_b + 1/2 sum_{|a-b|=k} x_a y_b over a, b in 1..K
#pragma unroll
  for (int k = 0; k <= 2 * K; ++k) {
    double se = 0.0, sf = 0.0;
#pragma unroll
    for (int a = 1; a <= K; ++a) {
      const int b1 = k - a, b2 = a - k, b3 = a + k;
      if (b1 >= 1 && b1 <= K) { se = fma(gm[a], gm[b1], se); sf = fma(gm[a], l0[b1], sf); }
      if (b2 >= 1) { se = fma(gm[a], gm[b2], se); sf = fma(gm[a], l0[b2], sf); }
      if (k > 0 && b3 <= K) { se = fma(gm[a], gm[b3], se); sf = fma(gm[a], l0[b3], sf); }
    }
    ee[k] = 0.5 * se;
    ef[k] = 0.5 * sf;
  }
  out[kLaneScratch - 2] = gm[0];
  out[kLaneScratch - 1] = l0[0];
}

// moments_tail for K <= kLaneK: the coefficients of all S systems at once,
// one lane each (moments_coefs_lane), then a warp per system, a lane per row.
// Threads [0, nthr) take part and synchronise on named barrier `bar_id`
// (0 with nthr = blockDim.x is __syncthreads); msh holds S x kLaneScratch
// doubles.
template <int UP>
__device__ __forceinline__ void moments_tail_lanes(const KernelParams& p, const float2* ws,
                                                   const WsOffsets& W, long sc, int Kmax,
                                                   const float* hist, const float2* Vs,
                                                   const uint8_t* sys_st, double* msh, int nthr,
                                                   int bar_id, int vstride = UP) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = nthr >> 5;
  const int S = p.S, U = p.U, K = p.K;
  const float2 cdv = ws[W.cd];
  const double* mom = reinterpret_cast<const double*>(ws + W.t);
  for (int s = threadIdx.x; s < S; s += nthr) {
    const float* hs = hist + s * Kmax * 2;
    double* o = msh + s * kLaneScratch;
    switch (K) {
      case 1: moments_coefs_lane<1>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
      case 2: moments_coefs_lane<2>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
      case 3: moments_coefs_lane<3>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
      case 4: moments_coefs_lane<4>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
      case 5: moments_coefs_lane<5>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
      default: moments_coefs_lane<6>(hs, cdv.x, cdv.y, p.rho_inv_u, o); break;
    }
  }
  named_sync(bar_id, nthr);
  for (int s = warp; s < S; s += nw) {
    const double* sh = msh + s * kLaneScratch;
    const MomCoef c = {sh[kLaneScratch - 2], sh[kLaneScratch - 1]};
    const bool ok = sys_st[s] == 0;
    for (int i = lane; i < U; i += 32) {
      float mu, rho;
      moments_row(sh, c, K, mom, UP, i, p.es, p.n0, mu, rho, kLaneK);
      const long o = (sc * S + s) * static_cast<long>(U) + i;
      const float2 xh = ok ? Vs[s * vstride + i] : make_float2(0.f, 0.f);
      if (!ok) mu = rho = 0.f;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = mu;
      if (p.rho) p.rho[o] = rho;
      if (p.llr) store_llrs_fast(xh, mu, rho, p.bits, p.llr + o * p.bits);
    }
    if (p.status && lane == 0) p.status[sc * S + s] = ok ? 0 : 1;
  }
  named_sync(bar_id, nthr);  // msh is reused by the next subcarrier
}

// Exact-tracker outputs of a subcarrier's S uplink systems after the CG
// (CTA-wide, warp per system): hist holds each system's (alpha, beta)
// history (stride Kmax), Vs its v_K, sys_st its breakdown flag; msh is
// nt/32 x kMomScratch doubles of shared scratch.
template <int UP>
__device__ __forceinline__ void moments_tail(const KernelParams& p, const float2* ws,
                                             const WsOffsets& W, long sc, int Kmax,
                                             const float* hist, const float2* Vs,
                                             const uint8_t* sys_st, int nt, double* msh,
                                             int vstride = UP, int msh_doubles = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = nt >> 5;
  const int S = p.S, U = p.U, K = p.K;
  const float2 cdv = ws[W.cd];
  const double* mom = reinterpret_cast<const double*>(ws + W.t);
  if (K <= kLaneK && S * kLaneScratch <= (msh_doubles > 0 ? msh_doubles : nw * kMomScratch)) {
    moments_tail_lanes<UP>(p, ws, W, sc, Kmax, hist, Vs, sys_st, msh, nt, 0, vstride);
    return;
  }
  double* sh = msh + warp * kMomScratch;
  for (int s = warp; s < S; s += nw) {
    const MomCoef c = moments_coefs(hist + s * Kmax * 2, K, cdv.x, cdv.y, p.rho_inv_u, sh);
    const bool ok = sys_st[s] == 0;
    for (int i = lane; i < U; i += 32) {
      float mu, rho;
      moments_row(sh, c, K, mom, UP, i, p.es, p.n0, mu, rho);
      const long o = (sc * S + s) * static_cast<long>(U) + i;
      const float2 xh = ok ? Vs[s * vstride + i] : make_float2(0.f, 0.f);
      if (!ok) mu = rho = 0.f;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = mu;
      if (p.rho) p.rho[o] = rho;
      if (p.llr) store_llrs_fast(xh, mu, rho, p.bits, p.llr + o * p.bits);
    }
    if (p.status && lane == 0) p.status[sc * S + s] = ok ? 0 : 1;
    __syncwarp();  // sh is reused by the next system
  }
}

}  // namespace cgm
