// cgm_basis.cuh -- the exact tracker's Chebyshev basis as its own kernel.
//
// The exact SINR tracker (detect.cpp:330-395) needs, per subcarrier, the
// matrices T_1..T_K of Ahat = (A - cI)/d, A = G + rho^-1 I (cgm_split.cuh
// explains the basis argument): (K - 1) Hermitian U x U products
//   T_{m+1} = 2 Ahat T_m - T_{m-1},  T_0 = I,
// which dominate the FLOPs of the exact configurations (cfg4: U^3 per
// product against U^2 B for the Gram).  Inside the channel kernels they ran
// on the 8 epilogue warps of a one-CTA-per-SM tensor-core pipeline; here
// they get a kernel of their own, sized for the FP32 pipe:
//   * one thread per 4 x 4 tile of the LOWER triangle (the product of two
//     commuting Hermitian matrices is Hermitian; the upper triangle is the
//     conjugate mirror), (UP/4)(UP/4 + 1)/2 tiles per subcarrier;
//   * Ahat, T_m, T_{m-1} of each subcarrier in shared memory; per k the
//     thread reads four entries of row k of Ahat (= conj of column k, the
//     matrix is Hermitian) and four of row k of T_m (two LDS.128 each) and
//     issues 32 packed FFMA2 into one accumulator pair per entry:
//       acc += (t.x, t.y) * ahat.x + (t.y, t.x) * (ahat.y, -ahat.y)
//          = conj(ahat) t  (swap / negated broadcast are operand modifiers);
//   * U = 32: two subcarriers per 96-thread CTA (72 busy threads; four CTAs
//     fit the shared memory of an SM),
//     U = 64: one per 160-thread CTA (136 busy).
// The centre / half-width (c, d) comes from the same power iteration as
// before (cheb_interval, one warp per subcarrier).  Output: (c, d) and
// T_1..T_K in the workspace, the layout K2's extraction reads.
#pragma once

#include "cgm_rows32.cuh"  // f2dup_lo / f2dup_hi

namespace cgm {

template <int UP>
struct BasisGeo {
  static constexpr int NB = UP / 4;                  // tile rows
  static constexpr int NTILE = NB * (NB + 1) / 2;    // lower-triangle tiles
  static constexpr int SPC = UP == 32 ? 2 : 1;       // subcarriers per CTA (smem: 4 CTAs / SM)
  static constexpr int NT = ((SPC * NTILE + 31) / 32) * 32;
  static constexpr int LD = UP + 2;                  // padded row (bank spread, 16 B aligned)
  static constexpr int MAT = UP * LD;                // float2 per matrix in smem
  static constexpr int SMEM = SPC * 3 * MAT * 8;     // Ahat, T_m, T_{m-1}
};

// FX (one vector per subcarrier, p.fx): the basis never leaves the chip --
// the CG kernel left (alpha, beta) in the workspace, the coefficients of L_K
// and B = L_K G are formed here first, every tile accumulates its entries of
// B and L while the products run, and the extraction (detect.cpp:375-395)
// and the LLRs finish in this kernel.  Saves writing and re-reading K U x U
// matrices per subcarrier (cfg4b K = 8: 34 GB of HBM traffic).
template <int UP, bool FX = false>
__global__ void __launch_bounds__(BasisGeo<UP>::NT, UP == 32 ? 4 : 2) basis_kernel(const KernelParams p) {
  using BG = BasisGeo<UP>;
  constexpr int MAT = BG::MAT, SPC = BG::SPC, LD = BG::LD;
  extern __shared__ __align__(128) unsigned char smem[];
  float2* base = reinterpret_cast<float2*>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = p.K;
  WsOffsets W;
  W.plan(UP, p.S, K, true, p.fx);
  const long sc0 = static_cast<long>(blockIdx.x) * SPC;
  const int nsc = static_cast<int>(p.n_sc - sc0 < SPC ? p.n_sc - sc0 : SPC);
  auto Ah = [&](int s) { return base + (s * 3 + 0) * MAT; };
  // --------------------------------------------------------------- G in
  // (padded smem matrix) <-> (dense UP x UP workspace matrix), float4 = 2 entries
  auto load = [&](float2* dst, const float2* src) {
    for (int e = tid; e < UP * UP / 2; e += BG::NT) {
      const int r = e / (UP / 2), c2 = e - r * (UP / 2);
      *reinterpret_cast<float4*>(dst + r * LD + 2 * c2) = reinterpret_cast<const float4*>(src)[e];
    }
  };
  auto store = [&](float2* dst, const float2* src) {
    for (int e = tid; e < UP * UP / 2; e += BG::NT) {
      const int r = e / (UP / 2), c2 = e - r * (UP / 2);
      reinterpret_cast<float4*>(dst)[e] = *reinterpret_cast<const float4*>(src + r * LD + 2 * c2);
    }
  };
  for (int s = 0; s < nsc; ++s) load(Ah(s), p.ws + (sc0 + s) * W.stride + W.g);
  __syncthreads();
  if (FX && p.fx == 2) {  // exact Hermitian from the lower triangle (the fused Gram writes full rows)
    for (int e = tid; e < nsc * UP * UP; e += BG::NT) {
      const int s = e / (UP * UP), r = (e / UP) % UP, c = e % UP;
      float2* a = Ah(s);
      if (c == r) a[r * LD + c].y = 0.f;
    }
    for (int e = tid; e < nsc * UP * UP; e += BG::NT) {
      const int s = e / (UP * UP), r = (e / UP) % UP, c = e % UP;
      float2* a = Ah(s);
      if (c > r) a[r * LD + c] = cconj(a[c * LD + r]);
    }
    __syncthreads();
  }
  // ------------------------------------- (c, d) by power iteration, warp s
  __shared__ float2 cds[SPC];
  // FX: also the Chebyshev coefficients of L_K and B from the CG history
  __shared__ float coefs[FX ? SPC : 1][2][kMaxK + 2];
  if (warp < nsc) {
    // cheb_interval returns the same (c, d) on every lane of the warp
    const float2 cd = cheb_interval<UP, LD>(Ah(warp), p.rho_inv_u, base + (warp * 3 + 1) * MAT, lane);
    if (lane == 0) {
      cds[warp] = cd;
      p.ws[(sc0 + warp) * W.stride + W.cd] = cd;
    }
    if (FX) {
      const float* hist = reinterpret_cast<const float*>(p.ws + (sc0 + warp) * W.stride + W.t);
      cheb_coef_warp(hist, K, cd.x, cd.y, p.rho_inv_u, coefs[warp][0], coefs[warp][1]);
    }
  }
  __syncthreads();
  // --------------------------------------- T_1 = Ahat = (A - cI)/d, in place
  for (int s = 0; s < nsc; ++s) {
    const float cc = cds[s].x, invd = 1.f / cds[s].y;
    float2* a = Ah(s);
    float2* Tw = p.ws + (sc0 + s) * W.stride + W.t;
    for (int e = tid; e < UP * UP; e += BG::NT) {
      const int r = e / UP, c = e - r * UP;
      float2 v = a[r * LD + c];
      if (r == c) v.x += p.rho_inv_u - cc;
      v = cscale(invd, v);
      a[r * LD + c] = v;
      if (!FX) Tw[e] = v;
    }
  }
  __syncthreads();
  // ------------------------------------------------------------ products
  const int slot = tid / BG::NTILE;
  const int tile = tid - slot * BG::NTILE;
  int rb = 0;
  while ((rb + 1) * (rb + 2) / 2 <= tile) ++rb;
  const int cb = tile - rb * (rb + 1) / 2;
  const bool busy = slot < nsc;
  const int i0 = rb * 4, j0 = cb * 4;
  const float2* A = base + (slot * 3 + 0) * MAT;
  // FX: this tile's entries of B = sum_m cb_m T_m and L = sum_{m<K} cl_m T_m
  float2 Bacc[FX ? 4 : 1][FX ? 4 : 1], Lacc[FX ? 4 : 1][FX ? 4 : 1];
  if constexpr (FX) {
    const float* cl = coefs[busy ? slot : 0][0];
    const float* cbq = coefs[busy ? slot : 0][1];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + r, j = j0 + c;
        const float2 t1 = busy ? A[i * LD + j] : make_float2(0.f, 0.f);  // T_1
        const float d0 = i == j ? 1.f : 0.f;                             // T_0 = I
        Bacc[r][c] = make_float2(cbq[0] * d0 + cbq[1] * t1.x, cbq[1] * t1.y);
        Lacc[r][c] = K > 1 ? make_float2(cl[0] * d0 + cl[1] * t1.x, cl[1] * t1.y)
                           : make_float2(cl[0] * d0, 0.f);
      }
  }
  // T_m in buffer `cur`, T_{m-1} in `prv` (1 and 2 alternate)
  int cur = 0, prv = 1;  // cur 0 == Ahat itself for m = 1
  for (int m = 1; m < K; ++m) {
    if (busy) {
      const float2* Tc = base + (slot * 3 + cur) * MAT;
      // one packed accumulator per entry: conj(ahat) t = t * ahat.x + swap(t) * (ahat.y, -ahat.y)
      // (the swap and the negated broadcast are FFMA2 operand modifiers);
      // operands of row k + 1 are loaded while row k is consumed
      unsigned long long acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0ull;
      auto ld = [&](int k, ulonglong2 (&av)[2], ulonglong2 (&tv)[2]) {
        av[0] = *reinterpret_cast<const ulonglong2*>(A + k * LD + i0);
        av[1] = *reinterpret_cast<const ulonglong2*>(A + k * LD + i0 + 2);
        tv[0] = *reinterpret_cast<const ulonglong2*>(Tc + k * LD + j0);
        tv[1] = *reinterpret_cast<const ulonglong2*>(Tc + k * LD + j0 + 2);
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
      // T_{m+1} = 2 Ahat T_m - T_{m-1} into the T_{m-1} buffer (lower +
      // mirror; only this thread reads these lower entries of T_{m-1})
      float2* Tn = base + (slot * 3 + (m == 1 ? 1 : prv)) * MAT;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = i0 + r, j = j0 + c;
          if (j > i) continue;
          const float2 prod = f2unpack(acc[r][c]);
          const float2 prev = m == 1 ? make_float2(i == j ? 1.f : 0.f, 0.f) : Tn[i * LD + j];
          float2 val = make_float2(2.f * prod.x - prev.x, 2.f * prod.y - prev.y);
          if (i == j) val.y = 0.f;
          Tn[i * LD + j] = val;
          if (i != j) Tn[j * LD + i] = cconj(val);
          if constexpr (FX) {  // T_{m+1} into this tile's B and L
            const float cbm = coefs[slot][1][m + 1];
            Bacc[r][c].x = fmaf(cbm, val.x, Bacc[r][c].x);
            Bacc[r][c].y = fmaf(cbm, val.y, Bacc[r][c].y);
            if (m + 1 < K) {
              const float clm = coefs[slot][0][m + 1];
              Lacc[r][c].x = fmaf(clm, val.x, Lacc[r][c].x);
              Lacc[r][c].y = fmaf(clm, val.y, Lacc[r][c].y);
            }
          }
        }
    }
    __syncthreads();
    if (!FX) {  // T_{m+1} -> workspace, coalesced
      const int nb = m == 1 ? 1 : prv;
      for (int s = 0; s < nsc; ++s)
        store(p.ws + (sc0 + s) * W.stride + W.t + m * UP * UP, base + (s * 3 + nb) * MAT);
    }
    // rotate: T_{m+1} (just written) becomes current, T_m previous
    const int nw = m == 1 ? 1 : prv;
    prv = m == 1 ? 2 : cur;
    cur = nw;
    if (m == 1) {  // T_1 (= Ahat, buffer 0) must stay intact: copy it to buffer 2 as T_{m-1}
      for (int s = 0; s < nsc; ++s) {
        const float4* src = reinterpret_cast<const float4*>(Ah(s));
        float4* dst = reinterpret_cast<float4*>(base + (s * 3 + 2) * MAT);
        for (int e = tid; e < MAT / 2; e += BG::NT) dst[e] = src[e];
      }
      __syncthreads();
    }
  }
  if constexpr (FX) {
    // ---------------- extraction (detect.cpp:375-395) from the tile sums:
    // per lower entry (i, j): |B_ij|^2 and Re(B_ij conj(L_ij)) count for row
    // i and (i != j, Hermitian) for row j; mu_i = Re B_ii.  Row parts go to
    // Rb[i][cb], column parts to Cb[j][rb] (each slot written by one tile),
    // summed in a fixed order below.  Both alias a T buffer no longer read.
    constexpr int NB = BG::NB;
    float* Rb = reinterpret_cast<float*>(base + (slot * 3 + 1) * MAT);  // [UP][NB][2]
    float* Cb = Rb + UP * NB * 2;                                       // [UP][NB][2]
    float* Mb = Cb + UP * NB * 2;                                       // [UP]
    static_assert(2 * 2 * 32 * (32 / 4) + 32 <= 32 * (32 + 2) * 2, "partials fit a T buffer");
    // T buffer 1 may still hold T_K (read by no one now); all products ended at the barrier above
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
    for (int e = tid; e < nsc * UP; e += BG::NT) {
      const int s = e / UP, i = e - s * UP;
      if (i >= p.U) continue;
      const float* R = reinterpret_cast<const float*>(base + (s * 3 + 1) * MAT);
      const float* C = R + UP * NB * 2;
      const float* M = C + UP * NB * 2;
      const int rbi = i / 4;
      float ib2 = 0.f, ibl = 0.f;
      for (int q = 0; q <= rbi; ++q) { ib2 += R[(i * NB + q) * 2]; ibl += R[(i * NB + q) * 2 + 1]; }
      for (int q = rbi; q < NB; ++q) { ib2 += C[(i * NB + q) * 2]; ibl += C[(i * NB + q) * 2 + 1]; }
      const long sc = p.sc_base + sc0 + s;  // S = 1: vector index == subcarrier
      const long o = sc * static_cast<long>(p.U) + i;
      const bool ok = p.status ? p.status[sc] == 0 : true;
      const float mu_i = M[i];
      const float nu2 = ib2 * p.es + ibl * p.n0;
      const float mu = ok ? mu_i : 0.f;
      const float rho = ok ? (nu2 <= 0.f ? 0.f : mu_i * mu_i / nu2) : 0.f;  // safe_rho
      const float2 xh = p.xhat ? p.xhat[o] : make_float2(0.f, 0.f);
      if (p.mu) p.mu[o] = mu;
      if (p.rho) p.rho[o] = rho;
      if (p.llr) store_llrs_fast(xh, mu, rho, p.bits, p.llr + o * p.bits);
    }
  }
}

}  // namespace cgm
