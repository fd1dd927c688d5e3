// cgm_solve32.cuh -- K2 for U = 32: the CG of all systems of a subcarrier
// as one small block GEMM per iteration.
//
// One CTA per subcarrier; thread t owns the 4 x TS tile (rows 4 rb .. 4 rb+3,
// systems TS sb ..), rb = t % 8, sb = t / 8.  Per CG iteration
// (solvers.cpp:37-72) the matvec E = A P of the tile is 32 k-steps of 4 x TS
// complex MACs on the packed FP32x2 pipe (two fma.rn.f32x2 per complex MAC,
// bitwise equal to the scalar FMA order), fed per k-step by LDS.128 of
// conj(G) (row k, 4 rows of the tile) and P (row k, TS systems); the
// (-Im, Im) operand pairs are formed in registers (storing them doubled the
// shared-memory wavefronts, which bound the first version).
// CG vectors x, r, p, e of the tile live in registers (packed); the dot
// products are 4-row partials reduced over the 8 row tiles with butterflies.
// Versus the lane-per-row kernel (solve_kernel): no per-FMA shared loads of
// p, no per-system 32-lane reductions, half the FMA instructions.
//
// After the CG the approximate tracker's outputs (detect.cpp:397-441) are
// written from the tiles; the exact tracker and the precoder reuse
// k2_exact_tail / k2_precode_tail of cgm_split.cuh.
#pragma once

#include "cgm_split.cuh"

namespace cgm {

struct S32Smem {
  int vs, qs, hist, sys_st, mu, rho, coef, gpart;  // as K2Smem (the shared tails)
  int gc, gn, pk, ftr, total, nsp;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int St, int K, bool exact, int ts) {
    const int nsys = S + St;
    nsp = (nsys + ts - 1) / ts * ts;  // systems padded to whole tiles
    int o = 0;
    gc = o; o = align(o + 32 * 32 * 8);
    pk = o; o = align(o + 32 * nsp * 8);
    gn = o; o = align(o + 32 * nsp * 8);  // pkn: (-Im p, Im p) companion of P
    ftr = o; o = align(o + (exact ? 0 : 3 * nsp * 32 * 4));
    vs = o; o = align(o + nsys * 32 * 8);
    qs = o; o = align(o + St * B * 8);
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    sys_st = o; o = align(o + nsys);
    mu = o; o = align(o + (exact ? S * 32 * 4 : 0));
    rho = o; o = align(o + (exact ? S * 32 * 4 : 0));
    coef = o; o = align(o + (exact ? S * 2 * (K + 2) * 4 : 0));
    gpart = o; o = align(o + ((B + 31) / 32) * (St > 0 ? St : 1) * 4);
    total = o;
  }
};

__device__ __forceinline__ unsigned long long f2swap(unsigned long long v) {
  const float2 t = f2unpack(v);
  return f2pack(t.y, t.x);
}
// d = a * b + c (packed)
__device__ __forceinline__ unsigned long long ffma2v(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Butterfly sum over the 8 row tiles (lanes differing in bits 0..2).
template <int TS>
__device__ __forceinline__ void rowtile_sum(float (&v)[TS]) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1)
#pragma unroll
    for (int j = 0; j < TS; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
}

// TS systems per tile (4 x TS tiles): TS = 2 halves the registers per
// thread (more resident warps), TS = 4 halves the shared loads per FMA.
template <bool EXACT, int TS>
__global__ void __launch_bounds__(256, 2) solve32_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  S32Smem L;
  L.plan(p.B, S, St, Kmax, EXACT, TS);
  WsOffsets W;
  W.plan(UP, S, p.K, EXACT, p.fx);
  const int nsp = L.nsp;
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* MUs = reinterpret_cast<float*>(smem + L.mu);
  float* RHOs = reinterpret_cast<float*>(smem + L.rho);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  float* gpart = reinterpret_cast<float*>(smem + L.gpart);
  float2* gc = reinterpret_cast<float2*>(smem + L.gc);                          // A[u][k] at [k][u]
  unsigned long long* pk = reinterpret_cast<unsigned long long*>(smem + L.pk);  // P[k][s]
  unsigned long long* pkn = reinterpret_cast<unsigned long long*>(smem + L.gn);  // (-Im, Im) of P
  float* ftr = reinterpret_cast<float*>(smem + L.ftr);  // approx tracker f0,f1,f2 [3][nsp][32]
  const int nt = blockDim.x, tid = threadIdx.x;
  const long lsc = blockIdx.x;
  const long sc = p.sc_base + lsc;
  const float2* ws = p.ws + lsc * W.stride;

  // G (Hermitian, row-major in the workspace) -> conj(G) row-major, which is
  // A[u][k] stored at [k][u] (column k of A contiguous over u)
  for (int e = tid; e < UP * UP; e += nt) {
    const float2 g = ws[W.g + e];
    gc[e] = make_float2(g.x, -g.y);
  }
  const int rb = tid & 7, sb = tid >> 3;
  const int u0 = rb * 4, s0 = sb * TS;
  const bool tile_live = s0 < nsys;
  float reg[TS];
  int iters[TS];
  bool down[TS], live[TS];
#pragma unroll
  for (int j = 0; j < TS; ++j) {
    const int s = s0 + j;
    live[j] = s < nsys;
    down[j] = s >= S;
    reg[j] = down[j] ? p.rho_inv_d : p.rho_inv_u;
    iters[j] = live[j] ? (down[j] ? p.Kt : p.K) : 0;
  }
  // right-hand sides: uplink b = MF (H^H y), downlink b = t
  unsigned long long x[4][TS], r[4][TS], pp[4][TS];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TS; ++j) {
      const int u = u0 + i, s = s0 + j;
      float2 b = make_float2(0.f, 0.f);
      if (live[j] && u < U)
        b = down[j] ? p.T[(sc * St + (s - S)) * static_cast<long>(U) + u] : ws[W.mf + s * UP + u];
      x[i][j] = 0ull;
      r[i][j] = f2pack(b.x, b.y);
      pp[i][j] = r[i][j];
      if (tile_live) {
        pk[u * nsp + s] = r[i][j];
        pkn[u * nsp + s] = f2pack(-b.y, b.y);
      }
      if (!EXACT && tile_live) {
        ftr[(0 * nsp + s) * 32 + u] = 0.f;
        ftr[(1 * nsp + s) * 32 + u] = 0.f;
        ftr[(2 * nsp + s) * 32 + u] = 0.f;
      }
    }
  float rn[TS], rn0[TS];
#pragma unroll
  for (int j = 0; j < TS; ++j) {
    rn[j] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 v = f2unpack(r[i][j]);
      rn[j] = fmaf(v.x, v.x, fmaf(v.y, v.y, rn[j]));
    }
  }
  rowtile_sum<TS>(rn);
  bool broke[TS];
  float am1[TS], am2[TS], bm1[TS], bm2[TS];
#pragma unroll
  for (int j = 0; j < TS; ++j) {
    rn0[j] = rn[j];
    broke[j] = false;
    am1[j] = am2[j] = 1.f;
    bm1[j] = bm2[j] = 0.f;
  }
  __syncthreads();
  float gdiag[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) gdiag[i] = gc[(u0 + i) * UP + u0 + i].x;

  for (int k = 1; k <= Kmax; ++k) {
    // ---- E = A P on the tile (k-steps over the 32 columns of A)
    unsigned long long e[4][TS];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < TS; ++j) e[i][j] = 0ull;
    if (tile_live) {
#pragma unroll 4
      for (int kk = 0; kk < UP; ++kk) {
        // e += a p with p broadcast: (p.x, p.x)(a.x, a.y) + (-p.y, p.y)(a.y, a.x);
        // the broadcast and the swapped pair are free operand selectors
        const ulonglong2 a01 = *reinterpret_cast<const ulonglong2*>(gc + kk * UP + u0);
        const ulonglong2 a23 = *reinterpret_cast<const ulonglong2*>(gc + kk * UP + u0 + 2);
        const unsigned long long av[4] = {a01.x, a01.y, a23.x, a23.y};
        float px[TS];
        unsigned long long pn[TS];
#pragma unroll
        for (int j2 = 0; j2 < TS; j2 += 2) {
          const float4 b = *reinterpret_cast<const float4*>(pk + kk * nsp + s0 + j2);
          const ulonglong2 bn = *reinterpret_cast<const ulonglong2*>(pkn + kk * nsp + s0 + j2);
          px[j2] = b.x;
          px[j2 + 1] = b.z;
          pn[j2] = bn.x;
          pn[j2 + 1] = bn.y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const unsigned long long as = f2swap(av[i]);
#pragma unroll
          for (int j = 0; j < TS; ++j) {
            e[i][j] = ffma2v(f2pack(px[j], px[j]), av[i], e[i][j]);  // (a.x p.x, a.y p.x)
            e[i][j] = ffma2v(pn[j], as, e[i][j]);                    // (-a.y p.y, a.x p.y)
          }
        }
      }
    }
    // ---- + reg p, curvature p^H A p (solvers.cpp:50-57)
    float curv[TS];
#pragma unroll
    for (int j = 0; j < TS; ++j) {
      curv[j] = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        e[i][j] = ffma2v(f2pack(reg[j], reg[j]), pp[i][j], e[i][j]);
        const float2 pv = f2unpack(pp[i][j]), ev = f2unpack(e[i][j]);
        curv[j] += pv.x * ev.x + pv.y * ev.y;
      }
    }
    rowtile_sum<TS>(curv);
    float alpha[TS], rnx[TS];
    bool upd[TS];
#pragma unroll
    for (int j = 0; j < TS; ++j) {
      const bool step = k <= iters[j];
      const bool frozen = !(rn[j] > 1e-28f * rn0[j]);  // solvers.cpp:21,25-27
      const bool go = step && !frozen && !broke[j];
      if (go && curv[j] < 1e-30f) broke[j] = true;     // solvers.cpp:55-57
      upd[j] = go && !broke[j];
      alpha[j] = upd[j] ? __fdividef(rn[j], curv[j]) : 1.f;
      rnx[j] = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (upd[j]) {
          x[i][j] = ffma2v(f2pack(alpha[j], alpha[j]), pp[i][j], x[i][j]);
          r[i][j] = ffma2v(f2pack(-alpha[j], -alpha[j]), e[i][j], r[i][j]);
        }
        const float2 v = f2unpack(r[i][j]);
        rnx[j] = fmaf(v.x, v.x, fmaf(v.y, v.y, rnx[j]));
      }
    }
    rowtile_sum<TS>(rnx);
    __syncthreads();  // every tile's reads of P done
#pragma unroll
    for (int j = 0; j < TS; ++j) {
      float beta = 0.f;
      if (upd[j]) {
        beta = __fdividef(rnx[j], rn[j]);
        rn[j] = rnx[j];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          pp[i][j] = ffma2v(f2pack(beta, beta), pp[i][j], r[i][j]);
          pk[(u0 + i) * nsp + s0 + j] = pp[i][j];
          const float2 pv = f2unpack(pp[i][j]);
          pkn[(u0 + i) * nsp + s0 + j] = f2pack(-pv.y, pv.y);
        }
      }
      if (k <= iters[j]) {
        const int s = s0 + j;
        if (!down[j]) {
          if (EXACT) {
            if (rb == 0) {
              hist[(s * Kmax + (k - 1)) * 2 + 0] = alpha[j];
              hist[(s * Kmax + (k - 1)) * 2 + 1] = beta;
            }
          } else {
            // Eq. (11) on the diagonal (detect.cpp:409-427)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int u = u0 + i;
              float* f = ftr + s * 32 + u;
              const float f0 = f[0], f1 = f[nsp * 32], f2 = f[2 * nsp * 32];
              float nf;
              if (k == 1) {
                nf = alpha[j];
              } else {
                const float c1 = __fdividef(alpha[j] * (1.f + bm1[j]), am1[j]);
                const float c2 = __fdividef(alpha[j] * bm2[j], am2[j]);
                nf = f0 + (c1 - alpha[j] * (gdiag[i] + reg[j])) * (f0 - f1) - c2 * (f1 - f2);
              }
              f[2 * nsp * 32] = f1;
              f[nsp * 32] = f0;
              f[0] = nf;
            }
          }
        }
        am2[j] = am1[j];
        am1[j] = alpha[j];
        bm2[j] = bm1[j];
        bm1[j] = beta;
      }
    }
    __syncthreads();  // P complete for the next matvec
  }

  // ---- per-tile outputs
#pragma unroll
  for (int j = 0; j < TS; ++j) {
    const int s = s0 + j;
    if (!live[j]) continue;
    if (rb == 0) sys_st[s] = broke[j] ? 1 : 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = u0 + i;
      const float2 xv = f2unpack(x[i][j]);
      if (EXACT || down[j]) {
        Vs[s * UP + u] = xv;
        continue;
      }
      if (u >= U) continue;
      // approx uplink: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
      const long o = (sc * S + s) * static_cast<long>(U) + u;
      const bool ok = !broke[j];
      const float2 xh = ok ? xv : make_float2(0.f, 0.f);
      const float mu_u = ok ? ftr[s * 32 + u] * gdiag[i] : 0.f;
      const float rho_u = ok ? gdiag[i] / p.n0 : 0.f;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = mu_u;
      if (p.rho) p.rho[o] = rho_u;
      if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
      if (p.status && i == 0 && rb == 0) p.status[sc * S + s] = ok ? 0 : 1;
    }
  }
  if (EXACT && S > 0) {
    __syncthreads();
    k2_exact_tail<UP>(p, ws, W, sc, Kmax, hist, coef, MUs, RHOs, Vs, sys_st, nt,
                      [] { __syncthreads(); });
  }
  if (St > 0) {
    __syncthreads();
    k2_precode_tail<UP>(p, sc, Vs, Qs, gpart, sys_st, nt, [] { __syncthreads(); });
  }
}

}  // namespace cgm
