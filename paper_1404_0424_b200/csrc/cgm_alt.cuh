// cgm_alt.cuh -- the other detectors and precoders of the reference's
// trade-off study, batched on the GPU:
//
//   detect_cholesky   detect.cpp:122-181   (Cholesky inverse of A, Eq. 3-5)
//   detect_cgls       detect.cpp:238-272   (CGLS on the augmented LS problem
//                                           + approximate SINR tracker)
//   detect_neumann    detect.cpp:274-326   (truncated Neumann series of A^-1)
//   precode_explicit  precode.cpp:45-54    (Cholesky inverse of A_d)
//   precode_cgls      precode.cpp:73-82    (min-norm CGLS, solvers.cpp:196-235)
//   precode_neumann   precode.cpp:84-93
//
// with the solver cores cholesky_factor / cholesky_inverse (solvers.cpp:
// 237-321), neumann_inverse (:323-359), cgls_core / cgls_solve_regularized
// (:87-194) restated for one CTA per subcarrier.  These are not GEMM-sized
// (U x U with U <= 64 per subcarrier): everything lives in shared memory,
// the subcarrier's channel is read from HBM once, threads split the rows /
// columns of each small product and the sequential parts (Cholesky columns,
// CGLS iterations) synchronise at block level.  FP32 storage and arithmetic
// like the CG path; status bits as in cgmimo_b200.h (bit 0 SolverBreakdown,
// bit 1 zero_input, bit 2 not positive definite / zero diagonal, where the
// reference throws NotPositiveDefinite / std::domain_error).
#pragma once

#include "cgm_kernels.cuh"

namespace cgm {
namespace alt {

enum Method { kCholesky = 0, kCg = 1, kCgls = 2, kNeumann = 3 };  // sim.hpp:34 order

constexpr int NT = 256;
constexpr int NW = NT / 32;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float s, float2 a) { return make_float2(s * a.x, s * a.y); }
__device__ __forceinline__ float cabs2(float2 a) { return a.x * a.x + a.y * a.y; }

// block-wide sum of one float per thread (all threads get the result)
__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}

// Shared-memory plan (float2 units) for one subcarrier.  The U x U blocks
// exist only for the methods that use them; Neumann's two term buffers
// alias the staged channel when it is large enough (it is dead once the
// Gram matrix and matched filters are formed; the precoder restages it).
struct AltSmem {
  int hs, a, g, inv, term, next, mf, xs, vec, red, total;
  bool alias;
  __host__ __device__ void plan(int B, int U, int S, int method) {
    const int UU = U * U;
    const bool mat = method != kCgls, neu = method == kNeumann;
    int o = 0;
    hs = o;   o += B * (mat ? U : U + 1);  // H_u [b][u] (downlink: conj(H_d)^T), row stride U (+1 CGLS)
    a = o;    o += mat ? UU : 0;      // A = G + reg I (Cholesky: then L in place)
    g = o;    o += neu ? UU : 0;      // unregularised Gram G (Neumann mu)
    inv = o;  o += mat ? UU : 0;      // A^-1 (Cholesky) / Neumann sum
    alias = neu && B * U >= 2 * UU;
    term = alias ? hs : o; o += (neu && !alias) ? UU : 0;
    next = alias ? hs + UU : o; o += (neu && !alias) ? UU : 0;
    mf = o;   o += S * U;             // matched filters / transmit vectors per system
    xs = o;   o += S * U;             // equalised outputs per system
    vec = o;  o += (mat ? B : NW * (B + U)) + 2 * U;  // q [B] / CGLS per-warp r|w [B], d [U]; 3 U floats
    red = o;  o += NW;                // block reduction
    total = o;
  }
};

// out[b] = sum_u Hs[b][u] v[u], b < B
__device__ __forceinline__ void mv(const float2* Hs, int B, int U, const float2* v, float2* out) {
  for (int b = threadIdx.x; b < B; b += NT) {
    float2 acc = make_float2(0.f, 0.f);
    for (int u = 0; u < U; ++u) acc = cadd(acc, cmul(Hs[b * U + u], v[u]));
    out[b] = acc;
  }
}

// G = Hs^H Hs (one triangle + conjugate mirror, real diagonal:
// linalg.cpp:59-101), A = G + reg I
__device__ __forceinline__ void gram(const float2* Hs, int B, int U, float reg, float2* G, float2* A) {
  const int npairs = U * (U + 1) / 2;
  for (int e = threadIdx.x; e < npairs; e += NT) {
    // e -> (i, j), i >= j
    int i = static_cast<int>((sqrtf(8.f * e + 1.f) - 1.f) * 0.5f);
    while (i * (i + 1) / 2 > e) --i;
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    const int j = e - i * (i + 1) / 2;
    float2 acc = make_float2(0.f, 0.f);
    for (int b = 0; b < B; ++b) acc = cadd(acc, cmulc(Hs[b * U + i], Hs[b * U + j]));
    if (i == j) {
      G[i * U + i] = make_float2(acc.x, 0.f);
      A[i * U + i] = make_float2(acc.x + reg, 0.f);
    } else {
      G[i * U + j] = acc;
      G[j * U + i] = make_float2(acc.x, -acc.y);
      A[i * U + j] = acc;
      A[j * U + i] = make_float2(acc.x, -acc.y);
    }
  }
  __syncthreads();
}

// cholesky_factor (solvers.cpp:237-259) in place over the lower triangle of
// A (left-looking, column by column), then cholesky_inverse (:289-321):
// thread c solves L z = e_c forward and L^H x = z backward into Inv[:, c].
// Returns false when a pivot is not positive (NotPositiveDefinite).
__device__ __forceinline__ bool cholesky_inverse(float2* A, float2* Inv, int U) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < U; ++j) {
    if (threadIdx.x < 32) {
      float d = 0.f;
      for (int k = threadIdx.x; k < j; k += 32) d += cabs2(A[j * U + k]);
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (threadIdx.x == 0) {
        const float dd = A[j * U + j].x - d;
        if (!(dd > 0.f)) bad = 1;
        A[j * U + j] = make_float2(dd > 0.f ? sqrtf(dd) : 1.f, 0.f);
      }
    }
    __syncthreads();
    const float piv = A[j * U + j].x;
    for (int i = j + 1 + threadIdx.x; i < U; i += NT) {
      float2 s = A[i * U + j];
      for (int k = 0; k < j; ++k) s = csub(s, cmul(A[i * U + k], make_float2(A[j * U + k].x, -A[j * U + k].y)));
      A[i * U + j] = make_float2(s.x / piv, s.y / piv);
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < U; c += NT) {
    for (int i = 0; i < c; ++i) Inv[i * U + c] = make_float2(0.f, 0.f);
    Inv[c * U + c] = make_float2(1.f / A[c * U + c].x, 0.f);
    for (int i = c + 1; i < U; ++i) {
      float2 s = make_float2(0.f, 0.f);
      for (int k = c; k < i; ++k) s = csub(s, cmul(A[i * U + k], Inv[k * U + c]));
      Inv[i * U + c] = cscale(1.f / A[i * U + i].x, s);
    }
    for (int ii = U - 1; ii >= 0; --ii) {
      float2 s = Inv[ii * U + c];
      for (int k = ii + 1; k < U; ++k) s = csub(s, cmulc(A[k * U + ii], Inv[k * U + c]));
      Inv[ii * U + c] = cscale(1.f / A[ii * U + ii].x, s);
    }
  }
  __syncthreads();
  return bad == 0;
}

// neumann_inverse (solvers.cpp:323-359): Sum = D^-1 + T D^-1 + T^2 D^-1 +
// ..., T = -D^-1 E; higher terms fill one triangle and mirror it.  inv_d in
// `dinv`.  Returns false on a zero diagonal entry (std::domain_error).
__device__ __forceinline__ bool neumann_inverse(const float2* A, float2* Sum, float2* term,
                                                float2* next, float* dinv, int U, int terms) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < U; i += NT) {
    const float d = A[i * U + i].x;
    if (d == 0.f) bad = 1;
    dinv[i] = d == 0.f ? 0.f : 1.f / d;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < U * U; e += NT) {
    const int i = e / U, j = e - i * U;
    if (i == j) {
      Sum[e] = make_float2(dinv[i], 0.f);
      term[e] = make_float2(0.f, 0.f);
    } else {
      const float2 t = cscale(-dinv[i], A[e]);  // T(i, j)
      term[e] = cscale(dinv[j], t);
      Sum[e] = terms > 1 ? term[e] : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  for (int extra = 2; extra < terms; ++extra) {
    const int npairs = U * (U + 1) / 2;
    for (int e = threadIdx.x; e < npairs; e += NT) {
      // (i, j), j >= i: row-major upper triangle
      int i = 0, rem = e;
      while (rem >= U - i) { rem -= U - i; ++i; }
      const int j = i + rem;
      float2 s = make_float2(0.f, 0.f);
      for (int k = 0; k < U; ++k)
        if (k != i) s = cadd(s, cmul(cscale(-dinv[i], A[i * U + k]), term[k * U + j]));
      next[i * U + j] = s;
      if (j != i) next[j * U + i] = make_float2(s.x, -s.y);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < U * U; e += NT) {
      Sum[e] = cadd(Sum[e], next[e]);
      term[e] = next[e];
    }
    __syncthreads();
  }
  return bad == 0;
}

// out[s][i] = sum_j M[i][j] v[s][j] for S systems
__device__ __forceinline__ void apply(const float2* M, const float2* v, float2* out, int U, int S) {
  for (int e = threadIdx.x; e < S * U; e += NT) {
    const int s = e / U, i = e - s * U;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < U; ++j) acc = cadd(acc, cmul(M[i * U + j], v[s * U + j]));
    out[e] = acc;
  }
}

// ApproxSinrTracker::step (detect.cpp:400-428) for all users; st = {filt,
// filt_m1, filt_m2} in smem, scalar history in regs (uniform)
struct Tracker {
  int k = 0;
  float am1 = 1.f, am2 = 1.f, bm1 = 0.f, bm2 = 0.f;
  __device__ void step(float* f, float* f1, float* f2, const float* a_diag, int U, float alpha,
                       float beta) {
    ++k;
    for (int i = threadIdx.x; i < U; i += NT) {
      const float cur = f[i], m1 = f1[i], m2 = f2[i];
      float nx;
      if (k == 1) {
        nx = alpha;
      } else {
        const float c1 = alpha * (1.f + bm1) / am1;
        const float c2 = alpha * bm2 / am2;
        nx = cur + (c1 - alpha * a_diag[i]) * (cur - m1) - c2 * (m1 - m2);
      }
      f2[i] = m1;
      f1[i] = cur;
      f[i] = nx;
    }
    am2 = am1;
    am1 = alpha;
    bm2 = bm1;
    bm1 = beta;
    __syncthreads();
  }
};

__device__ __forceinline__ float safe_rho(float mu, float nu2) {  // detect.cpp:26-29
  return nu2 <= 0.f ? 0.f : mu * mu / nu2;
}

// write one detected system's outputs (xhat, mu, rho, LLRs; zeros on error)
__device__ __forceinline__ void put_detect(const KernelParams& p, long sc, int s, int i, float2 xh,
                                           float mu, float rho, bool ok) {
  const long o = (sc * p.S + s) * static_cast<long>(p.U) + i;
  if (!ok) {
    xh = make_float2(0.f, 0.f);
    mu = rho = 0.f;
  }
  if (p.xhat) p.xhat[o] = xh;
  if (p.mu) p.mu[o] = mu;
  if (p.rho) p.rho[o] = rho;
  if (p.llr) {
    if (ok) {
      store_llrs(xh, mu, rho, p.bits, p.llr + o * p.bits);
    } else {
      for (int b = 0; b < p.bits; ++b) p.llr[o * p.bits + b] = 0.f;
    }
  }
}

// ---------------------------------------------------------------- CGLS
// One warp per system: lane l owns users u = l + 32m (m < 2, U <= 64) and
// antenna rows b = l + 32k.  H sits in shared memory with row stride U + 1,
// so both the row reads of H d (lane <-> row) and the column reads of H^H r
// (lane <-> user) are conflict-free; the vector each product broadcasts
// (d, or r / w) goes through the warp's own shared-memory slot.
constexpr int kRU = 2;  // users per lane
constexpr int kRB = 8;  // antenna rows per lane (B <= 256)

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// detect_cgls (detect.cpp:238-272): cgls_solve_regularized (solvers.cpp:
// 141-194) on [H; sqrt(rho^-1) I] over cgls_core (:87-139), the approximate
// tracker on the Gram diagonal, extraction (detect.cpp:430-441).
__device__ void cgls_detect_warps(const KernelParams& p, long sc, const float2* Hs, int HS,
                                  float2* V, const float* gdg, const float* adg, float reg) {
  const int B = p.B, U = p.U, S = p.S, K = p.K;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float2* rv = V + w * (B + U);  // residual rows [B]
  float2* dv = rv + B;           // direction [U]
  const float aug = sqrtf(reg);
  for (int s = w; s < S; s += NW) {
    float2 x[kRU], d[kRU], ra[kRU];  // solution, direction, residual tail (identity block)
    float f0[kRU], f1[kRU], f2[kRU];
    for (int k = 0; k < kRB; ++k) {
      const int b = l + 32 * k;
      if (b < B) rv[b] = p.Y[(sc * B + b) * static_cast<long>(S) + s];
    }
    __syncwarp();
    float gs = 0.f;
#pragma unroll
    for (int m = 0; m < kRU; ++m) {
      const int u = l + 32 * m;
      x[m] = d[m] = ra[m] = make_float2(0.f, 0.f);
      f0[m] = f1[m] = f2[m] = 0.f;
      if (u < U) {  // first adjoint: the matched filter H^H y
        float2 acc = make_float2(0.f, 0.f);
        for (int b = 0; b < B; ++b) acc = cadd(acc, cmulc(Hs[b * HS + u], rv[b]));
        d[m] = acc;
        dv[u] = acc;
        gs += cabs2(acc);
      }
    }
    float gamma = warp_sum(gs);
    const float gamma0 = gamma;
    float am1 = 1.f, am2 = 1.f, bm1 = 0.f, bm2 = 0.f;
    bool broke = false;
    for (int k = 1; k <= K; ++k) {
      float alpha = 1.f, beta = 0.f;
      if (!(gamma <= 1e-28f * gamma0)) {
        __syncwarp();
        float2 q[kRB];
        float qs = 0.f;
#pragma unroll
        for (int kb = 0; kb < kRB; ++kb) {
          const int b = l + 32 * kb;
          q[kb] = make_float2(0.f, 0.f);
          if (b < B) {
            const float2* hr = Hs + b * HS;
            for (int u = 0; u < U; ++u) q[kb] = cadd(q[kb], cmul(hr[u], dv[u]));
            qs += cabs2(q[kb]);
          }
        }
#pragma unroll
        for (int m = 0; m < kRU; ++m)
          if (l + 32 * m < U) qs += aug * aug * cabs2(d[m]);
        const float qn2 = warp_sum(qs);
        if (qn2 < 1e-30f) {  // solvers.cpp:115-116
          broke = true;
          break;
        }
        alpha = gamma / qn2;
#pragma unroll
        for (int m = 0; m < kRU; ++m) {
          x[m] = cadd(x[m], cscale(alpha, d[m]));
          ra[m] = csub(ra[m], cscale(alpha * aug, d[m]));
        }
        __syncwarp();
#pragma unroll
        for (int kb = 0; kb < kRB; ++kb) {
          const int b = l + 32 * kb;
          if (b < B) rv[b] = csub(rv[b], cscale(alpha, q[kb]));
        }
        __syncwarp();
        float gn = 0.f;
        float2 sv[kRU];
#pragma unroll
        for (int m = 0; m < kRU; ++m) {
          const int u = l + 32 * m;
          sv[m] = make_float2(0.f, 0.f);
          if (u < U) {
            float2 acc = cscale(aug, ra[m]);
            for (int b = 0; b < B; ++b) acc = cadd(acc, cmulc(Hs[b * HS + u], rv[b]));
            sv[m] = acc;
            gn += cabs2(acc);
          }
        }
        gn = warp_sum(gn);
        beta = gn / gamma;
        gamma = gn;
#pragma unroll
        for (int m = 0; m < kRU; ++m) {
          const int u = l + 32 * m;
          d[m] = cadd(sv[m], cscale(beta, d[m]));
          if (u < U) dv[u] = d[m];
        }
      }
      // ApproxSinrTracker::step (detect.cpp:400-428)
#pragma unroll
      for (int m = 0; m < kRU; ++m) {
        const int u = l + 32 * m;
        float nx = alpha;
        if (k > 1 && u < U) {
          const float c1 = alpha * (1.f + bm1) / am1, c2 = alpha * bm2 / am2;
          nx = f0[m] + (c1 - alpha * adg[u]) * (f0[m] - f1[m]) - c2 * (f1[m] - f2[m]);
        }
        f2[m] = f1[m];
        f1[m] = f0[m];
        f0[m] = nx;
      }
      am2 = am1; am1 = alpha; bm2 = bm1; bm1 = beta;
    }
#pragma unroll
    for (int m = 0; m < kRU; ++m) {
      const int u = l + 32 * m;
      if (u < U)
        put_detect(p, sc, s, u, x[m], f0[m] * gdg[u], p.n0 > 0.f ? gdg[u] / p.n0 : 0.f, !broke);
    }
    if (l == 0 && p.status) p.status[sc * S + s] = broke ? 1 : 0;
    __syncwarp();
  }
}

// precode_cgls (precode.cpp:73-82): cgls_solve_min_norm (solvers.cpp:196-235),
// q accumulated as x += alpha H_d^H p, then normalize (precode.cpp:22-36).
__device__ void cgls_precode_warps(const KernelParams& p, long sc, const float2* Hs, int HS,
                                   float2* V, float reg) {
  const int B = p.B, U = p.U, S = p.St, K = p.Kt;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float2* wv = V + w * (B + U);  // w = H_d^H p [B]
  float2* dv = wv + B;           // direction [U]
  for (int s = w; s < S; s += NW) {
    float2 r[kRU], d[kRU], x[kRB];
    float rs = 0.f;
#pragma unroll
    for (int m = 0; m < kRU; ++m) {
      const int u = l + 32 * m;
      r[m] = u < U ? p.T[(sc * S + s) * static_cast<long>(U) + u] : make_float2(0.f, 0.f);
      d[m] = r[m];
      if (u < U) dv[u] = d[m];
      rs += cabs2(r[m]);
    }
#pragma unroll
    for (int kb = 0; kb < kRB; ++kb) x[kb] = make_float2(0.f, 0.f);
    float rn2 = warp_sum(rs);
    const float rn0 = rn2;
    bool broke = false;
    for (int k = 1; k <= K; ++k) {
      if (rn2 <= 1e-28f * rn0) continue;  // frozen (solvers.cpp:25-27)
      __syncwarp();
      float2 wr[kRB];
#pragma unroll
      for (int kb = 0; kb < kRB; ++kb) {
        const int b = l + 32 * kb;
        wr[kb] = make_float2(0.f, 0.f);
        if (b < B) {
          const float2* hr = Hs + b * HS;
          for (int u = 0; u < U; ++u) wr[kb] = cadd(wr[kb], cmul(hr[u], dv[u]));
          wv[b] = wr[kb];
        }
      }
      __syncwarp();
      float2 e[kRU];
      float cs = 0.f;
#pragma unroll
      for (int m = 0; m < kRU; ++m) {
        const int u = l + 32 * m;
        e[m] = make_float2(0.f, 0.f);
        if (u < U) {
          float2 acc = cscale(reg, d[m]);
          for (int b = 0; b < B; ++b) acc = cadd(acc, cmulc(Hs[b * HS + u], wv[b]));
          e[m] = acc;
          cs += cmulc(d[m], acc).x;
        }
      }
      const float curv = warp_sum(cs);
      if (curv < 1e-30f) {  // solvers.cpp:217-218
        broke = true;
        break;
      }
      const float alpha = rn2 / curv;
#pragma unroll
      for (int kb = 0; kb < kRB; ++kb) x[kb] = cadd(x[kb], cscale(alpha, wr[kb]));
      float rsn = 0.f;
#pragma unroll
      for (int m = 0; m < kRU; ++m) {
        r[m] = csub(r[m], cscale(alpha, e[m]));
        rsn += cabs2(r[m]);
      }
      const float rn = warp_sum(rsn);
      const float beta = rn / rn2;
      rn2 = rn;
#pragma unroll
      for (int m = 0; m < kRU; ++m) {
        const int u = l + 32 * m;
        d[m] = cadd(r[m], cscale(beta, d[m]));
        if (u < U) dv[u] = d[m];
      }
    }
    float qs = 0.f;
#pragma unroll
    for (int kb = 0; kb < kRB; ++kb) qs += cabs2(x[kb]);
    const float gain = sqrtf(warp_sum(qs));
    const bool zero = gain < 1e-30f;
    const long o = (sc * S + s) * static_cast<long>(B);
#pragma unroll
    for (int kb = 0; kb < kRB; ++kb) {
      const int b = l + 32 * kb;
      if (b >= B) continue;
      const float2 qv = broke ? make_float2(0.f, 0.f) : x[kb];
      if (p.q) p.q[o + b] = qv;
      if (p.s_out) p.s_out[o + b] = (broke || zero) ? make_float2(0.f, 0.f) : cscale(1.f / gain, qv);
    }
    if (l == 0) {
      if (p.gain) p.gain[sc * S + s] = (broke || zero) ? 0.f : gain;
      if (p.pstatus) p.pstatus[sc * S + s] = broke ? 1 : (zero ? 2 : 0);
    }
    __syncwarp();
  }
}

// One instantiation per method (M = sim::Method): each gets its own register
// allocation (the CGLS warps hold 8 antenna rows per lane in registers).
template <int M>
__global__ void __launch_bounds__(NT) alt_kernel(const KernelParams p) {
  extern __shared__ float2 sm[];
  const bool down = p.St > 0;
  const int B = p.B, U = p.U, S = down ? p.St : p.S;
  const int K = down ? p.Kt : p.K;
  const float reg = down ? p.rho_inv_d : p.rho_inv_u;
  AltSmem L;
  L.plan(B, U, S, M);
  const int HS = M == kCgls ? U + 1 : U;  // staged row stride of H
  float2* Hs = sm + L.hs;
  float2* A = sm + L.a;
  float2* G = sm + L.g;
  float2* Inv = sm + L.inv;
  float2* term = sm + L.term;
  float2* nxt = sm + L.next;
  float2* MF = sm + L.mf;
  float2* XS = sm + L.xs;
  float2* V = sm + L.vec;
  float* red = reinterpret_cast<float*>(sm + L.red);
  // CGLS: per-warp slots V[w (B + U) ..] (cgls_*_warps); explicit / Neumann
  // precoding: q = H_d^H v in V[0 .. B); then 3 x U floats: a_diag, g_diag, 1 / diag
  float2* vq = V;
  float* fl = reinterpret_cast<float*>(V + (M == kCgls ? NW * (B + U) : B));
  float* adg = fl;
  float* gdg = fl + U;
  float* dinv = fl + 2 * U;

  for (long sc = blockIdx.x; sc < p.n_sc; sc += gridDim.x) {
    // ---- stage H_u (downlink: H_u = H_d^H)
    auto stage_h = [&] {
      if (p.hd_layout) {
        const float2* src = p.H + sc * static_cast<long>(U) * B;
        for (int e = threadIdx.x; e < U * B; e += NT) {
          const int u = e / B, b = e - u * B;
          const float2 h = src[e];
          Hs[b * HS + u] = make_float2(h.x, -h.y);
        }
      } else {
        const float2* src = p.H + sc * static_cast<long>(B) * U;
        if (HS == U) {
          for (int e = threadIdx.x; e < U * B; e += NT) Hs[e] = src[e];
        } else {
          for (int e = threadIdx.x; e < U * B; e += NT) {
            const int b = e / U, u = e - b * U;
            Hs[b * HS + u] = src[e];
          }
        }
      }
      __syncthreads();
    };
    stage_h();
    if (!down) {
      // ================================================= detection
      if (M == kCgls) {
        // only the Gram diagonal (detect.cpp:249-256)
        for (int i = threadIdx.x; i < U; i += NT) {
          float d = 0.f;
          for (int b = 0; b < B; ++b) d += cabs2(Hs[b * HS + i]);
          gdg[i] = d;
          adg[i] = d + reg;
        }
        __syncthreads();
        cgls_detect_warps(p, sc, Hs, HS, V, gdg, adg, reg);
        __syncthreads();
        continue;
      }
      gram(Hs, B, U, reg, G, A);
      // matched filters b_s = H^H y_s
      for (int e = threadIdx.x; e < S * U; e += NT) {
        const int s = e / U, i = e - s * U;
        float2 acc = make_float2(0.f, 0.f);
        for (int b = 0; b < B; ++b)
          acc = cadd(acc, cmulc(Hs[b * U + i], p.Y[(sc * B + b) * static_cast<long>(S) + s]));
        MF[e] = acc;
      }
      __syncthreads();
      bool ok;
      if (M == kCholesky) {
        ok = cholesky_inverse(A, Inv, U);
        apply(Inv, MF, XS, U, S);  // xhat_s = A^-1 b_s (detect.cpp:145-152)
        __syncthreads();
        // mu / nu through WH = I - rho^-1 A^-1 (detect.cpp:154-178)
        for (int i = threadIdx.x; i < U; i += NT) {
          const float2 vii = Inv[i * U + i];
          const float mu = 1.f - reg * vii.x;
          float interf = 0.f, col = 0.f;
          for (int j = 0; j < U; ++j) {
            const float2 v = Inv[i * U + j];
            if (j != i) interf += reg * reg * cabs2(v);
            col += cabs2(Inv[j * U + i]);
          }
          const float noise = p.n0 * (vii.x - reg * col);
          const float rho = safe_rho(mu, p.es * interf + noise);
          for (int s = 0; s < S; ++s) put_detect(p, sc, s, i, XS[s * U + i], mu, rho, ok);
        }
      } else {  // Neumann (detect.cpp:274-326)
        ok = neumann_inverse(A, Inv, term, nxt, dinv, U, K);
        for (int i = threadIdx.x; i < U; i += NT) {
          float mu;
          if (K == 1) {
            mu = Inv[i * U + i].x * G[i * U + i].x;
          } else {
            float2 dg = make_float2(0.f, 0.f);
            for (int j = 0; j < U; ++j) dg = cadd(dg, cmul(Inv[i * U + j], G[j * U + i]));
            mu = dg.x;
          }
          const float nu2 = fmaxf(p.es * (mu - mu * mu), 1e-12f);
          const float rho = safe_rho(mu, nu2);
          for (int s = 0; s < S; ++s) {
            float2 acc = make_float2(0.f, 0.f);
            if (K == 1) {
              acc = cscale(Inv[i * U + i].x, MF[s * U + i]);
            } else {
              for (int j = 0; j < U; ++j) acc = cadd(acc, cmul(Inv[i * U + j], MF[s * U + j]));
            }
            put_detect(p, sc, s, i, acc, mu, rho, ok);
          }
        }
      }
      if (p.status)
        for (int s = threadIdx.x; s < S; s += NT) p.status[sc * S + s] = ok ? 0 : 4;
      __syncthreads();
      continue;
    }
    // =================================================== precoding
    const long ob = static_cast<long>(B);
    if (M == kCgls) {
      cgls_precode_warps(p, sc, Hs, HS, V, reg);
      __syncthreads();
      continue;
    }
    // explicit (Cholesky) / Neumann: v_s = A_d^-1 t_s, q_s = H_d^H v_s
    gram(Hs, B, U, reg, G, A);
    for (int e = threadIdx.x; e < S * U; e += NT) MF[e] = p.T[(sc * S) * static_cast<long>(U) + e];
    __syncthreads();
    const bool ok = M == kCholesky ? cholesky_inverse(A, Inv, U)
                                          : neumann_inverse(A, Inv, term, nxt, dinv, U, K);
    apply(Inv, MF, XS, U, S);  // v_s = A_d^-1 t_s
    __syncthreads();
    if (L.alias) stage_h();    // the Neumann terms overwrote the staged channel
    for (int s = 0; s < S; ++s) {
      mv(Hs, B, U, XS + s * U, vq);  // q = H_d^H v
      __syncthreads();
      float qs = 0.f;
      for (int b = threadIdx.x; b < B; b += NT) qs += cabs2(vq[b]);
      const float gain = sqrtf(block_sum(qs, red));
      const bool zero = gain < 1e-30f;
      const long o = (sc * S + s) * ob;
      for (int b = threadIdx.x; b < B; b += NT) {
        const float2 qv = ok ? vq[b] : make_float2(0.f, 0.f);
        if (p.q) p.q[o + b] = qv;
        if (p.s_out) p.s_out[o + b] = (!ok || zero) ? make_float2(0.f, 0.f) : cscale(1.f / gain, qv);
      }
      if (threadIdx.x == 0) {
        if (p.gain) p.gain[sc * S + s] = (!ok || zero) ? 0.f : gain;
        if (p.pstatus) p.pstatus[sc * S + s] = !ok ? 4 : (zero ? 2 : 0);
      }
      __syncthreads();
    }
  }
}

}  // namespace alt
}  // namespace cgm
