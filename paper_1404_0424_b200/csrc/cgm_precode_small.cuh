// cgm_precode_small.cuh -- fused CG precoder for small U (U <= 16), H_d in
// the reference layout [U][B] (precode_cg, precode.cpp:56-71).
//
// One WARP per subcarrier, persistent over subcarriers, no block-level
// barriers: a CTA-wide version spent a quarter of its warp time waiting at
// the barrier behind the one warp running the (latency-bound) CG, so here
// every warp owns its subcarrier end to end and the SM interleaves ~9 of
// them.  Per subcarrier the U x B channel is read from HBM ONCE
// (cp.async.bulk, one copy per row into padded shared-memory rows) and
// everything else happens in the warp:
//   1. A_d = H_d H_d^H (downlink_gram, precode.cpp:38-41): lower 4 x 4 tiles
//      x KP antenna ranges on the FFMA pipe, partials summed in a fixed order
//      (G == G^H exactly: one triangle + conjugate mirror, real diagonal);
//   2. K CG iterations on A_d + rho_d^-1 I for every transmit vector t
//      (solvers.cpp:37-72, same freeze / breakdown rules as K2): a group of
//      UP lanes per system, G read by columns (conflict-free), warp-shuffle
//      reductions;
//   3. q = H_d^H v from the staged channel, gain = ||q|| (fixed butterfly
//      order), s = q / gain, zero_input (precode.cpp:22-36).
// The split path runs a channel kernel and a solve kernel (G through the
// workspace, H_d read a second time for q); for U <= 16 the per-subcarrier
// work is small enough that one warp does it all.
#pragma once

#include "cgm_rows32.cuh"  // f2dup_lo / f2dup_hi

namespace cgm {

template <int UP>
struct PrecodeSmallGeo {
  static constexpr int NT = 32;            // one warp per CTA
  static constexpr int NB = UP / 4;
  static constexpr int NTILE = NB * (NB + 1) / 2;
  static constexpr int GL = UP;            // lanes per CG system
  static constexpr int GPW = 32 / GL;      // systems per warp at a time
  static constexpr int KP = 32 / NTILE;    // antenna ranges per tile (3 / 10)
  static constexpr int MAXQ = 16;          // B <= 512: q held 16 per lane
};

struct PrecodeSmallSmem {
  int bar, h, part, gs, ps, vs, st, total, ldh;
  __host__ __device__ static int align(int x) { return (x + 15) & ~15; }
  __host__ __device__ void plan(int UP, int B, int St) {
    const int nb = UP / 4, ntile = nb * (nb + 1) / 2, kp = 32 / ntile;
    ldh = B + 2;  // padded row: consecutive rows start 16 B apart in the banks
    int o = 0;
    bar = o; o = align(o + 8);
    h = o; o = align(o + UP * ldh * 8);
    part = o; o = align(o + ntile * 16 * kp * 8);
    gs = o; o = align(o + UP * UP * 8);
    ps = o; o = align(o + 32 * 8);  // GPW broadcast rows of UP
    vs = o; o = align(o + (St > 0 ? St : 1) * UP * 8);
    st = o; o = align(o + (St > 0 ? St : 1));
    total = o;
  }
};

template <int UP>
__global__ void __launch_bounds__(32) precode_small_kernel(const KernelParams p) {
  using PG = PrecodeSmallGeo<UP>;
  constexpr int GL = PG::GL, GPW = PG::GPW, KP = PG::KP;
  extern __shared__ __align__(128) unsigned char smem[];
  const int B = p.B, U = p.U, St = p.St;
  PrecodeSmallSmem L;
  L.plan(UP, B, St);
  const int LDH = L.ldh;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Hs = reinterpret_cast<float2*>(smem + L.h);
  float2* P = reinterpret_cast<float2*>(smem + L.part);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.st);
  const int lane = threadIdx.x;
  const bool tma = p.use_tma != 0;

  if (U < UP)  // padded rows stay zero for the whole kernel
    for (int e = lane; e < (UP - U) * LDH; e += 32) Hs[U * LDH + e] = make_float2(0.f, 0.f);
  if (tma && lane == 0) mbar_init(bar, 1);
  __syncwarp();

  // Gram work item: lower tile (rb, cb) x antenna-pair range [q0, q1),
  // visited from a per-part rotated start (bank spread)
  const int item_part = lane / PG::NTILE, item_tile = lane - item_part * PG::NTILE;
  const bool gram_busy = item_part < KP;
  int rb = 0;
  while ((rb + 1) * (rb + 2) / 2 <= item_tile) ++rb;
  const int cb = item_tile - rb * (rb + 1) / 2;
  const int q0 = (item_part * (B / 2)) / KP, q1 = ((item_part + 1) * (B / 2)) / KP;
  const int nq = q1 - q0;

  uint32_t phase = 0;
  for (long sc = blockIdx.x; sc < p.n_sc; sc += gridDim.x) {
    // the first pass's transmit vectors, loaded now so the latency hides
    // under the channel staging and the Gram
    float2 t_first = make_float2(0.f, 0.f);
    {
      const int grp = lane / GL, gl = lane - grp * GL;
      if (grp < St && gl < U) t_first = p.T[(sc * St + grp) * static_cast<long>(U) + gl];
    }
    // ------------------------------------------------------ stage H_d rows
    const float2* src = p.H + sc * static_cast<long>(U) * B;
    if (tma) {
      if (lane == 0) {
        fence_proxy_async();  // this warp's generic reads of Hs happen-before the async write
        mbar_expect_tx(bar, static_cast<uint32_t>(U) * B * 8u);
        for (int u = 0; u < U; ++u) bulk_g2s(Hs + u * LDH, src + u * B, B * 8u, bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      for (int e = lane; e < U * B; e += 32) {
        const int u = e / B, b = e - u * B;
        Hs[u * LDH + b] = src[e];
      }
      __syncwarp();
    }
    // ------------------------------------------ 1. A_d = H_d H_d^H partials
    if (gram_busy) {
      // packed FFMA2: a += x (pair) * y.x, b += x (pair) * y.y;
      // x conj(y) = (a.x + b.y, a.y - b.x)
      unsigned long long a[4][4], bb[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[r][c] = bb[r][c] = 0ull;
      const float2* hu = Hs + (rb * 4) * LDH;
      const float2* hv = Hs + (cb * 4) * LDH;
      int q = nq > 0 ? item_tile % nq : 0;
      for (int t = 0; t < nq; ++t) {
        const int b = 2 * (q0 + q);
        q = q + 1 == nq ? 0 : q + 1;
        ulonglong2 x[4], y[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          x[r] = *reinterpret_cast<const ulonglong2*>(hu + r * LDH + b);
          y[r] = *reinterpret_cast<const ulonglong2*>(hv + r * LDH + b);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ffma2(a[r][c], x[r].x, f2dup_lo(y[c].x));
            ffma2(bb[r][c], x[r].x, f2dup_hi(y[c].x));
            ffma2(a[r][c], x[r].y, f2dup_lo(y[c].y));
            ffma2(bb[r][c], x[r].y, f2dup_hi(y[c].y));
          }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 A2 = f2unpack(a[r][c]), B2 = f2unpack(bb[r][c]);
          P[((item_tile * 16) + r * 4 + c) * KP + item_part] = make_float2(A2.x + B2.y, A2.y - B2.x);
        }
    }
    __syncwarp();
    for (int e = lane; e < UP * UP; e += 32) {  // fixed-order part sums, lower entries
      const int u = e / UP, v = e - u * UP;
      if (v > u) continue;
      const int t = (u / 4) * (u / 4 + 1) / 2 + v / 4;
      const float2* pp = P + (t * 16 + (u % 4) * 4 + (v % 4)) * KP;
      float2 g = pp[0];
#pragma unroll
      for (int k = 1; k < KP; ++k) g = cadd(g, pp[k]);
      if (u == v) {
        Gs[u * UP + u] = make_float2(g.x, 0.f);
      } else {
        Gs[u * UP + v] = g;
        Gs[v * UP + u] = cconj(g);
      }
    }
    __syncwarp();
    // ------------------------------------------------------- 2. CG per t
    {
      const int grp = lane / GL, gl = lane - grp * GL;
      float2* Pw = Ps + grp * UP;
      for (int base = 0; base < St; base += GPW) {
        const int sys = base + grp;
        const bool live = sys < St;
        float2 b = make_float2(0.f, 0.f);
        if (live && gl < U)
          b = base == 0 ? t_first : p.T[(sc * St + sys) * static_cast<long>(U) + gl];
        float2 v = make_float2(0.f, 0.f), r = b, pp = b;
        Pw[gl] = b;
        float rn = cnorm(b);
        for (int o = GL / 2; o > 0; o >>= 1) rn += __shfl_xor_sync(0xffffffffu, rn, o);
        const float rn0 = rn;
        bool broke = false;
        __syncwarp();
        for (int k = 1; k <= p.Kt; ++k) {
          float2 e = make_float2(0.f, 0.f), e2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < UP; j += 2) {
            cfma_conj(e, Gs[j * UP + gl], Pw[j]);  // G[gl][j] = conj(G[j][gl])
            cfma_conj(e2, Gs[(j + 1) * UP + gl], Pw[j + 1]);
          }
          e = cadd(e, e2);
          e.x = fmaf(p.rho_inv_d, pp.x, e.x);
          e.y = fmaf(p.rho_inv_d, pp.y, e.y);
          float curv = pp.x * e.x + pp.y * e.y;
          for (int o = GL / 2; o > 0; o >>= 1) curv += __shfl_xor_sync(0xffffffffu, curv, o);
          const bool frozen = !(rn > 1e-28f * rn0);  // solvers.cpp:21,25-27
          const bool go = live && !frozen && !broke;
          if (go && curv < 1e-30f) broke = true;     // solvers.cpp:55-57
          const bool upd = go && !broke;
          const float alpha = upd ? __fdividef(rn, curv) : 1.f;
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
            const float beta = __fdividef(rnx, rn);
            rn = rnx;
            pp.x = fmaf(beta, pp.x, r.x);
            pp.y = fmaf(beta, pp.y, r.y);
            Pw[gl] = pp;
          }
          __syncwarp();
        }
        if (live) {
          Vs[sys * UP + gl] = v;
          if (gl == 0) sys_st[sys] = broke ? 1 : 0;
        }
      }
    }
    __syncwarp();
    // ------------------------------ 3. q = H_d^H v, gain, s (precode.cpp:22-36)
    for (int s = 0; s < St; ++s) {
      const bool ok = sys_st[s] == 0;
      float2 qv[PG::MAXQ];
      float nrm = 0.f;
#pragma unroll
      for (int m = 0; m < PG::MAXQ; ++m) {
        const int b = lane + 32 * m;
        qv[m] = make_float2(0.f, 0.f);
        if (b < B) {
#pragma unroll
          for (int u = 0; u < UP; ++u) cfma_conj(qv[m], Hs[u * LDH + b], Vs[s * UP + u]);
          nrm += cnorm(qv[m]);
        }
      }
      nrm = group_sum<32>(nrm);  // fixed butterfly order
      const float g = sqrtf(nrm);
      const bool zero = ok && !(g > 0.f);
      const float inv = (ok && !zero) ? 1.f / g : 0.f;
      const long ob = (sc * St + s) * static_cast<long>(B);
#pragma unroll
      for (int m = 0; m < PG::MAXQ; ++m) {
        const int b = lane + 32 * m;
        if (b < B) {
          if (p.q) p.q[ob + b] = ok ? qv[m] : make_float2(0.f, 0.f);
          if (p.s_out) p.s_out[ob + b] = cscale(inv, qv[m]);
        }
      }
      if (lane == 0) {
        if (p.gain) p.gain[sc * St + s] = (ok && !zero) ? g : 0.f;
        if (p.pstatus) p.pstatus[sc * St + s] = ok ? (zero ? 2 : 0) : 1;
      }
    }
    __syncwarp();  // Hs / Vs reads done before the next subcarrier's copy
  }
}

}  // namespace cgm
