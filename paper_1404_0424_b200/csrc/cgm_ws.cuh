// cgm_ws.cuh -- persistent, warp-specialised pipeline kernel for U = 32
// (BASELINE configs 2, 4a and 5), sm_100a.
//
//   warps [0, gw)   "Gram warps": consume a ring of NST shared-memory stages
//                   filled by TMA bulk copies (cp.async.bulk + mbarrier
//                   complete_tx) with CB-row chunks of H and of the S
//                   received vectors, accumulate G = H^H H (lower triangle)
//                   and the matched filter H^H Y in 4x4 register tiles
//                   (split-K lanes reduced with shuffles), publish them to
//                   one of two G/MF buffers, and (exact tracker) build the
//                   Chebyshev basis T_1..T_K of that subcarrier.
//   warps [gw, 16)  "CG warps": for the previous subcarrier, run K CG
//                   iterations for every uplink / downlink system (one warp
//                   per system slot, lane = user, up to NSMAX systems per
//                   warp interleaved), the SINR tracker, the LLR epilogue,
//                   and the precoder's q = H_d^H v (H re-read from L2).
//
// mbarriers: full[NST] / empty[NST] for the chunk ring (the producer is
// lane 0 of warp 0, running NST chunks ahead across subcarrier boundaries),
// gfull[2] / gempty[2] for the G/MF(/basis) double buffer.  Named barriers
// sync inside a role; the two roles never __syncthreads.  The per-instance
// mathematics is exactly that of cgm_kernels.cuh (same reference citations).
#pragma once

#include "cgm_kernels.cuh"

namespace cgm {

constexpr int WS_UP = 32;
constexpr int WS_NT = 512;
constexpr int WS_NW = WS_NT / 32;
constexpr int WS_CB = 64;    // rows of H / Y per ring stage
constexpr int WS_NST = 4;    // ring stages
constexpr int WS_NSMAX = 2;  // systems per CG warp per pass

struct WsLayout {
  int bars, ring, stage_bytes, ys_off;
  int gm, gm_bytes, g_off, mf_off, t_off, cd_off;
  int ps, vs, qs, hist, sys_st, mu, rho, coef, gpart, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int St, int K, bool exact) {
    constexpr int UP = WS_UP;
    const int nsys = S + St;
    int o = 0;
    bars = o; o = align(o + (2 * WS_NST + 4) * 8);
    // stage = CB rows of H [CB][32] then CB rows of Y [CB][S] (+64 B so the
    // last row's 4-wide tile reads stay in bounds)
    ys_off = WS_CB * UP * 8;
    stage_bytes = align(ys_off + WS_CB * S * 8 + 64);
    ring = o; o = align(o + WS_NST * stage_bytes);
    g_off = 0;
    mf_off = UP * UP * 8;
    cd_off = mf_off + S * UP * 8;
    t_off = align(cd_off + 16);
    gm_bytes = align(t_off + (exact ? K * UP * UP * 8 : 0));
    gm = o; o = align(o + 2 * gm_bytes);
    ps = o; o = align(o + nsys * UP * 8);
    vs = o; o = align(o + nsys * UP * 8);
    qs = o; o = align(o + St * B * 8);
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    sys_st = o; o = align(o + nsys);
    mu = o; o = align(o + (exact ? S * UP * 4 : 0));
    rho = o; o = align(o + (exact ? S * UP * 4 : 0));
    coef = o; o = align(o + (exact ? S * 2 * (K + 2) * 4 : 0));
    gpart = o; o = align(o + ((B + 31) / 32) * (St > 0 ? St : 1) * 4);
    total = o;
  }
};

// Issue ring chunk g (= local subcarrier i, chunk c) into its stage.
__device__ __forceinline__ void ws_issue(const KernelParams& p, unsigned char* smem,
                                         const WsLayout& L, uint64_t* full, long g, int nch) {
  constexpr int UP = WS_UP;
  const int st = static_cast<int>(g % WS_NST);
  const long i = g / nch;
  const int c = static_cast<int>(g - i * nch);
  const long sc = blockIdx.x + i * gridDim.x;
  const int b0 = c * WS_CB;
  const int rows = min(WS_CB, p.B - b0);
  unsigned char* stage = smem + L.ring + st * L.stage_bytes;
  fence_proxy_async();
  mbar_expect_tx(full + st, static_cast<uint32_t>(rows) * (UP * 8 + p.S * 8));
  bulk_g2s(stage, p.H + (sc * p.B + b0) * UP, static_cast<uint32_t>(rows) * UP * 8, full + st);
  if (p.S > 0)
    bulk_g2s(stage + L.ys_off, p.Y + (sc * p.B + b0) * p.S, static_cast<uint32_t>(rows) * p.S * 8,
             full + st);
}

// Gram role with SPL split lanes per tile.
template <int SPL, bool EXACT>
__device__ __forceinline__ void ws_gram_role(const KernelParams& p, unsigned char* smem,
                                             const WsLayout& L, int gw, long n_local) {
  constexpr int UP = WS_UP;
  constexpr int TPW = 32 / SPL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + WS_NST;
  uint64_t* gfull = bars + 2 * WS_NST;
  uint64_t* gempty = gfull + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gtid = threadIdx.x;  // Gram warps are the first gw warps
  const int S = p.S;
  const int nb = UP / 4, n_gram = nb * (nb + 1) / 2, nsb = (S + 3) / 4;
  const int n_tiles = n_gram + nb * nsb;
  const int tile = warp * TPW + lane / SPL, part = lane % SPL;
  const bool active = tile < n_tiles;
  int ib = 0, jb = 0;
  const bool is_gram = tile < n_gram;
  if (active) {
    if (is_gram) {
      tri_block(tile, ib, jb);
    } else {  // neighbouring lanes share the Y block (broadcast loads)
      jb = (tile - n_gram) / nb;
      ib = (tile - n_gram) - jb * nb;
    }
  }
  const int nch = (p.B + WS_CB - 1) / WS_CB;
  const long total = n_local * nch;
  const bool producer = (warp == 0 && lane == 0);
  if (producer)
    for (long g = 0; g < total && g < WS_NST; ++g) ws_issue(p, smem, L, full, g, nch);
  constexpr int rpl = WS_CB / SPL;
  for (long i = 0; i < n_local; ++i) {
    float2 acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
    for (int c = 0; c < nch; ++c) {
      const long g = i * nch + c;
      const int st = static_cast<int>(g % WS_NST);
      const uint32_t ph = static_cast<uint32_t>((g / WS_NST) & 1);
      mbar_wait(full + st, ph);
      const float2* hc = reinterpret_cast<const float2*>(smem + L.ring + st * L.stage_bytes);
      const float2* yc = reinterpret_cast<const float2*>(smem + L.ring + st * L.stage_bytes + L.ys_off);
      const int rows = min(WS_CB, p.B - c * WS_CB);
      const int r0 = part * rpl, r1 = min(rows, r0 + rpl);
      if (active && !(p.debug & 2)) {
        if (is_gram)
          tile4x4<true>(acc, hc, UP, ib * 4, hc, UP, 1, jb * 4, 1 << 30, r0, r1);
        else if ((S & 1) == 0)
          tile4x4<true>(acc, hc, UP, ib * 4, yc, S, 1, jb * 4, 1 << 30, r0, r1);
        else
          tile4x4<false>(acc, hc, UP, ib * 4, yc, S, 1, jb * 4, S, r0, r1);
      }
      mbar_arrive(empty + st);
      if (producer && g + WS_NST < total) {
        mbar_wait(empty + st, ph);  // every Gram thread is done with chunk g
        ws_issue(p, smem, L, full, g + WS_NST, nch);
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
    const int b = static_cast<int>(i & 1);
    mbar_wait(gempty + b, static_cast<uint32_t>(((i >> 1) & 1) ^ 1));
    unsigned char* gmb = smem + L.gm + b * L.gm_bytes;
    float2* Gs = reinterpret_cast<float2*>(gmb + L.g_off);
    float2* MF = reinterpret_cast<float2*>(gmb + L.mf_off);
    if (active && part == 0) {
      if (is_gram) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ii = ib * 4 + r, j = jb * 4 + c;
            if (j < ii) {
              Gs[ii * UP + j] = acc[r][c];
              Gs[j * UP + ii] = cconj(acc[r][c]);
            } else if (j == ii) {
              Gs[ii * UP + ii] = make_float2(acc[r][c].x, 0.f);
            }
          }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int s = jb * 4 + c;
            if (s < S) MF[s * UP + ib * 4 + r] = acc[r][c];
          }
      }
    }
    if (EXACT && S > 0) {
      // Chebyshev basis of A = G + rho_u^-1 I for this subcarrier
      const int K = p.K;
      float* cd = reinterpret_cast<float*>(gmb + L.cd_off);
      float2* Tb = reinterpret_cast<float2*>(gmb + L.t_off);
      named_sync(2, gw * 32);
      if (warp == 0) {
        float tr = 0.f, fr = 0.f;
        tr = Gs[lane * UP + lane].x + p.rho_inv_u;
        tr = group_sum<32>(tr);
        const float cc = tr / UP;
        for (int e = lane; e < UP * UP; e += 32) {
          float2 a = Gs[e];
          if (e / UP == e % UP) a.x += p.rho_inv_u - cc;
          fr += cnorm(a);
        }
        fr = group_sum<32>(fr);
        float d = 2.f * sqrtf(fr / UP);
        if (!(d > 1e-6f * fmaxf(fabsf(cc), 1e-30f))) d = fmaxf(fabsf(cc), 1.f);
        if (lane == 0) { cd[0] = cc; cd[1] = d; }
      }
      named_sync(2, gw * 32);
      const float cc = cd[0], invd = 1.f / cd[1];
      for (int e = gtid; e < UP * UP; e += gw * 32) {
        float2 a = Gs[e];
        if (e / UP == e % UP) a.x += p.rho_inv_u - cc;
        Tb[e] = cscale(invd, a);
      }
      named_sync(2, gw * 32);
      for (int m = 1; m < K; ++m) {
        const float2* T1 = Tb;
        const float2* Tm = Tb + (m - 1) * UP * UP;
        float2* Tn = Tb + m * UP * UP;
        const float2* Tp = m >= 2 ? Tb + (m - 2) * UP * UP : nullptr;
        // 36 lower 4x4 tiles, 4 split lanes each, over the gw Gram warps
        for (int base = warp * 8; base < n_gram; base += gw * 8) {
          const int t = base + lane / 4, pt = lane % 4;
          float2 a2[4][4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) a2[r][c] = make_float2(0.f, 0.f);
          int tib = 0, tjb = 0;
          if (t < n_gram) {
            tri_block(t, tib, tjb);
            tile4x4<true>(a2, T1, UP, tib * 4, Tm, UP, 1, tjb * 4, 1 << 30, pt * 8, pt * 8 + 8);
          }
#pragma unroll
          for (int o = 1; o < 4; o <<= 1)
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                a2[r][c].x += __shfl_xor_sync(0xffffffffu, a2[r][c].x, o);
                a2[r][c].y += __shfl_xor_sync(0xffffffffu, a2[r][c].y, o);
              }
          if (t < n_gram && pt == 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int ii = tib * 4 + r, j = tjb * 4 + c;
                if (j > ii) continue;
                const float2 prev = Tp ? Tp[ii * UP + j] : make_float2(ii == j ? 1.f : 0.f, 0.f);
                const float2 val =
                    make_float2(2.f * a2[r][c].x - prev.x, 2.f * a2[r][c].y - prev.y);
                if (ii == j) {
                  Tn[ii * UP + ii] = make_float2(val.x, 0.f);
                } else {
                  Tn[ii * UP + j] = val;
                  Tn[j * UP + ii] = cconj(val);
                }
              }
          }
        }
        named_sync(2, gw * 32);
      }
    }
    mbar_arrive(gfull + b);
  }
}

template <bool EXACT>
__device__ __forceinline__ void ws_cg_role(const KernelParams& p, unsigned char* smem,
                                           const WsLayout& L, int gw, long n_local) {
  constexpr int UP = WS_UP;
  const int cw = WS_NW - gw;
  const int ctid = threadIdx.x - gw * 32;
  const int cwarp = (threadIdx.x >> 5) - gw, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* gfull = bars + 2 * WS_NST;
  uint64_t* gempty = gfull + 2;
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* MUs = reinterpret_cast<float*>(smem + L.mu);
  float* RHOs = reinterpret_cast<float*>(smem + L.rho);
  float* coef = reinterpret_cast<float*>(smem + L.coef);
  float* gpart = reinterpret_cast<float*>(smem + L.gpart);
  const int S = p.S, St = p.St, B = p.B;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  const int u = lane;  // lane = user (U = 32)

  for (long i = 0; i < n_local; ++i) {
    const long sc = blockIdx.x + i * gridDim.x;
    const int b = static_cast<int>(i & 1);
    mbar_wait(gfull + b, static_cast<uint32_t>((i >> 1) & 1));
    const unsigned char* gmb = smem + L.gm + b * L.gm_bytes;
    const float2* Gs = reinterpret_cast<const float2*>(gmb + L.g_off);
    const float2* MF = reinterpret_cast<const float2*>(gmb + L.mf_off);
    const float gdiag = Gs[u * UP + u].x;

    // ------------------------------------------------------------- CG
    for (int base = cwarp; base < ((p.debug & 1) ? 0 : nsys); base += cw * WS_NSMAX) {
      int sys[WS_NSMAX];
      bool live[WS_NSMAX], down[WS_NSMAX];
      float reg[WS_NSMAX];
      int iters[WS_NSMAX];
      float2 v[WS_NSMAX], r[WS_NSMAX], pp[WS_NSMAX];
      int nact = 0;
#pragma unroll
      for (int s = 0; s < WS_NSMAX; ++s) {
        sys[s] = base + s * cw;
        live[s] = sys[s] < nsys;
        nact += live[s] ? 1 : 0;
        down[s] = sys[s] >= S;
        reg[s] = down[s] ? p.rho_inv_d : p.rho_inv_u;
        iters[s] = live[s] ? (down[s] ? p.Kt : p.K) : 0;
        float2 bv = make_float2(0.f, 0.f);
        if (live[s])
          bv = down[s] ? p.T[(sc * St + (sys[s] - S)) * UP + u] : MF[sys[s] * UP + u];
        v[s] = make_float2(0.f, 0.f);
        r[s] = bv;
        pp[s] = bv;
        if (live[s]) Ps[sys[s] * UP + u] = bv;
      }
      float rn[WS_NSMAX], rn0[WS_NSMAX];
#pragma unroll
      for (int s = 0; s < WS_NSMAX; ++s) rn[s] = cnorm(r[s]);
      group_sum_n<32, WS_NSMAX>(rn);
      bool broke[WS_NSMAX];
      float f0[WS_NSMAX], f1[WS_NSMAX], f2[WS_NSMAX];
      float am1[WS_NSMAX], am2[WS_NSMAX], bm1[WS_NSMAX], bm2[WS_NSMAX];
#pragma unroll
      for (int s = 0; s < WS_NSMAX; ++s) {
        rn0[s] = rn[s];
        broke[s] = false;
        am1[s] = am2[s] = 1.f;
        bm1[s] = bm2[s] = 0.f;
        f0[s] = f1[s] = f2[s] = 0.f;
      }
      __syncwarp();
      for (int k = 1; k <= Kmax; ++k) {
        // e = (G + reg I) p: G read as column u (conflict-free), p_j
        // broadcast; the G loads are shared by the warp's systems
        float2 e[WS_NSMAX], e2[WS_NSMAX];
#pragma unroll
        for (int s = 0; s < WS_NSMAX; ++s) e[s] = e2[s] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int j = 0; j < UP; j += 2) {
          const float2 g0 = cconj(Gs[j * UP + u]);        // G[u][j]
          const float2 g1 = cconj(Gs[(j + 1) * UP + u]);  // G[u][j+1]
#pragma unroll
          for (int s = 0; s < WS_NSMAX; ++s) {
            if (s < nact) {
              const float4 pj = *reinterpret_cast<const float4*>(Ps + sys[s] * UP + j);
              cfma(e[s], g0, make_float2(pj.x, pj.y));
              cfma(e2[s], g1, make_float2(pj.z, pj.w));
            }
          }
        }
#pragma unroll
        for (int s = 0; s < WS_NSMAX; ++s) e[s] = cadd(e[s], e2[s]);
        float curv[WS_NSMAX];
#pragma unroll
        for (int s = 0; s < WS_NSMAX; ++s) {
          e[s].x = fmaf(reg[s], pp[s].x, e[s].x);
          e[s].y = fmaf(reg[s], pp[s].y, e[s].y);
          curv[s] = pp[s].x * e[s].x + pp[s].y * e[s].y;  // Re p^H e
        }
        group_sum_n<32, WS_NSMAX>(curv);
        float alpha[WS_NSMAX], beta[WS_NSMAX], rnx[WS_NSMAX];
        bool upd[WS_NSMAX];
#pragma unroll
        for (int s = 0; s < WS_NSMAX; ++s) {
          const bool step = k <= iters[s];
          const bool frozen = !(rn[s] > 1e-28f * rn0[s]);  // solvers.cpp:21,25-27
          const bool go = step && !frozen && !broke[s];
          if (go && curv[s] < 1e-30f) broke[s] = true;    // solvers.cpp:55-57
          upd[s] = go && !broke[s];
          alpha[s] = upd[s] ? rn[s] / curv[s] : 1.f;
          beta[s] = 0.f;
          if (upd[s]) {
            v[s].x = fmaf(alpha[s], pp[s].x, v[s].x);
            v[s].y = fmaf(alpha[s], pp[s].y, v[s].y);
            r[s].x = fmaf(-alpha[s], e[s].x, r[s].x);
            r[s].y = fmaf(-alpha[s], e[s].y, r[s].y);
          }
          rnx[s] = cnorm(r[s]);
        }
        group_sum_n<32, WS_NSMAX>(rnx);
        __syncwarp();
#pragma unroll
        for (int s = 0; s < WS_NSMAX; ++s) {
          if (upd[s]) {
            beta[s] = rnx[s] / rn[s];
            rn[s] = rnx[s];
            pp[s].x = fmaf(beta[s], pp[s].x, r[s].x);
            pp[s].y = fmaf(beta[s], pp[s].y, r[s].y);
            Ps[sys[s] * UP + u] = pp[s];
          }
          if (k <= iters[s]) {
            if (!down[s]) {
              if (EXACT) {
                if (lane == 0) {
                  hist[(sys[s] * Kmax + (k - 1)) * 2 + 0] = alpha[s];
                  hist[(sys[s] * Kmax + (k - 1)) * 2 + 1] = beta[s];
                }
              } else {
                // Eq. (11) on the diagonal (detect.cpp:409-427)
                float nf;
                if (k == 1) {
                  nf = alpha[s];
                } else {
                  const float c1 = alpha[s] * (1.f + bm1[s]) / am1[s];
                  const float c2 = alpha[s] * bm2[s] / am2[s];
                  nf = f0[s] + (c1 - alpha[s] * (gdiag + reg[s])) * (f0[s] - f1[s]) -
                       c2 * (f1[s] - f2[s]);
                }
                f2[s] = f1[s];
                f1[s] = f0[s];
                f0[s] = nf;
              }
            }
            am2[s] = am1[s]; am1[s] = alpha[s];
            bm2[s] = bm1[s]; bm1[s] = beta[s];
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int s = 0; s < WS_NSMAX; ++s) {
        if (!live[s]) continue;
        if (lane == 0) sys_st[sys[s]] = broke[s] ? 1 : 0;
        if (EXACT || down[s]) {
          Vs[sys[s] * UP + u] = v[s];
          continue;
        }
        // approx uplink epilogue (detect.cpp:435-441, :68-86), straight from the lane
        if (u < p.U) {
          const long o = (sc * S + sys[s]) * static_cast<long>(p.U) + u;
          const bool ok = !broke[s];
          const float2 xh = ok ? v[s] : make_float2(0.f, 0.f);
          const float mu_u = ok ? f0[s] * gdiag : 0.f;
          const float rho_u = ok ? gdiag / p.n0 : 0.f;
          if (p.xhat) p.xhat[o] = xh;
          if (p.mu) p.mu[o] = mu_u;
          if (p.rho) p.rho[o] = rho_u;
          if (p.llr) store_llrs(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
          if (p.status && lane == 0) p.status[sc * S + sys[s]] = ok ? 0 : 1;
        }
      }
    }

    // ------------------------------------------ exact tracker extraction
    if (EXACT && S > 0) {
      const int K = p.K;
      const float* cd = reinterpret_cast<const float*>(gmb + L.cd_off);
      const float2* Tb = reinterpret_cast<const float2*>(gmb + L.t_off);
      named_sync(1, cw * 32);
      const double cc = cd[0], dd = cd[1];
      for (int s = ctid; s < S; s += cw * 32) {
        double l0[kMaxK + 2], l1[kMaxK + 2], l2[kMaxK + 2], tmp[kMaxK + 2], d1[kMaxK + 2];
        const int n = K + 2;
        for (int m = 0; m < n; ++m) l0[m] = l1[m] = l2[m] = 0.0;
        double a_m1 = 1.0, a_m2 = 1.0, b_m1 = 0.0, b_m2 = 0.0;
        auto mulA = [&](const double* x, double* out) {
          for (int m = 0; m < n; ++m) out[m] = cc * x[m];
          for (int m = 0; m < n; ++m) {
            const double h = dd * x[m];
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
            l0[0] = a;
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
      named_sync(1, cw * 32);
      {
        const int ii = lane;
        for (int s0 = cwarp; s0 < S; s0 += cw * 2) {
          const int s1 = s0 + cw;
          const bool has1 = s1 < S;
          const float* cl0 = coef + s0 * 2 * (K + 2);
          const float* cb0 = cl0 + (K + 2);
          const float* cl1 = coef + (has1 ? s1 : s0) * 2 * (K + 2);
          const float* cb1 = cl1 + (K + 2);
          float ib2[2] = {0.f, 0.f}, ibl[2] = {0.f, 0.f}, mu_i[2] = {0.f, 0.f};
          for (int j = 0; j < UP; ++j) {
            float2 B0 = make_float2(ii == j ? cb0[0] : 0.f, 0.f), L0 = make_float2(ii == j ? cl0[0] : 0.f, 0.f);
            float2 B1 = make_float2(ii == j ? cb1[0] : 0.f, 0.f), L1 = make_float2(ii == j ? cl1[0] : 0.f, 0.f);
            for (int m = 1; m <= K; ++m) {
              const float2 t = cconj(Tb[(m - 1) * UP * UP + j * UP + ii]);  // T_m[i][j]
              B0.x = fmaf(cb0[m], t.x, B0.x); B0.y = fmaf(cb0[m], t.y, B0.y);
              B1.x = fmaf(cb1[m], t.x, B1.x); B1.y = fmaf(cb1[m], t.y, B1.y);
              if (m < K) {
                L0.x = fmaf(cl0[m], t.x, L0.x); L0.y = fmaf(cl0[m], t.y, L0.y);
                L1.x = fmaf(cl1[m], t.x, L1.x); L1.y = fmaf(cl1[m], t.y, L1.y);
              }
            }
            if (j == ii) { mu_i[0] = B0.x; mu_i[1] = B1.x; }
            else { ib2[0] += cnorm(B0); ib2[1] += cnorm(B1); }
            ibl[0] += B0.x * L0.x + B0.y * L0.y;
            ibl[1] += B1.x * L1.x + B1.y * L1.y;
          }
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (t == 1 && !has1) break;
            const int s = t ? s1 : s0;
            const float nu2 = ib2[t] * p.es + ibl[t] * p.n0;
            MUs[s * UP + ii] = mu_i[t];
            RHOs[s * UP + ii] = nu2 <= 0.f ? 0.f : mu_i[t] * mu_i[t] / nu2;
          }
        }
      }
      named_sync(1, cw * 32);
      for (int e = ctid; e < S * p.U; e += cw * 32) {
        const int s = e / p.U, uu = e - s * p.U;
        const long o = (sc * S + s) * static_cast<long>(p.U) + uu;
        const bool ok = sys_st[s] == 0;
        const float2 xh = ok ? Vs[s * UP + uu] : make_float2(0.f, 0.f);
        const float m = ok ? MUs[s * UP + uu] : 0.f;
        const float rr = ok ? RHOs[s * UP + uu] : 0.f;
        if (p.xhat) p.xhat[o] = xh;
        if (p.mu) p.mu[o] = m;
        if (p.rho) p.rho[o] = rr;
        if (p.llr) store_llrs(xh, m, rr, p.bits, p.llr + o * p.bits);
      }
      if (p.status)
        for (int s = ctid; s < S; s += cw * 32) p.status[sc * S + s] = sys_st[s];
    }

    // --------------------------------------------- precode q = H_d^H v
    if (St > 0) {
      named_sync(1, cw * 32);
      const float2* Hg = p.H + sc * static_cast<long>(B) * UP;  // L2-resident re-read
      const int nrb = (B + 31) / 32;
      for (int rb = cwarp; rb < nrb; rb += cw) {
        const int bidx = rb * 32 + lane;
        const bool okb = bidx < B;
        for (int ts0 = 0; ts0 < St; ts0 += 8) {
          float2 acc[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[t] = make_float2(0.f, 0.f);
          const float4* hrow = reinterpret_cast<const float4*>(Hg + (okb ? bidx : 0) * UP);
#pragma unroll 4
          for (int uu = 0; uu < UP; uu += 2) {
            const float4 h = __ldg(hrow + uu / 2);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (ts0 + t < St) {
                const float4 vv = *reinterpret_cast<const float4*>(Vs + (S + ts0 + t) * UP + uu);
                cfma(acc[t], make_float2(h.x, h.y), make_float2(vv.x, vv.y));
                cfma(acc[t], make_float2(h.z, h.w), make_float2(vv.z, vv.w));
              }
            }
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            if (ts0 + t < St) {
              if (okb) Qs[(ts0 + t) * B + bidx] = acc[t];
              float n = okb ? cnorm(acc[t]) : 0.f;
              n = group_sum<32>(n);
              if (lane == 0) gpart[rb * St + ts0 + t] = n;
            }
          }
        }
      }
      named_sync(1, cw * 32);
      for (int ts = cwarp; ts < St; ts += cw) {
        const int sysi = S + ts;
        const bool ok = sys_st[sysi] == 0;
        float nrm = 0.f;
        for (int rb = 0; rb < nrb; ++rb) nrm += gpart[rb * St + ts];  // fixed order
        const float g = sqrtf(nrm);
        const bool zero = ok && !(g > 0.f);
        const float inv = (ok && !zero) ? 1.f / g : 0.f;
        const long ob = (sc * St + ts) * static_cast<long>(B);
        for (int bb = lane; bb < B; bb += 32) {
          const float2 q = Qs[ts * B + bb];
          if (p.q) p.q[ob + bb] = ok ? q : make_float2(0.f, 0.f);
          if (p.s_out) p.s_out[ob + bb] = cscale(inv, q);
        }
        if (lane == 0) {
          if (p.gain) p.gain[sc * St + ts] = (ok && !zero) ? g : 0.f;
          if (p.pstatus) p.pstatus[sc * St + ts] = ok ? (zero ? 2 : 0) : 1;
        }
      }
    }
    named_sync(1, cw * 32);  // CG-private buffers are reused by the next subcarrier
    mbar_arrive(gempty + b);
  }
}

template <bool EXACT>
__global__ void __launch_bounds__(WS_NT, 1) ws_kernel(const KernelParams p, int gw) {
  extern __shared__ __align__(128) unsigned char smem[];
  WsLayout L;
  L.plan(p.B, p.S, p.St, p.K > p.Kt ? p.K : p.Kt, EXACT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  const int cw = WS_NW - gw;
  if (threadIdx.x == 0) {
    for (int s = 0; s < WS_NST; ++s) {
      mbar_init(bars + s, 1);                    // full: producer arrive + tx bytes
      mbar_init(bars + WS_NST + s, gw * 32);     // empty: every Gram thread
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bars + 2 * WS_NST + b, gw * 32);  // gfull
      mbar_init(bars + 2 * WS_NST + 2 + b, cw * 32);  // gempty
    }
  }
  __syncthreads();
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int warp = threadIdx.x >> 5;
  if (warp < gw) {
    const int S = p.S;
    const int n_tiles = 36 + 8 * ((S + 3) / 4);
    if (n_tiles <= gw * 8)
      ws_gram_role<4, EXACT>(p, smem, L, gw, n_local);
    else if (n_tiles <= gw * 16)
      ws_gram_role<2, EXACT>(p, smem, L, gw, n_local);
    else
      ws_gram_role<1, EXACT>(p, smem, L, gw, n_local);
  } else {
    ws_cg_role<EXACT>(p, smem, L, gw, n_local);
  }
}

}  // namespace cgm
