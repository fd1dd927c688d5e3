// cgm_split.cuh -- the production path: two kernels per chunk of subcarriers.
//
//   K1 channel_kernel  (one CTA per subcarrier, persistent grid-stride)
//      TMA-stage H and Y, form G = H^H H (lower 4x4 tiles + mirror) and the
//      matched filter H^H Y in register tiles with shuffle-reduced split-K,
//      Writes them to a workspace sized to stay L2-resident for the next
//      kernels (the exact tracker's row moments, cgm_moments.cuh, and K2).
//        replaces gram_regularized (linalg.cpp:59-101), matvec_adjoint
//        (linalg.cpp:116-126) and the U^3 part of ExactSinrTracker::step
//        (detect.cpp:336-368, see cgm_kernels.cuh for the basis argument)
//   K2 solve_kernel    (one CTA per subcarrier, many CTAs per SM)
//      one lane group per system (uplink vector or downlink t): K CG
//      iterations on G + rho^-1 I (solvers.cpp:37-72) with the approximate
//      tracker (detect.cpp:397-441) or the exact one's coefficient recursion
//      + extraction from the basis (detect.cpp:330-395), max-log LLRs
//      (detect.cpp:57-86), and the precoder's q = H_d^H v, gain, s
//      (precode.cpp:22-71).
//
// The split keeps both kernels at high occupancy: K1 is FFMA/tile bound,
// K2 is latency bound (short dependent CG chains) and needs many resident
// warps -- fusing them into one CTA serialises the two regimes.
#pragma once

#include <type_traits>

#include "cgm_moments.cuh"

namespace cgm {

// K1 shared memory: two TMA stages of {H [B][UP], Y [B][S]} (the next
// subcarrier is prefetched while the current one is contracted), the Gram
// matrix.
template <int UP>
struct K1Smem {
  int bar, slot, hs, ys, gs, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int nstage) {
    const int Sp = (S + 1) & ~1;  // Y rows padded to an even length (16B aligned)
    int o = 0;
    bar = o; o = align(o + 32);
    hs = o;
    ys = align(B * UP * 8);
    slot = align(ys + B * Sp * 8 + 64);  // +64: last-row 4-wide tile reads
    o = align(o + nstage * slot);
    gs = o; o = align(o + UP * UP * 8);
    lut = o; o = align(o + 2 * 512);  // per-tile (ib, jb), <= 512 tiles
    total = o;
  }
  int lut;
};

// Host/device-consistent work split of K1: 4x4 tiles x `spl` k-parts as
// thread-granular work items (item = part * n_tiles + tile); all parts'
// partial tiles are parked in the consumed TMA stage and summed by every
// thread in a fixed order.
struct K1Split {
  int nstage, spl, wpp, n_tiles;
  __host__ __device__ void plan(int UP, int B, int S) {
    const int nb = UP / 4;
    n_tiles = nb * (nb + 1) / 2 + nb * ((S + 3) / 4);
    const int Sp = (S + 1) & ~1;
    const int stage_bytes = B * UP * 8 + B * Sp * 8;
    int s = 320 / n_tiles;                                  // <= 10 warps per CTA
    const int cap_k = B / 16 > 0 ? B / 16 : 1;              // >= 16 rows per part
    const int cap_m = stage_bytes / (n_tiles * 128);        // partials fit in the stage
    s = s > cap_k ? cap_k : s;
    s = s > cap_m ? cap_m : s;
    spl = s < 1 ? 1 : s;
    wpp = (spl * n_tiles + 31) / 32;  // total warps (name kept for the params field)
    if (wpp > 10) wpp = 10;           // more tiles than threads: the kernel loops over tiles
    nstage = 2;
  }
};

__device__ __forceinline__ void k1_issue(const KernelParams& p, float2* Hs, float2* Ys,
                                         uint64_t* bar, long sc, int UP) {
  const uint32_t hbytes = static_cast<uint32_t>(p.B) * UP * 8u;
  // use_tma == 2 (odd S): Y rows are padded in shared memory, loaded by threads
  const uint32_t ybytes = p.use_tma == 1 ? static_cast<uint32_t>(p.B) * p.S * 8u : 0u;
  fence_proxy_async();
  mbar_expect_tx(bar, hbytes + ybytes);
  bulk_g2s(Hs, p.H + sc * static_cast<long>(p.B) * UP, hbytes, bar);
  if (p.S > 0 && ybytes) bulk_g2s(Ys, p.Y + sc * static_cast<long>(p.B) * p.S, ybytes, bar);
}

// MINB: CTAs per SM the register budget is sized for; PIPE: software-
// pipelined tile loop (operands of row k+1 in flight) or the plain one.
template <int UP, bool EXACT, int MINB = 2, bool PIPE = true>
__global__ void __launch_bounds__(320, MINB) channel_kernel(const KernelParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int spl = p.k1_spl, nstage = p.k1_pair;
  K1Smem<UP> L;
  L.plan(p.B, p.S, nstage);
  WsOffsets W;
  W.plan(UP, p.S, p.K, EXACT, p.fx, p.zs);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  const int nt = blockDim.x;
  const int tid = threadIdx.x;
  const int B = p.B, S = p.S, U = p.U;
  const int nb = UP / 4, n_gram = nb * (nb + 1) / 2, nsb = (S + 3) / 4;
  const int n_tiles = n_gram + nb * nsb;
  auto Hs_of = [&](int st) { return reinterpret_cast<float2*>(smem + L.hs + st * L.slot); };
  auto Ys_of = [&](int st) {
    return reinterpret_cast<float2*>(smem + L.hs + st * L.slot + L.ys);
  };

  uint8_t* tile_ib = reinterpret_cast<uint8_t*>(smem + L.lut);
  uint8_t* tile_jb = tile_ib + 512;
  for (int t = tid; t < n_tiles; t += nt) {
    int a, b;
    if (t < n_gram) {
      tri_block(t, a, b);
    } else {
      b = (t - n_gram) / nb;
      a = (t - n_gram) - b * nb;
    }
    tile_ib[t] = static_cast<uint8_t>(a);
    tile_jb[t] = static_cast<uint8_t>(b);
  }
  const int n_items = spl * n_tiles;
  const int part = tid / n_tiles;
  const int tile = tid - part * n_tiles;
  const bool active = tid < n_items;
  const bool is_gram = tile < n_gram;
  int ib = 0, jb = 0;
  if (is_gram) {
    tri_block(tile, ib, jb);  // row-major: neighbouring lanes share X
  } else {
    const int m = tile - n_gram;  // neighbouring lanes share the Y block
    jb = m / nb;
    ib = m - jb * nb;
  }
  const int kchunk = (B + spl - 1) / spl;
  const int k0 = part * kchunk, k1 = min(B, k0 + kchunk);
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto sc_of = [&](long i) { return p.sc_base + blockIdx.x + i * gridDim.x; };

  if (tid == 0 && p.use_tma) {
    for (int st = 0; st < nstage; ++st) mbar_init(bars + st, 1);
  }
  __syncthreads();
  if (tid == 0 && p.use_tma)
    for (int st = 0; st < nstage && st < n_local; ++st) k1_issue(p, Hs_of(st), Ys_of(st), bars + st, sc_of(st), UP);

  for (long i = 0; i < n_local; ++i) {
    const int st = static_cast<int>(i % nstage);
    const uint32_t ph = static_cast<uint32_t>((i / nstage) & 1);
    const long lsc = blockIdx.x + i * gridDim.x;  // within the chunk
    const long sc = p.sc_base + lsc;
    float2* Hs = Hs_of(st);
    float2* Ys = Ys_of(st);
    float2* ws = p.ws + lsc * W.stride;
    // ------------------------------------------------------ stage H, Y
    const int Sp = (S + 1) & ~1;
    if (p.use_tma) {
      if (p.use_tma == 2) {  // H by bulk copy, the (padded) Y rows by the threads
        for (int e = tid; e < Sp * B; e += nt) {
          const int b = e / Sp, s = e - b * Sp;
          Ys[e] = s < S ? p.Y[(sc * B + b) * static_cast<long>(S) + s] : make_float2(0.f, 0.f);
        }
      }
      mbar_wait(bars + st, ph);
      if (p.use_tma == 2) __syncthreads();
    } else {
      if (p.hd_layout) {
        // downlink H_d [U][B] -> Hs[b][u] = conj(H_d[u][b])  (= H_u = H_d^H)
        const float2* src = p.H + sc * static_cast<long>(U) * B;
        for (int e = tid; e < UP * B; e += nt) {
          const int u = e / B, b = e - u * B;
          Hs[b * UP + u] = u < U ? cconj(src[u * B + b]) : make_float2(0.f, 0.f);
        }
      } else {
        const float2* src = p.H + sc * static_cast<long>(B) * U;
        for (int e = tid; e < UP * B; e += nt) {
          const int b = e / UP, u = e - b * UP;
          Hs[e] = u < U ? src[b * U + u] : make_float2(0.f, 0.f);
        }
      }
      for (int e = tid; e < Sp * B; e += nt) {
        const int b = e / Sp, s = e - b * Sp;
        Ys[e] = s < S ? p.Y[(sc * B + b) * static_cast<long>(S) + s] : make_float2(0.f, 0.f);
      }
      __syncthreads();
    }
    // --------------------------------------- Gram + matched-filter tiles
    float2* MFw = ws + W.mf;
    // results of tile t, row r: G (one triangle + conjugate mirror, G == G^H
    // exactly) or the matched filter
    auto write_row = [&](int t, int r, const float2 (&v)[4]) {
      const int tib = tile_ib[t], tjb = tile_jb[t];
      if (t < n_gram) {
        const int ii = tib * 4 + r;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = tjb * 4 + c;
          if (j < ii) {
            Gs[ii * UP + j] = v[c];
            Gs[j * UP + ii] = cconj(v[c]);
          } else if (j == ii) {
            Gs[ii * UP + ii] = make_float2(v[c].x, 0.f);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int s_ = tjb * 4 + c;
          if (s_ < S) MFw[s_ * UP + tib * 4 + r] = v[c];
        }
      }
    };
    if (n_items > nt) {
      // more tiles than threads (U = 64 with many vectors; spl == 1): each
      // thread loops over whole tiles and writes its results directly
      for (int t = tid; t < n_tiles; t += nt) {
        float2 acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
        const bool g = t < n_gram;
        tile4x4_pipe(acc, Hs, UP, tile_ib[t] * 4, g ? Hs : Ys, g ? UP : Sp, tile_jb[t] * 4, 0, B);
#pragma unroll
        for (int r = 0; r < 4; ++r) write_row(t, r, acc[r]);
      }
    } else {
      // one branch-free loop for both tile kinds (a warp may hold both): the
      // second operand is H itself (Gram) or the Y block (matched filter)
      float2 acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);
      if (active) {
        const float2* Z = is_gram ? Hs : Ys;
        const int ldz = is_gram ? UP : Sp;
        if (PIPE)
          tile4x4_pipe(acc, Hs, UP, ib * 4, Z, ldz, jb * 4, k0, k1);
        else
          tile4x4<true>(acc, Hs, UP, ib * 4, Z, ldz, 1, jb * 4, 1 << 30, k0, k1);
      }
      __syncthreads();  // (A) every k loop done: the stage may hold partials
      {
        // partials parked entry-major / tile-minor ([part][16][n_tiles]) so a
        // warp's stores and the reduction's loads are contiguous (no conflicts)
        float2* pb = Hs;
        if (active) {
          float2* dst = pb + part * 16 * n_tiles + tile;
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[(r * 4 + c) * n_tiles] = acc[r][c];
        }
        __syncthreads();  // (B)
        // thread <-> (tile, row r): fixed-order sum of the k-parts for the 4
        // entries of the row, then G (one triangle + conjugate mirror, G == G^H
        // exactly) or the matched filter.  Loads are tile-contiguous.
        for (int e = tid; e < n_tiles * 4; e += nt) {
          const int r = e / n_tiles, t = e - r * n_tiles;
          float2 v[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            v[c] = pb[(r * 4 + c) * n_tiles + t];
            for (int sp = 1; sp < spl; ++sp) v[c] = cadd(v[c], pb[(sp * 16 + r * 4 + c) * n_tiles + t]);
          }
          write_row(t, r, v);
        }
      }
    }
    __syncthreads();  // (C) stage consumed, G complete
    if (tid == 0 && p.use_tma && i + nstage < n_local)
      k1_issue(p, Hs, Ys, bars + st, sc_of(i + nstage), UP);  // prefetch into the freed stage
    {  // G -> workspace (coalesced)
      const float4* src = reinterpret_cast<const float4*>(Gs);
      float4* dst = reinterpret_cast<float4*>(ws + W.g);
      for (int e = tid; e < UP * UP / 2; e += nt) dst[e] = src[e];
    }
    __syncthreads();  // Gs is rewritten by the next subcarrier
  }
}

// ------------------------------------------------------------------- K2
template <int UP, int NSO = 0>
struct K2Geo {
  static constexpr int G = UP < 32 ? UP : 32;  // lanes per system
  static constexpr int RU = UP / G;            // rows per lane
  static constexpr int GPW = 32 / G;           // groups per warp
  static constexpr int NS = NSO > 0 ? NSO : (UP == 32 ? 2 : 1);  // systems per group, interleaved
};

template <int UP>
struct K2Smem {
  int gs, ps, vs, qs, hist, msh, sys_st, gpart, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int B, int S, int St, int K, bool exact) {
    const int nsys = S + St;
    int o = 0;
    gs = o; o = align(o + UP * UP * 8);
    ps = o; o = align(o + nsys * UP * 8);
    vs = o; o = align(o + nsys * UP * 8);
    qs = o; o = align(o + St * B * 8);
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    msh = o; o = align(o + (exact ? 8 * kMomScratch * 8 : 0));  // per-warp extraction scratch
    sys_st = o; o = align(o + nsys);
    gpart = o; o = align(o + ((B + 31) / 32) * (St > 0 ? St : 1) * 4);
    total = o;
  }
};

// ---------------------------------------------------------- solve tails
// Shared by the CTA-per-subcarrier solve kernels, after the CG: Vs[sys][u]
// holds v, sys_st the breakdown flags (the exact tracker's tail is
// moments_tail, cgm_moments.cuh).
// Precoder (precode.cpp:22-71): q = H_d^H v, gain = ||q||, s = q / gain.
template <int UP, class Sync>
__device__ __forceinline__ void k2_precode_tail(const KernelParams& p, long sc, const float2* Vs,
                                                float2* Qs, float* gpart, const uint8_t* sys_st,
                                                int nt, Sync&& sync) {
  const int nw = nt >> 5, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = p.S, St = p.St, B = p.B, U = p.U;
  // ------------------------------------------------ precode q = H_d^H v
  // q_b = sum_u H_u[b][u] v_u = sum_u conj(H_d[u][b]) v_u (precode.cpp:69),
  // then gain = ||q||, s = q / gain, zero_input when ||q|| vanishes (:22-36)
    const int nrb = (B + 31) / 32;
    for (int rb = warp; rb < nrb; rb += nw) {
      const int bidx = rb * 32 + lane;
      const bool okb = bidx < B;
      const int bb = okb ? bidx : 0;
      for (int ts0 = 0; ts0 < St; ts0 += 8) {
        float2 acc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = make_float2(0.f, 0.f);
        if (p.hd_layout) {
          const float2* hd = p.H + sc * static_cast<long>(U) * B;  // [U][B], coalesced in b
          for (int u = 0; u < U; ++u) {
            const float2 h = cconj(__ldg(hd + u * B + bb));
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (ts0 + t < St) cfma(acc[t], h, Vs[(S + ts0 + t) * UP + u]);
          }
        } else if (U != UP) {
          const float2* hu = p.H + (sc * static_cast<long>(B) + bb) * U;  // row b of H_u
          for (int u = 0; u < U; ++u) {
            const float2 h = __ldg(hu + u);
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (ts0 + t < St) cfma(acc[t], h, Vs[(S + ts0 + t) * UP + u]);
          }
        } else {
          const float2* hu = p.H + sc * static_cast<long>(B) * UP + bb * UP;  // row b of H_u
#pragma unroll 8
          for (int u = 0; u < UP; u += 2) {
            const float4 h = __ldg(reinterpret_cast<const float4*>(hu + u));
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (ts0 + t < St) {
                const float4 vv = *reinterpret_cast<const float4*>(Vs + (S + ts0 + t) * UP + u);
                cfma(acc[t], make_float2(h.x, h.y), make_float2(vv.x, vv.y));
                cfma(acc[t], make_float2(h.z, h.w), make_float2(vv.z, vv.w));
              }
            }
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (ts0 + t < St) {
            if (okb) Qs[(ts0 + t) * B + bidx] = acc[t];
            float nrm = okb ? cnorm(acc[t]) : 0.f;
            nrm = group_sum<32>(nrm);
            if (lane == 0) gpart[rb * St + ts0 + t] = nrm;
          }
        }
      }
    }
    sync();
    for (int ts = warp; ts < St; ts += nw) {
      const int sysi = S + ts;
      const bool ok = sys_st[sysi] == 0;
      float nrm = 0.f;
      for (int rb = 0; rb < nrb; ++rb) nrm += gpart[rb * St + ts];  // fixed order
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

// GREG: row u of G held in registers for the whole subcarrier (U = 32, one
// system per lane group at a time); p_j is read in 8-column chunks so the
// loads of a chunk are in flight together, with 4 independent FMA chains.
// The whole per-subcarrier solve (CG, trackers, LLRs, precoder) for one
// subcarrier `lsc` of the chunk, run by threads [0, nt) (warps 0..nt/32-1)
// with `sync` a barrier over exactly those; smem holds the K2Smem plan.
// Called by solve_kernel (one CTA per subcarrier) and, fused, by the
// epilogue warps of channel_tc_kernel.
template <int UP, bool EXACT, int NSO = 0, bool GREG = false, class Sync>
__device__ __forceinline__ void solve_sc(const KernelParams& p, long lsc, unsigned char* smem,
                                         int nt, Sync&& sync, const float2* pre = nullptr) {
  using GE = K2Geo<UP, NSO>;
  static_assert(!GREG || (UP == 32 && GE::NS == 1), "GREG needs U = 32, one system per warp");
  constexpr int G = GE::G, RU = GE::RU, GPW = GE::GPW, NS = GE::NS;
  const int S = p.S, St = p.St, B = p.B, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  K2Smem<UP> L;
  L.plan(B, S, St, Kmax, EXACT);
  WsOffsets W;
  W.plan(UP, S, p.K, EXACT, p.fx, p.zs);
  // G (and the matched filters) from the prefetched shared-memory copy of
  // the workspace when the persistent kernel staged one
  const float2* Gs = pre ? pre + W.g : reinterpret_cast<float2*>(smem + L.gs);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float2* Qs = reinterpret_cast<float2*>(smem + L.qs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  float* gpart = reinterpret_cast<float*>(smem + L.gpart);
  const int nw = nt >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long sc = p.sc_base + lsc;
  const float2* ws = p.ws + lsc * W.stride;

  const float2* mfsrc = pre ? pre + W.mf : ws + W.mf;
  if (!pre) {  // G <- workspace
    const float4* src = reinterpret_cast<const float4*>(ws + W.g);
    float4* dst = reinterpret_cast<float4*>(smem + L.gs);
    for (int e = tid; e < UP * UP / 2; e += nt) dst[e] = src[e];
    sync();
  }

  // ------------------------------------------------------------------ CG
  {
    const int grp = lane / G, gl = lane - grp * G;
    const int n_slots = nw * GPW * NS;
    float gdiag[RU];
#pragma unroll
    for (int m = 0; m < RU; ++m) gdiag[m] = Gs[(gl + m * G) * UP + gl + m * G].x;
    float2 grow[GREG ? UP : 1];
    if constexpr (GREG) {
#pragma unroll
      for (int j = 0; j < UP; ++j) grow[j] = cconj(Gs[j * UP + gl]);  // G[u][j]
    }
    // warp-uniform trip count (the shuffles below use the full mask)
    for (int wbase = warp * GPW * NS; wbase < nsys; wbase += n_slots) {
      const int base = wbase + grp * NS;
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
#pragma unroll
        for (int m = 0; m < RU; ++m) {
          const int u = gl + m * G;
          float2 b = make_float2(0.f, 0.f);
          if (live[s] && u < U)
            b = down[s] ? p.T[(sc * St + (sys[s] - S)) * static_cast<long>(U) + u]
                        : mfsrc[sys[s] * UP + u];
          v[s][m] = make_float2(0.f, 0.f);
          r[s][m] = b;
          pp[s][m] = b;
          if (live[s]) Ps[sys[s] * UP + u] = b;
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
      }
      __syncwarp();
      for (int k = 1; k <= Kmax; ++k) {
        // e = (G + reg I) p: G read as column (conflict-free), p broadcast;
        // two partial sums per component shorten the FMA chains
        float2 e[NS][RU], e2[NS][RU];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int m = 0; m < RU; ++m) e[s][m] = e2[s][m] = make_float2(0.f, 0.f);
        if constexpr (GREG) {
          const float4* prow = reinterpret_cast<const float4*>(Ps + (live[0] ? sys[0] : 0) * UP);
          float2 e3 = make_float2(0.f, 0.f), e4 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j0 = 0; j0 < UP; j0 += 8) {
            float4 pj[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pj[q] = prow[j0 / 2 + q];
            cfma(e[0][0], grow[j0 + 0], make_float2(pj[0].x, pj[0].y));
            cfma(e2[0][0], grow[j0 + 1], make_float2(pj[0].z, pj[0].w));
            cfma(e3, grow[j0 + 2], make_float2(pj[1].x, pj[1].y));
            cfma(e4, grow[j0 + 3], make_float2(pj[1].z, pj[1].w));
            cfma(e[0][0], grow[j0 + 4], make_float2(pj[2].x, pj[2].y));
            cfma(e2[0][0], grow[j0 + 5], make_float2(pj[2].z, pj[2].w));
            cfma(e3, grow[j0 + 6], make_float2(pj[3].x, pj[3].y));
            cfma(e4, grow[j0 + 7], make_float2(pj[3].z, pj[3].w));
          }
          e[0][0] = cadd(e[0][0], e3);
          e2[0][0] = cadd(e2[0][0], e4);
        } else {
#pragma unroll 4
        for (int j = 0; j < UP; j += 2) {
          float2 g0[RU], g1[RU];
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            g0[m] = cconj(Gs[j * UP + gl + m * G]);
            g1[m] = cconj(Gs[(j + 1) * UP + gl + m * G]);
          }
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int row = live[s] ? sys[s] : 0;
            const float4 pj = *reinterpret_cast<const float4*>(Ps + row * UP + j);
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              cfma(e[s][m], g0[m], make_float2(pj.x, pj.y));
              cfma(e2[s][m], g1[m], make_float2(pj.z, pj.w));
            }
          }
        }
        }
        float curv[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          curv[s] = 0.f;
#pragma unroll
          for (int m = 0; m < RU; ++m) {
            e[s][m] = cadd(e[s][m], e2[s][m]);
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
          alpha[s] = upd[s] ? __fdividef(rn[s], curv[s]) : 1.f;
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
            beta[s] = __fdividef(rnx[s], rn[s]);
            rn[s] = rnx[s];
#pragma unroll
            for (int m = 0; m < RU; ++m) {
              pp[s][m].x = fmaf(beta[s], pp[s][m].x, r[s][m].x);
              pp[s][m].y = fmaf(beta[s], pp[s][m].y, r[s][m].y);
              Ps[sys[s] * UP + gl + m * G] = pp[s][m];
            }
          }
          if (k <= iters[s]) {
            if (!down[s]) {
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
                    const float c1 = __fdividef(alpha[s] * (1.f + bm1[s]), am1[s]);
                    const float c2 = __fdividef(alpha[s] * bm2[s], am2[s]);
                    nf = f0[s][m] + (c1 - alpha[s] * (gdiag[m] + reg[s])) * (f0[s][m] - f1[s][m]) -
                         c2 * (f1[s][m] - f2[s][m]);
                  }
                  f2[s][m] = f1[s][m];
                  f1[s][m] = f0[s][m];
                  f0[s][m] = nf;
                }
              }
            }
            am2[s] = am1[s]; am1[s] = alpha[s];
            bm2[s] = bm1[s]; bm1[s] = beta[s];
          }
        }
        __syncwarp();
      }
      // ------------------------------------------------ per-system epilogue
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (!live[s]) continue;
        if (gl == 0) sys_st[sys[s]] = broke[s] ? 1 : 0;
        if (EXACT || down[s]) {
#pragma unroll
          for (int m = 0; m < RU; ++m) Vs[sys[s] * UP + gl + m * G] = v[s][m];
          continue;
        }
        // approx uplink: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441),
        // LLRs and stores straight from the lane
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
          if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
          if (p.status && gl == 0) p.status[sc * S + sys[s]] = ok ? 0 : 1;
        }
      }
    }
  }

  // ------------------------------------------ exact tracker extraction
  if (EXACT && S > 0 && p.fx) {  // moments_kernel<..., FX> finishes from the workspace
    sync();
    fx_handoff<UP>(p, const_cast<float2*>(ws), W, sc, hist, Kmax, Vs, sys_st[0], tid, nt);
  } else if (EXACT && S > 0) {
    sync();
    moments_tail<UP>(p, ws, W, sc, Kmax, hist, Vs, sys_st, nt,
                     reinterpret_cast<double*>(smem + L.msh));
  }
  // ------------------------------------------------ precode q = H_d^H v
  if (St > 0) {
    sync();
    k2_precode_tail<UP>(p, sc, Vs, Qs, gpart, sys_st, nt, sync);
  }
}

template <int UP, bool EXACT, int MINB = 3, int NSO = 0, bool GREG = false>
__global__ void __launch_bounds__(256, MINB) solve_kernel(const KernelParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  solve_sc<UP, EXACT, NSO, GREG>(p, blockIdx.x, smem, blockDim.x, [] { __syncthreads(); });
}

// Persistent variant: each CTA walks subcarriers blockIdx.x, +gridDim.x, ...
// and bulk-copies the next one's G + matched filters (one contiguous
// workspace span) into a second shared-memory buffer while solving the
// current one, so the per-subcarrier load latency leaves the critical path.
__host__ __device__ inline int k2_pre_bytes(int UP, int S) {
  return ((UP * UP + S * UP + 2) * 8 + 127) & ~127;
}

template <int UP, bool EXACT, int MINB = 3>
__global__ void __launch_bounds__(256, MINB) solve_kernel_pf(const KernelParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  WsOffsets W;
  W.plan(UP, p.S, p.K, EXACT, p.fx, p.zs);
  const int pb = k2_pre_bytes(UP, p.S);
  const uint32_t bytes = static_cast<uint32_t>(W.cd * 8);  // G + MF
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  float2* buf[2] = {reinterpret_cast<float2*>(smem + 128), reinterpret_cast<float2*>(smem + 128 + pb)};
  unsigned char* rest = smem + 128 + 2 * pb;
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  auto issue = [&](long i) {
    const long lsc = blockIdx.x + i * gridDim.x;
    fence_proxy_async();  // generic reads of this buffer (two uses ago) before the async write
    mbar_expect_tx(bar + (i & 1), bytes);
    bulk_g2s(buf[i & 1], p.ws + lsc * W.stride, bytes, bar + (i & 1));
  };
  if (threadIdx.x == 0 && n_local > 0) issue(0);
  for (long i = 0; i < n_local; ++i) {
    if (threadIdx.x == 0 && i + 1 < n_local) issue(i + 1);
    mbar_wait(bar + (i & 1), static_cast<uint32_t>((i >> 1) & 1));
    solve_sc<UP, EXACT>(p, blockIdx.x + i * gridDim.x, rest, blockDim.x, [] { __syncthreads(); },
                        buf[i & 1]);
    __syncthreads();
  }
}

}  // namespace cgm
