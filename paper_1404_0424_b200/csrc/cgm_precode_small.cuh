// cgm_precode_small.cuh -- fused CG precoder for small U (U <= 16), H_d in
// the reference layout [U][B] (precode_cg, precode.cpp:56-71).
//
// One WARP per subcarrier, persistent over subcarriers, no block-level
// barriers (a CTA-wide version spent a quarter of its warp time waiting at
// the barrier behind the one warp running the latency-bound CG).  The
// channel never sits in shared memory as a whole: it STREAMS through a
// two-slot ring of 64-antenna chunks (16-byte cp.async, lane = antenna pair,
// one warp instruction per user row, one commit group per chunk), twice per
// subcarrier -- once for the Gram (from HBM) and once per transmit vector
// for q (from L2, the same SM read it microseconds ago) -- so the next
// chunks, including the next subcarrier's first two, load while the warp
// computes and no warp ever waits on its own load.  Per subcarrier:
//   1. A_d = H_d H_d^H (downlink_gram, precode.cpp:38-41): lower 4 x 4 tiles
//      x KP antenna ranges of every chunk on the FFMA2 pipe, accumulators in
//      registers across the chunks, partials summed in a fixed order
//      (G == G^H exactly: one triangle + conjugate mirror, real diagonal);
//   2. K CG iterations on A_d + rho_d^-1 I for every transmit vector t
//      (solvers.cpp:37-72, same freeze / breakdown rules as K2): the whole
//      warp on one system, the 32 / UP lane groups splitting the columns of
//      the matvec (partial sums combined by xor shuffles), warp-shuffle
//      reductions;
//   3. q = H_d^H v chunk by chunk (lane = antenna), gain = ||q|| (fixed
//      butterfly order), s = q / gain, zero_input (precode.cpp:22-36).
#pragma once

#include "cgm_rows32.cuh"  // f2dup_lo / f2dup_hi

#ifndef CGM_PS_CB
#define CGM_PS_CB 64
#endif

namespace cgm {

template <int UP>
struct PrecodeSmallGeo {
  static constexpr int NT = 32;            // one warp per CTA
  static constexpr int NB = UP / 4;
  static constexpr int NTILE = NB * (NB + 1) / 2;
  static constexpr int GL = UP;            // lanes per row group
  static constexpr int GPW = 32 / GL;      // column groups of the CG matvec
  static constexpr int KP = 32 / NTILE;    // antenna ranges per tile (3 / 10)
  static constexpr int CB = CGM_PS_CB;     // antennas per staged chunk
};

struct PrecodeSmallSmem {
  static constexpr int CB = CGM_PS_CB, LDH = CB + 2;  // padded row: consecutive rows 16 B apart in the banks
  static constexpr int LDP = 17;               // partials: [lane][16 entries + 1]
  static constexpr int H = 0;                  // the two ring slots come first
  int hb, gs, ps, vs, st, part, total;
  __host__ __device__ static int align(int x) { return (x + 15) & ~15; }
  __host__ __device__ void plan(int UP, int B, int St) {
    (void)B;
    hb = UP * LDH * 8;  // bytes per ring slot
    int o = H + 2 * hb;
    gs = o; o = align(o + UP * UP * 8);
    ps = o; o = align(o + UP * 8);
    vs = o; o = align(o + (St > 0 ? St : 1) * UP * 8);
    st = o; o = align(o + (St > 0 ? St : 1));
    part = o; o = align(o + (UP <= 8 ? 32 * LDP * 8 : 0));  // U > 8 sums its 3 parts by shuffles
    total = o;
  }
};

// MQ = chunks per antenna pass held in registers (B <= 32 MQ): 4 for B <= 128
// (16 warps per SM), 16 up to B = 512.
// Launch bound = the warps per SM that shared memory allows: 11 for U = 16
// (19.2 KB per warp; a bound of 15 capped the kernel at 128 registers with
// spills, 11 gives 167 and none at the same occupancy), 15 for U <= 8.
template <int UP, int MQ>
__global__ void __launch_bounds__(32, MQ > 4 ? 10 : UP == 16 ? 11 : 15) precode_small_kernel(const KernelParams p) {
  using PG = PrecodeSmallGeo<UP>;
  constexpr int GL = PG::GL, GPW = PG::GPW, KP = PG::KP, CB = PG::CB;
  constexpr int LDH = PrecodeSmallSmem::LDH, LDP = PrecodeSmallSmem::LDP;
  constexpr int HB = UP * LDH * 8;  // bytes per ring slot
  static_assert(CB == 64 || CB == 32, "a warp instruction copies 32 antenna pairs: 1 or 2 rows");
  constexpr int PR = CB / 2, RPI = 32 / PR;  // pairs per row, rows per copy instruction
  extern __shared__ __align__(128) unsigned char smem[];
  const int B = p.B, U = p.U, St = p.St;
  PrecodeSmallSmem L;
  L.plan(UP, B, St);
  float2* P = reinterpret_cast<float2*>(smem + L.part);
  float2* Gs = reinterpret_cast<float2*>(smem + L.gs);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.st);
  const int lane = threadIdx.x;
  const bool tma = p.use_tma != 0;
  unsigned char* ring = smem + PrecodeSmallSmem::H;
  auto slot = [&](unsigned j) { return reinterpret_cast<float2*>(ring + (j & 1u) * HB); };
  const int cp_r = lane / PR, cp_p = lane - cp_r * PR;  // this lane's row (of RPI) and antenna pair
  const uint32_t row0 = smem_u32(ring) + cp_r * (LDH * 8) + cp_p * 16;  // ... in slot 0

  if (U < UP)  // padded rows of both slots stay zero for the whole kernel
    for (int e = lane; e < 2 * (UP - U) * LDH; e += 32) {
      const int s = e / ((UP - U) * LDH), r = e - s * (UP - U) * LDH;
      slot(s)[U * LDH + r] = make_float2(0.f, 0.f);
    }
  __syncwarp();

  // chunk jobs: per subcarrier nchunk Gram chunks, then nchunk chunks per
  // transmit vector; job j lives in slot j & 1.  Every lane copies its
  // antenna pair of each user row with a 16-byte cp.async (one warp
  // instruction per row -- a per-lane cp.async.bulk is serialised lane by
  // lane through the uniform datapath, ~20 instructions per row), one commit
  // group per job, so "job j landed" is wait_group<1> after job j + 1 (or
  // an empty group) was committed.
  const int nchunk = (B + CB - 1) / CB;
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const unsigned n_jobs = static_cast<unsigned>(n_local) * static_cast<unsigned>(nchunk * (1 + St));
  const long sc_step = static_cast<long>(gridDim.x) * U * B;  // float2 between this warp's subcarriers
  unsigned nj = 0;             // next job to issue
  int nj_c = 0, nj_pass = 0;   // its chunk and pass (0 = Gram)
  const float2* nj_row = p.H + (static_cast<long>(blockIdx.x) * U + cp_r) * B + 2 * cp_p;  // its subcarrier
  auto issue = [&]() {  // after a __syncwarp that follows every read of the slot
    if (nj < n_jobs) {
      const int c0 = nj_c * CB, nb = B - c0 < CB ? B - c0 : CB;
      if (2 * cp_p < nb) {
        uint32_t dst = row0 + (nj & 1u) * HB;
        const float2* src = nj_row + c0;
        if (RPI == 1 && B == 128 && U == UP) {
          // cfg3's shape: constant row strides, every copy is
          // [pointer + immediate] (no per-row address arithmetic)
#pragma unroll
          for (int u = 0; u < UP; ++u)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + u * (LDH * 8)),
                         "l"(src + u * 128)
                         : "memory");
        } else
#pragma unroll 4
        for (int u = cp_r; u < U; u += RPI) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          dst += RPI * LDH * 8;
          src += RPI * B;
        }
      }
      ++nj;
      if (++nj_c == nchunk) {
        nj_c = 0;
        if (++nj_pass == 1 + St) {
          nj_pass = 0;
          nj_row += sc_step;
        }
      }
    }
    cp_async_commit();  // also when nothing is left: keeps one group per job slot
  };
  unsigned cj = 0;  // job being consumed
  // slot of job cj ready; returns its antenna count
  auto acquire = [&](long sc, int c) {
    const int c0 = c * CB, nb = B - c0 < CB ? B - c0 : CB;
    if (tma) {
      cp_async_wait<1>();
      __syncwarp();  // every lane's copies of the job are visible to the warp
    } else {
      float2* dst = slot(cj);
      for (int e = lane; e < U * nb; e += 32) {
        const int u = e / nb, b = e - u * nb;
        dst[u * LDH + b] = p.H[(sc * U + u) * static_cast<long>(B) + c0 + b];
      }
      __syncwarp();
    }
    return nb;
  };
  auto release = [&]() {  // every lane is done with the slot of job cj
    __syncwarp();
    ++cj;
    if (tma) issue();
  };
  if (tma) {
    issue();
    issue();
  }

  // Gram work item: lower tile (rb, cb) x antenna-pair range of the chunk,
  // visited from a per-tile rotated start (bank spread)
  const int item_part = lane / PG::NTILE, item_tile = lane - item_part * PG::NTILE;
  const bool gram_busy = item_part < KP;
  int rb = 0;
  while ((rb + 1) * (rb + 2) / 2 <= item_tile) ++rb;
  const int cb = item_tile - rb * (rb + 1) / 2;
  const int grp = lane / GL, gl = lane - grp * GL;
  // a full chunk's pair range and rotated start (the tail chunk recomputes)
  constexpr int NPF = CB / 2;
  const int fq0 = (item_part * NPF) / KP, fnq = ((item_part + 1) * NPF) / KP - fq0;
  // the rotated start spreads a quarter-warp's LDS.128 over the eight 16-byte
  // bank groups; for U = 16 and 64-antenna chunks a searched table makes
  // the x / y loads of a full chunk nearly conflict-free (tools/ps_rotation.py:
  // 96 wavefronts per chunk, 88 = none, instead of 178 with tile mod range)
  int fst = fnq > 0 ? item_tile % fnq : 0;
  if constexpr (UP == 16 && CB == 64) {
    constexpr unsigned char kRot[32] = {2, 2, 2, 1, 0, 0, 1, 1, 0, 0, 7, 1, 1, 1, 1, 0,
                                        10, 5, 5, 10, 5, 5, 5, 10, 0, 0, 6, 1, 0, 5, 0, 0};
    fst = kRot[lane];
  }

  for (long it = 0; it < n_local; ++it) {
    const long sc = blockIdx.x + it * gridDim.x;
    // the first transmit vector, loaded now so the latency hides under the Gram
    float2 t_first = make_float2(0.f, 0.f);
    if (St > 0 && gl < U) t_first = p.T[(sc * St) * static_cast<long>(U) + gl];
    // ------------------------------------------ 1. A_d = H_d H_d^H partials
    {
      // packed FFMA2: a += x (pair) * y.x, b += x (pair) * y.y;
      // x conj(y) = (a.x + b.y, a.y - b.x)
      unsigned long long a[4][4], bb[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[r][c] = bb[r][c] = 0ull;
      for (int ch = 0; ch < nchunk; ++ch) {
        const int nb = acquire(sc, ch);
        if (gram_busy) {
          const float2* Hb = slot(cj);
          const float2* hu = Hb + (rb * 4) * LDH;
          const float2* hv = Hb + (cb * 4) * LDH;
          int q0 = fq0, nq = fnq, q = fst;
          if (nb != CB) {
            const int np = nb >> 1;
            q0 = (item_part * np) / KP;
            nq = ((item_part + 1) * np) / KP - q0;
            q = nq > 0 ? item_tile % nq : 0;
          }
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
        }
        release();
      }
      // part sums in a fixed order (part 0 + part 1 + ...), lower entries,
      // exact Hermitian mirror.  Few parts (U > 8): the tile's part lanes sit
      // NTILE apart, so the tile's first lane pulls them in by shuffles and
      // writes the tile; many parts (U <= 8): through shared memory.
      if constexpr (KP <= 4) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 A2 = f2unpack(a[r][c]), B2 = f2unpack(bb[r][c]);
            const float2 x = make_float2(A2.x + B2.y, A2.y - B2.x);
            float2 g = x;
#pragma unroll
            for (int k = 1; k < KP; ++k) {
              g.x += __shfl_down_sync(0xffffffffu, x.x, k * PG::NTILE);
              g.y += __shfl_down_sync(0xffffffffu, x.y, k * PG::NTILE);
            }
            const int u = rb * 4 + r, v = cb * 4 + c;
            if (lane < PG::NTILE && v <= u) {
              if (u == v) {
                Gs[u * UP + u] = make_float2(g.x, 0.f);
              } else {
                Gs[u * UP + v] = g;
                Gs[v * UP + u] = cconj(g);
              }
            }
          }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 A2 = f2unpack(a[r][c]), B2 = f2unpack(bb[r][c]);
            P[lane * LDP + r * 4 + c] = make_float2(A2.x + B2.y, A2.y - B2.x);
          }
        __syncwarp();
        for (int e = lane; e < PG::NTILE * 16; e += 32) {
          const int t = e >> 4, rc = e & 15;
          int trb = 0;
          while ((trb + 1) * (trb + 2) / 2 <= t) ++trb;
          const int u = trb * 4 + (rc >> 2), v = (t - trb * (trb + 1) / 2) * 4 + (rc & 3);
          if (v > u) continue;
          float2 g = P[t * LDP + rc];
#pragma unroll
          for (int k = 1; k < KP; ++k) g = cadd(g, P[(k * PG::NTILE + t) * LDP + rc]);
          if (u == v) {
            Gs[u * UP + u] = make_float2(g.x, 0.f);
          } else {
            Gs[u * UP + v] = g;
            Gs[v * UP + u] = cconj(g);
          }
        }
      }
    }
    __syncwarp();
    // ------------------------------------------------------- 2. CG per t
    // every lane group holds the system's (v, r, p) for row gl and sums the
    // columns [grp * UP / GPW, (grp + 1) * UP / GPW) of the matvec
    for (int sys = 0; sys < St; ++sys) {
      float2 b = make_float2(0.f, 0.f);
      if (gl < U) b = sys == 0 ? t_first : p.T[(sc * St + sys) * static_cast<long>(U) + gl];
      float2 v = make_float2(0.f, 0.f), r = b, pp = b;
      if (grp == 0) Ps[gl] = b;
      float rn = group_sum<GL>(cnorm(b));
      const float rn0 = rn;
      bool broke = false;
      __syncwarp();
      for (int k = 1; k <= p.Kt; ++k) {
        constexpr int NC = UP / GPW;  // columns per group
        float2 e = make_float2(0.f, 0.f), e2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int jj = 0; jj < NC; jj += 2) {
          const int j = grp * NC + jj;
          cfma_conj(e, Gs[j * UP + gl], Ps[j]);  // G[gl][j] = conj(G[j][gl])
          cfma_conj(e2, Gs[(j + 1) * UP + gl], Ps[j + 1]);
        }
        e = cadd(e, e2);
#pragma unroll
        for (int o = GL; o < 32; o <<= 1) {  // the groups' column parts, fixed order
          e.x += __shfl_xor_sync(0xffffffffu, e.x, o);
          e.y += __shfl_xor_sync(0xffffffffu, e.y, o);
        }
        e.x = fmaf(p.rho_inv_d, pp.x, e.x);
        e.y = fmaf(p.rho_inv_d, pp.y, e.y);
        const float curv = group_sum<GL>(pp.x * e.x + pp.y * e.y);
        const bool frozen = !(rn > 1e-28f * rn0);  // solvers.cpp:21,25-27
        const bool go = !frozen && !broke;
        if (go && curv < 1e-30f) broke = true;     // solvers.cpp:55-57
        const bool upd = go && !broke;
        const float alpha = upd ? __fdividef(rn, curv) : 1.f;
        if (upd) {
          v.x = fmaf(alpha, pp.x, v.x);
          v.y = fmaf(alpha, pp.y, v.y);
          r.x = fmaf(-alpha, e.x, r.x);
          r.y = fmaf(-alpha, e.y, r.y);
        }
        const float rnx = group_sum<GL>(cnorm(r));
        __syncwarp();  // every lane's matvec reads of Ps are done
        if (upd) {
          const float beta = __fdividef(rnx, rn);
          rn = rnx;
          pp.x = fmaf(beta, pp.x, r.x);
          pp.y = fmaf(beta, pp.y, r.y);
          if (grp == 0) Ps[gl] = pp;
        }
        __syncwarp();
      }
      if (grp == 0) {
        Vs[sys * UP + gl] = v;
        if (gl == 0) sys_st[sys] = broke ? 1 : 0;
      }
    }
    __syncwarp();
    // ------------------------------ 3. q = H_d^H v, gain, s (precode.cpp:22-36)
    for (int s = 0; s < St; ++s) {
      const bool ok = sys_st[s] == 0;
      // conj(h) v = h.x (v.x, v.y) + h.y (v.y, -v.x)
      unsigned long long v1[UP], v2[UP];
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const float2 vv = Vs[s * UP + u];
        v1[u] = f2pack(vv.x, vv.y);
        v2[u] = f2pack(vv.y, -vv.x);
      }
      float2 qv[MQ];
      float nrm = 0.f;
      constexpr int QH = CB / 32;  // 32-antenna lane passes per chunk
      int nbq = 0;
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
        qv[m] = make_float2(0.f, 0.f);
        if (m * 32 < B) {
          if (m % QH == 0) nbq = acquire(sc, m / QH);
          const int bl = (m % QH) * 32 + lane;  // antenna within the chunk
          if (bl < nbq) {
            const float2* Hb = slot(cj) + bl;
            unsigned long long acc = 0ull, acc2 = 0ull;
#pragma unroll
            for (int u = 0; u < UP; u += 2) {
              const float2 h0 = Hb[u * LDH], h1 = Hb[(u + 1) * LDH];
              ffma2(acc, f2pack(h0.x, h0.x), v1[u]);
              ffma2(acc2, f2pack(h1.x, h1.x), v1[u + 1]);
              ffma2(acc, f2pack(h0.y, h0.y), v2[u]);
              ffma2(acc2, f2pack(h1.y, h1.y), v2[u + 1]);
            }
            const float2 A = f2unpack(acc), A2 = f2unpack(acc2);
            qv[m] = make_float2(A.x + A2.x, A.y + A2.y);
            nrm += cnorm(qv[m]);
          }
          if (m % QH == QH - 1 || (m + 1) * 32 >= B) release();
        }
      }
      nrm = group_sum<32>(nrm);  // fixed butterfly order
      const float g = sqrtf(nrm);
      const bool zero = ok && !(g > 0.f);
      const float inv = (ok && !zero) ? 1.f / g : 0.f;
      const long ob = (sc * St + s) * static_cast<long>(B);
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
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
    __syncwarp();  // Gs / Vs reads done before the next subcarrier overwrites them
  }
}

}  // namespace cgm
