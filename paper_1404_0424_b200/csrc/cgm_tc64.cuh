// cgm_tc64.cuh -- the channel kernel (K1) on the 5th-generation tensor cores
// for U = 64 (BASELINE configs[3] second case, cfg4b: B = 128, U = 64).
//
// Same mathematics as cgm_tc.cuh: with X = [H | Y] read as real numbers
// (row b = antenna), D = X_H^T X over the B antennas gives
//     G[u][j]  = (D[2u][2j]     + D[2u+1][2j+1],  D[2u][2j+1]     - D[2u+1][2j])
//     MF[u][s] = (D[2u][128+2s] + D[2u+1][129+2s], D[2u][129+2s] - D[2u+1][128+2s]),
// here with 2U = 128 real rows: M = 128, the full-rate tcgen05 shape, and
// N = 128 + ceil16(2S).  The bf16 x 3 split (x = p0 + p1 + p2, six products
// p_a p_b with a + b <= 2, p0 p0 in its own TMEM accumulator) keeps FP32
// accuracy exactly as in cgm_tc.cuh.
//
// Differences from the U = 32 kernel, all forced by the shapes:
//   * 32-antenna k-blocks (KB = 32): a piece is three 32-row SWIZZLE_128B
//     atoms (H columns 0-63, H columns 64-127, Y columns), 12 KB, so two
//     piece slots and a 3-deep staging ring fit next to the 33 KB G staging;
//   * the MMA reads A = the two H atoms (M = 128, MN-major, LBO = one atom)
//     and B = all three atoms (N = 128 + ny), 2 k-steps of 16 per k-block;
//   * one TMEM subcarrier buffer (big + small accumulators of N <= 192
//     columns each): the next subcarrier's MMAs wait until the epilogue has
//     drained the accumulators into registers;
//   * M = 128 accumulator layout: TMEM lane m = row m, read with
//     tcgen05.ld.32x32b (thread = row); row 2u+1's entries reach row 2u's
//     thread (and back) by one shuffle per column pair.
// Roles (one CTA per SM, persistent over subcarriers): warps 0-7 epilogue
// (two per TMEM lane quarter, splitting the columns), warps 8-15 split, warp
// 16 TMA producer, warp 17 MMA issuer.
#pragma once

#include "cgm_tc.cuh"

namespace cgm {
namespace tc64 {

constexpr int U64 = 64;             // users (M = 2U = 128 real rows)
constexpr int KB = 32;              // antennas per k-block
constexpr int ATOM = KB * 128;      // one SW128 column block: 32 rows x 64 bf16
constexpr int NATOM = 3;            // H columns 0-63, H columns 64-127, Y columns
constexpr int PIECE = NATOM * ATOM;
constexpr int PSLOT = 3 * PIECE;    // the three bf16 pieces of one k-block
constexpr int NPS = 2;              // piece slots
constexpr int ACC_COLS = 256;       // small accumulator at +256 (N <= 192)
constexpr int TMEM_COLS = 512;
constexpr int GPS = U64 + 1;        // padded G row stride (float2) in smem
constexpr int MAX_STG = 4;
constexpr int NEP = 8, NSP = 8;     // epilogue / split warps
constexpr int NT = 32 * (NEP + NSP + 2);

struct Smem {
  int pieces, stage, stage_bytes, nstg, gp, mf, bar, total;
  __host__ __device__ static int align(int x, int a) { return (x + a - 1) / a * a; }
  __host__ __device__ void plan(int S, int nstage) {
    int o = 0;
    pieces = o;
    o += NPS * PSLOT;
    stage_bytes = align(KB * U64 * 8 + KB * S * 8, 128);
    nstg = nstage;
    stage = o;
    o += nstg * stage_bytes;
    gp = o;
    o = align(o + U64 * GPS * 8, 128);
    mf = o;
    o = align(o + 32 * U64 * 8, 128);
    bar = o;
    o += 16 * 8 + 16 + 16;  // mbarriers, TMEM base
    total = align(o, 128) + 1024;  // + alignment slack of the dynamic base
  }
};

// natural layout, U = 64, whole 32-antenna k-blocks, at most 32 vectors
__host__ __device__ inline bool supported(int U, int B, int S, int use_tma) {
  return use_tma && U == U64 && B > 0 && (B % KB) == 0 && S >= 0 && 2 * S <= 64;
}

}  // namespace tc64

__global__ void __launch_bounds__(tc64::NT, 1) channel_tc64_kernel(const KernelParams p) {
  using namespace tc64;
  using tc::tc_commit_elect;
  using tc::tc_fence_after;
  using tc::tc_fence_before;
  using tc::tmem_ld8;
  using tc::tmem_wait_ld;
  constexpr int UP = U64;
  constexpr int NTE = 32 * NEP, NTS = 32 * NSP;
  constexpr int SPLIT0 = NEP, WPROD = NEP + NSP, WMMA = NEP + NSP + 1;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  tc64::Smem L;
  L.plan(p.S, p.k1_pair);
  WsOffsets W;
  W.plan(UP, p.S, p.K, p.exact != 0, p.fx != 0, p.zs);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = p.S, B = p.B, nkb = B / KB, nstg = L.nstg;
  // Y columns fed to the MMA, zero padded to 16 (M = 128 needs N % 16 == 0)
  const int ny = S > 0 ? ((2 * S + 15) & ~15) : 0;
  const int N = 2 * UP + ny;
  const long n_local =
      p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = bars + MAX_STG;
  uint64_t* pcs_full = bars + 2 * MAX_STG;
  uint64_t* pcs_empty = pcs_full + NPS;
  uint64_t* acc_full = pcs_empty + NPS;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  if (warp == 0) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  if (tid == 0) {
    for (int s = 0; s < nstg; ++s) {
      mbar_init(stg_full + s, 1);
      mbar_init(stg_empty + s, NSP);
    }
    for (int s = 0; s < NPS; ++s) {
      mbar_init(pcs_full + s, NSP);
      mbar_init(pcs_empty + s, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, NEP);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WPROD) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t hb = KB * UP * 8u, yb = KB * static_cast<uint32_t>(S) * 8u;
      long q = 0;
      for (long i = 0; i < n_local; ++i) {
        const long sc = p.sc_base + blockIdx.x + i * gridDim.x;
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          const int s = static_cast<int>(q % nstg);
          const long r = q / nstg;
          if (r > 0) mbar_wait(stg_empty + s, static_cast<uint32_t>((r - 1) & 1));
          unsigned char* dst = smem + L.stage + s * L.stage_bytes;
          const long row0 = sc * B + kb * KB;
          fence_proxy_async();
          mbar_expect_tx(stg_full + s, hb + yb);
          bulk_g2s(dst, p.H + row0 * UP, hb, stg_full + s);
          if (S > 0) bulk_g2s(dst + hb, p.Y + row0 * S, yb, stg_full + s);
        }
      }
    }
  } else if (warp == WMMA) {
    // ------------------------------------------------------ MMA issuer
    // A = pieces' H atoms (M = 128), B = all three atoms (N = 128 + ny)
    const uint32_t idesc = tc::idesc_bf16_mn(2 * UP, N);
    const uint64_t dbase = tc::smem_desc(smem_u32(smem + L.pieces), ATOM, 1024);
    const uint32_t d_big = tmem, d_small = tmem + ACC_COLS;
    long mq = 0;
    for (long i = 0; i < n_local; ++i) {
      if (i >= 1) mbar_wait(acc_empty, static_cast<uint32_t>((i - 1) & 1));
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb, ++mq) {
        const int ps = static_cast<int>(mq % NPS);
        mbar_wait(pcs_full + ps, static_cast<uint32_t>((mq / NPS) & 1));
        tc_fence_after();
        const uint64_t dslot = dbase + static_cast<uint64_t>((ps * PSLOT) >> 4);
#pragma unroll
        for (int pass = 0; pass < 6; ++pass) {
          constexpr int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
          for (int ks = 0; ks < KB / 16; ++ks) {
            const uint64_t da = dslot + ((pa[pass] * PIECE + ks * 2048) >> 4);
            const uint64_t db = dslot + ((pb[pass] * PIECE + ks * 2048) >> 4);
            if (pass == 0)
              tc::mma_bf16_elect(d_big, da, db, idesc, (kb | ks) ? 1u : 0u);
            else
              tc::mma_bf16_elect(d_small, da, db, idesc, (pass > 1 || kb || ks) ? 1u : 0u);
          }
        }
        tc_commit_elect(pcs_empty + ps);  // piece slot free once these MMAs retire
        __syncwarp();
      }
      tc_commit_elect(acc_full);  // accumulators of subcarrier i complete
      __syncwarp();
    }
  } else if (warp >= SPLIT0) {
    // ------------------------------------------------------ split warps
    const int st = tid - SPLIT0 * 32;  // 0 .. NTS-1
    const int nyc = ny / 8;            // Y chunks (8 columns) per antenna row
    const bool hswap = (lane >> 2) & 1;  // conflict-free staging reads (cgm_tc.cuh)
    constexpr int HCH = KB * (2 * UP / 8);  // H chunks per k-block (32 rows x 16)
    constexpr int HPT = HCH / NTS;          // per thread
    static_assert(HCH % NTS == 0, "H chunks must divide evenly");
    long pq = 0;
    int stg_s = 0;
    uint32_t sph = 0;
    for (long i = 0; i < n_local; ++i) {
      for (int kb = 0; kb < nkb; ++kb, ++pq) {
        mbar_wait(stg_full + stg_s, sph);
        const int ps = static_cast<int>(pq % NPS);
        if (pq >= NPS) mbar_wait(pcs_empty + ps, static_cast<uint32_t>(((pq / NPS) - 1) & 1));
        const float* Hst = reinterpret_cast<const float*>(smem + L.stage + stg_s * L.stage_bytes);
        const float* Yst = Hst + KB * UP * 2;
        unsigned char* slot = smem + L.pieces + ps * PSLOT;
        float hx[HPT][8];
#pragma unroll
        for (int r = 0; r < HPT; ++r) {
          const int it = st + r * NTS, k = it >> 4, j = it & 15;
          const float* src = Hst + k * (2 * UP) + j * 8;
          const float4 a0 = *reinterpret_cast<const float4*>(src + (hswap ? 4 : 0));
          const float4 b0 = *reinterpret_cast<const float4*>(src + (hswap ? 0 : 4));
          const float4 a = hswap ? b0 : a0, b = hswap ? a0 : b0;
          hx[r][0] = a.x; hx[r][1] = a.y; hx[r][2] = a.z; hx[r][3] = a.w;
          hx[r][4] = b.x; hx[r][5] = b.y; hx[r][6] = b.z; hx[r][7] = b.w;
        }
#pragma unroll
        for (int r = 0; r < HPT; ++r) {
          const int it = st + r * NTS, k = it >> 4, j = it & 15;
          uint4 o0, o1, o2;
          tc::split8(hx[r], o0, o1, o2);
          const int off = (j >> 3) * ATOM + k * 128 + (((j & 7) ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(slot + off) = o0;
          *reinterpret_cast<uint4*>(slot + PIECE + off) = o1;
          *reinterpret_cast<uint4*>(slot + 2 * PIECE + off) = o2;
        }
        for (int it = st; it < KB * nyc; it += NTS) {  // Y chunks, zero padded past 2S
          const int k = it / nyc, j = it - k * nyc;
          float x[8];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int col = j * 8 + 2 * t;
            float2 v = make_float2(0.f, 0.f);
            if (col < 2 * S) v = *reinterpret_cast<const float2*>(Yst + k * 2 * S + col);
            x[2 * t] = v.x;
            x[2 * t + 1] = v.y;
          }
          uint4 o0, o1, o2;
          tc::split8(x, o0, o1, o2);
          const int off = 2 * ATOM + k * 128 + ((j ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(slot + off) = o0;
          *reinterpret_cast<uint4*>(slot + PIECE + off) = o1;
          *reinterpret_cast<uint4*>(slot + 2 * PIECE + off) = o2;
        }
        fence_proxy_async();  // generic-proxy piece writes -> the MMA (async proxy)
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(pcs_full + ps);
          mbar_arrive(stg_empty + stg_s);
        }
        if (++stg_s == nstg) {
          stg_s = 0;
          sph ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------ epilogue warps
    float* Gpf = reinterpret_cast<float*>(smem + L.gp);  // [UP][GPS] float2 as floats
    float* Mpf = reinterpret_cast<float*>(smem + L.mf);  // [S][UP] float2 as floats
    const int qd = warp & 3;                 // TMEM lane quarter
    const int m = qd * 32 + lane;            // accumulator row = H column
    const int u = m >> 1, odd = m & 1;
    const int half = warp >> 2;              // which half of the columns
    const int nch = (N + 7) / 8;             // 8-column chunks
    const int c_lo = half ? (nch + 1) / 2 : 0, c_hi = half ? nch : (nch + 1) / 2;
    const uint32_t tq = tmem + (static_cast<uint32_t>(qd * 32) << 16);
    for (long e = 0; e < n_local; ++e) {
      mbar_wait(acc_full, static_cast<uint32_t>(e & 1));
      tc_fence_after();
      const long lsc = blockIdx.x + e * gridDim.x;
      float2* ws = p.ws + lsc * W.stride;
      for (int c = c_lo; c < c_hi; c += 2) {  // two chunks per TMEM round trip
        uint32_t vb[2][8], vs[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (c + h < c_hi) {
            tmem_ld8(tq + 8 * (c + h), vb[h]);
            tmem_ld8(tq + ACC_COLS + 8 * (c + h), vs[h]);
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (c + h >= c_hi) continue;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float x0 = __fadd_rn(__uint_as_float(vb[h][2 * t]), __uint_as_float(vs[h][2 * t]));
            const float x1 =
                __fadd_rn(__uint_as_float(vb[h][2 * t + 1]), __uint_as_float(vs[h][2 * t + 1]));
            const float other = __shfl_xor_sync(0xffffffffu, x1, 1);  // row m ^ 1, same column pair
            // even row 2u: re = D[2u][2j] + D[2u+1][2j+1]; odd row: im = D[2u][2j+1] - D[2u+1][2j]
            const float val = odd ? __fsub_rn(other, x0) : __fadd_rn(x0, other);
            const int j = 4 * (c + h) + t;  // column pair
            if (j < UP)
              Gpf[(u * GPS + j) * 2 + odd] = val;  // full row; Hermitian fix-up below
            else if (j - UP < S)
              Mpf[((j - UP) * UP + u) * 2 + odd] = val;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);  // the accumulators may be overwritten
      named_sync(1, NTE);                     // G rows and MF complete in smem
      {
        const float2* Gp2 = reinterpret_cast<const float2*>(Gpf);
        float2* Gw = ws + W.g;
        for (int x = tid; x < UP * UP; x += NTE) {  // lower triangle + conjugate mirror
          const int r = x >> 6, cc = x & 63;
          float2 g = Gp2[(cc < r ? r : cc) * GPS + (cc < r ? cc : r)];
          if (cc > r) g.y = -g.y;
          if (cc == r) g.y = 0.f;
          Gw[x] = g;
        }
        const float2* Mp2 = reinterpret_cast<const float2*>(Mpf);
        float2* Mw = ws + W.mf;
        for (int x = tid; x < S * UP; x += NTE) Mw[x] = Mp2[x];
      }
      named_sync(1, NTE);  // the staging is reused by the next subcarrier
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace cgm
