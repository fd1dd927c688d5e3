// cgm_block32.cuh -- K2 for U = 32 with many systems per subcarrier (cfg5:
// 16 uplink vectors + 16 transmit vectors on the same channel).
//
// Persistent CTAs walk the subcarriers; the NEXT subcarrier's workspace
// span (G, matched filters, Chebyshev interval, row moments: one contiguous
// block) and transmit vectors land in a second shared-memory buffer by
// cp.async.bulk while the current one is solved, so the per-subcarrier load
// latency leaves the critical path.  G is shared by every warp; each warp
// runs NS = 4 systems of the subcarrier at once (lane u = user row u):
//   * matvec e_u = sum_j G[u][j] p_j: lane u reads conj(G[j][u]) (one
//     conflict-free LDS.64 per column, reused by the NS systems) and each
//     system's p_j pair by a broadcast LDS.128; 2 packed FFMA2 per
//     (column, system) -- 16 FFMA2 per 6 loads for two columns;
//   * the 2 x NS dot products of an iteration (curvature, residual norm) are
//     reduced together: warp_sum4 sums four values over the 32 lanes with 9
//     shuffles instead of 20;
//   * K CG iterations with the reference's freeze (||r||^2 <= 1e-28 ||r0||^2
//     -> alpha = 1, beta = 0) and breakdown (p^H A p < 1e-30) rules
//     (solvers.cpp:21-27, 37-72), the approximate tracker's Eq. (11)
//     (detect.cpp:409-427) or the exact tracker's (alpha, beta) history.
// Tails: the exact tracker's extraction from the row moments (moments_tail,
// cgm_moments.cuh, CTA-wide); transmit vectors leave v_K and their status in
// the workspace for precode_q_kernel: thread b owns antenna row b and forms
// q_b = sum_u H[b][u] v_u for every transmit vector with packed FFMA2 (H
// row from L2 / HBM, v broadcast from shared memory), the norms ||q|| by a
// fixed-order reduction, then writes q and s = q / ||q|| straight from
// registers (precode.cpp:22-71).
#pragma once

#include <cuda.h>  // CUtensorMap (type only)

#include "cgm_rows32.cuh"

namespace cgm {

constexpr int kBlkNS = 4;    // systems per warp
constexpr int kBlkMaxW = 8;  // warps per CTA

struct Block32Smem {
  int bar, buf, bufb, tb, ps, vs, hist, msh, sys_st, gpart, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  // span = bytes of the workspace prefix [g, z) of one subcarrier
  __host__ __device__ void plan(int S, int St, int K, bool exact, int span) {
    const int nsys = S + St;
    int o = 0;
    bar = o; o = align(o + 16);
    tb = align(span);                       // T of the subcarrier after its ws span
    bufb = align(tb + St * 32 * 8);         // bytes per buffer
    buf = o; o = align(o + 2 * bufb);
    ps = o; o = align(o + (nsys + kBlkNS - 1) / kBlkNS * kBlkNS * 32 * 8);
    vs = o; o = align(o + (exact ? S * 32 * 8 : 0));
    hist = o; o = align(o + (exact ? S * K * 2 * 4 : 0));
    msh = o; o = align(o + (exact ? kBlkMaxW * kMomScratch * 8 : 0));
    sys_st = o; o = align(o + nsys);
    gpart = o; o = align(o + (kBlkMaxW + 2) * 16 * 4);  // precoder: per-warp norms, 1/gain, flags
    total = o;
  }
};

// CG for the systems base .. base + NS - 1 of subcarrier sc on one warp;
// Gs = the subcarrier's G in shared memory, Ps = this warp's NS broadcast
// rows.  Approximate uplink systems write their outputs; exact / downlink
// systems leave v in Vs and (exact) the history in hist.
// Exact tracker (cfg5): the same CG with the per-system scalar work done by
// the system's 8 owner lanes only.  After each reduction lane L holds the sum
// of system (L >> 3) & 3 (warp_sum4_owned); it alone applies the freeze /
// breakdown rules, forms alpha (then beta) and records the (alpha, beta)
// history, and one shuffle per system hands the step lengths to the warp.
// A system that does not update at iteration k never updates again (frozen
// residuals stay frozen, breakdowns stick, k only grows past its iteration
// count), so it is given alpha = 0 -- v and r unchanged -- and its p may be
// overwritten freely.
__device__ __forceinline__ void block32_cg_exact(const KernelParams& p, const float2* mfsrc,
                                                 const float2* Ts, int base, const float2* Gs,
                                                 float2* Ps, float* hist, float2* Vs,
                                                 uint8_t* sys_st, float2* zout) {
  constexpr int UP = 32, NS = kBlkNS;
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  const int lane = threadIdx.x & 31;
  float reg[NS];
  float2 v[NS], r[NS], pp[NS];
  float nrm[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + s;
    const bool live = sy < nsys, down = sy >= S;
    reg[s] = down ? p.rho_inv_d : p.rho_inv_u;
    float2 b = make_float2(0.f, 0.f);
    if (live && lane < U) b = down ? Ts[(sy - S) * U + lane] : mfsrc[sy * UP + lane];
    v[s] = make_float2(0.f, 0.f);
    r[s] = b;
    pp[s] = b;
    Ps[s * UP + lane] = b;
    nrm[s] = cnorm(b);
  }
  // this lane's system
  const int my = (lane >> 3) & 3, sy_own = base + my;
  const bool live_own = sy_own < nsys, down_own = sy_own >= S;
  const int iters_own = live_own ? (down_own ? p.Kt : p.K) : 0;
  float rn = warp_sum4_owned(nrm);
  const float rn0 = rn;
  bool broke = false;
  __syncwarp();
  for (int k = 1; k <= Kmax; ++k) {
    // e = (G + reg I) p on the packed pipe; G[u][j] = conj(G[j][u])
    unsigned long long a0[NS], b0[NS], a1[NS], b1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a0[s] = b0[s] = a1[s] = b1[s] = 0ull;
#pragma unroll 4
    for (int j = 0; j < UP; j += 2) {
      const float2 gj0 = Gs[j * UP + lane], gj1 = Gs[(j + 1) * UP + lane];
      const unsigned long long g0 = f2pack(gj0.x, -gj0.y), g1 = f2pack(gj1.x, -gj1.y);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj = *reinterpret_cast<const ulonglong2*>(Ps + s * UP + j);
        ffma2(a0[s], g0, f2dup_lo(pj.x));
        ffma2(b0[s], g0, f2dup_hi(pj.x));
        ffma2(a1[s], g1, f2dup_lo(pj.y));
        ffma2(b1[s], g1, f2dup_hi(pj.y));
      }
    }
    float2 e[NS];
    float part[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float2 A0 = f2unpack(a0[s]), B0 = f2unpack(b0[s]);
      const float2 A1 = f2unpack(a1[s]), B1 = f2unpack(b1[s]);
      e[s].x = (A0.x - B0.y) + (A1.x - B1.y);
      e[s].y = (B0.x + A0.y) + (B1.x + A1.y);
      e[s].x = fmaf(reg[s], pp[s].x, e[s].x);
      e[s].y = fmaf(reg[s], pp[s].y, e[s].y);
      part[s] = pp[s].x * e[s].x + pp[s].y * e[s].y;  // Re p^H e
    }
    const float curv = warp_sum4_owned(part);
    // owner lanes: solvers.cpp:21-27 freeze, :55-57 breakdown
    const bool step = k <= iters_own;
    const bool frozen = !(rn > 1e-28f * rn0);
    const bool go = step && !frozen && !broke;
    if (go && curv < 1e-30f) broke = true;
    const bool upd = go && !broke;
    const float alpha = upd ? __fdividef(rn, curv) : 1.f;
    const float a_eff = upd ? alpha : 0.f;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float as = __shfl_sync(0xffffffffu, a_eff, s << 3);
      v[s].x = fmaf(as, pp[s].x, v[s].x);
      v[s].y = fmaf(as, pp[s].y, v[s].y);
      r[s].x = fmaf(-as, e[s].x, r[s].x);
      r[s].y = fmaf(-as, e[s].y, r[s].y);
      part[s] = cnorm(r[s]);
    }
    const float rnx = warp_sum4_owned(part);
    const float beta = upd ? rnx * __fdividef(1.f, rn) : 0.f;
    if (upd) rn = rnx;
    if (step && !down_own && (lane & 7) == 0) {  // the exact tracker's history
      hist[(sy_own * Kmax + (k - 1)) * 2 + 0] = alpha;
      hist[(sy_own * Kmax + (k - 1)) * 2 + 1] = beta;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float bs = __shfl_sync(0xffffffffu, beta, s << 3);
      pp[s].x = fmaf(bs, pp[s].x, r[s].x);
      pp[s].y = fmaf(bs, pp[s].y, r[s].y);
    }
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s) Ps[s * UP + lane] = pp[s];
    __syncwarp();
  }
  // ------------------------------------------------ per-system epilogue
  if (live_own && (lane & 7) == 0) {
    if (down_own) zout[St * UP + (sy_own - S)] = make_float2(broke ? 1.f : 0.f, 0.f);
    else sys_st[sy_own] = broke ? 1 : 0;
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + s;
    if (sy >= nsys) continue;
    if (sy >= S) zout[(sy - S) * UP + lane] = v[s];  // v_K for precode_q_kernel
    else Vs[sy * UP + lane] = v[s];
  }
}

// ---------------------------------------------------------------------------
// Register-tiled exact CG (cfg5 default): a warp runs 8 systems, lane L owns
// user rows 2 (L & 15), + 1 of the 4 systems (L >> 4) * 4 .. + 3 of its
// group.  Per column pair (j, j + 1) a lane issues 2 LDS.128 of G (its two
// rows, a 16-lane broadcast pair: 4 wavefronts per warp) and 4 broadcast
// LDS.128 of p (1 wavefront each: the two halves' rows sit 16 banks apart
// with the kPStr row stride) for 32 FFMA2 -- twice the math per shared-memory
// wavefront of the lane-per-row form, which was balanced between the two.
// The inner products reduce over 16 lanes (sum4_16_owned: 5 shuffles for the
// 4 systems of a half, lane L ends with system (L >> 2) & 3 of its half, the
// system's 4 owner lanes), the owners apply the freeze / breakdown rules and
// form alpha / beta, one shuffle per system hands them out.
constexpr int kTSpw = 8;   // systems per warp (tiled)
constexpr int kTWarps = 4;  // warps per CTA (tiled)
constexpr int kPStr = 34;   // float2 row stride of the broadcast p rows

__device__ __forceinline__ float sum4_16_owned(const float (&v)[4]) {
  const int lane = threadIdx.x & 31;
  const bool b3 = lane & 8, b2 = lane & 4;
  float k0 = b3 ? v[2] : v[0], k1 = b3 ? v[3] : v[1];
  const float s0 = b3 ? v[0] : v[2], s1 = b3 ? v[1] : v[3];
  k0 += __shfl_xor_sync(0xffffffffu, s0, 8);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 8);
  float k = b2 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, b2 ? k0 : k1, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;  // system ((L >> 3) & 1) * 2 + ((L >> 2) & 1) = (L >> 2) & 3 of half L >> 4
}

struct Block32TSmem {
  int bar, buf, bufb, tb, ps, hist, msh, msh_doubles, sys_st, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int S, int St, int K, int span) {
    const int nsys = S + St;
    int o = 0;
    bar = o; o = align(o + 16);
    tb = align(span);
    bufb = align(tb + St * 32 * 8);
    buf = o; o = align(o + 2 * bufb);
    ps = o; o = align(o + (nsys + kTSpw - 1) / kTSpw * kTSpw * kPStr * 8);  // p rows, then v_K (uplink)
    hist = o; o = align(o + S * K * 2 * 4);
    msh_doubles = kTWarps * kMomScratch > S * kLaneScratch ? kTWarps * kMomScratch : S * kLaneScratch;
    msh = o; o = align(o + msh_doubles * 8);
    sys_st = o; o = align(o + nsys);
    total = o;
  }
};

__device__ __forceinline__ void block32t_cg_exact(const KernelParams& p, const float2* mfsrc,
                                                  const float2* Ts, int base, const float2* Gs,
                                                  float2* Ps, float* hist, uint8_t* sys_st,
                                                  float2* zout) {
  constexpr int UP = 32, NS = 4;
  const int S = p.S, St = p.St;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  const int lane = threadIdx.x & 31;
  const int h = lane >> 4, u0 = 2 * (lane & 15);
  float reg[NS];
  float2 v[2][NS], r[2][NS], pp[2][NS];
  float nrm[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + 4 * h + s;
    const bool live = sy < nsys, down = sy >= S;
    reg[s] = down ? p.rho_inv_d : p.rho_inv_u;
    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live)
      b = *reinterpret_cast<const float4*>(down ? Ts + (sy - S) * UP + u0 : mfsrc + sy * UP + u0);
    v[0][s] = v[1][s] = make_float2(0.f, 0.f);
    r[0][s] = pp[0][s] = make_float2(b.x, b.y);
    r[1][s] = pp[1][s] = make_float2(b.z, b.w);
    *reinterpret_cast<float4*>(Ps + (4 * h + s) * kPStr + u0) = b;
    nrm[s] = cnorm(r[0][s]) + cnorm(r[1][s]);
  }
  // this lane's system (owner of its scalar work): (L >> 2) & 3 of half h
  const int my = (lane >> 2) & 3, sy_own = base + 4 * h + my;
  const bool live_own = sy_own < nsys, down_own = sy_own >= S;
  const int iters_own = live_own ? (down_own ? p.Kt : p.K) : 0;
  float rn = sum4_16_owned(nrm);
  const float rn0 = rn;
  bool broke = false;
  const float2* Pg = Ps + 4 * h * kPStr;  // this half's four p rows
  __syncwarp();
  for (int k = 1; k <= Kmax; ++k) {
    // e = (G + reg I) p: G[u][j] = conj(G[j][u]) (packed (re, -im) x p.x, p.y)
    unsigned long long a[2][NS], b[2][NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a[0][s] = a[1][s] = b[0][s] = b[1][s] = 0ull;
#pragma unroll 2
    for (int j = 0; j < UP; j += 2) {
      const float4 g0 = *reinterpret_cast<const float4*>(Gs + j * UP + u0);
      const float4 g1 = *reinterpret_cast<const float4*>(Gs + (j + 1) * UP + u0);
      const unsigned long long g00 = f2pack(g0.x, -g0.y), g01 = f2pack(g0.z, -g0.w);
      const unsigned long long g10 = f2pack(g1.x, -g1.y), g11 = f2pack(g1.z, -g1.w);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj = *reinterpret_cast<const ulonglong2*>(Pg + s * kPStr + j);
        const unsigned long long x0 = f2dup_lo(pj.x), y0 = f2dup_hi(pj.x);
        const unsigned long long x1 = f2dup_lo(pj.y), y1 = f2dup_hi(pj.y);
        ffma2(a[0][s], g00, x0);
        ffma2(b[0][s], g00, y0);
        ffma2(a[1][s], g01, x0);
        ffma2(b[1][s], g01, y0);
        ffma2(a[0][s], g10, x1);
        ffma2(b[0][s], g10, y1);
        ffma2(a[1][s], g11, x1);
        ffma2(b[1][s], g11, y1);
      }
    }
    float2 e[2][NS];
    float part[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      part[s] = 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float2 A = f2unpack(a[q][s]), B = f2unpack(b[q][s]);
        e[q][s].x = fmaf(reg[s], pp[q][s].x, A.x - B.y);
        e[q][s].y = fmaf(reg[s], pp[q][s].y, A.y + B.x);
        part[s] += pp[q][s].x * e[q][s].x + pp[q][s].y * e[q][s].y;  // Re p^H e
      }
    }
    const float curv = sum4_16_owned(part);
    // owner lanes: solvers.cpp:21-27 freeze, :55-57 breakdown
    const bool step = k <= iters_own;
    const bool frozen = !(rn > 1e-28f * rn0);
    const bool go = step && !frozen && !broke;
    if (go && curv < 1e-30f) broke = true;
    const bool upd = go && !broke;
    const float alpha = upd ? __fdividef(rn, curv) : 1.f;
    const float a_eff = upd ? alpha : 0.f;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float as = __shfl_sync(0xffffffffu, a_eff, (lane & 16) + 4 * s);
      part[s] = 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        v[q][s].x = fmaf(as, pp[q][s].x, v[q][s].x);
        v[q][s].y = fmaf(as, pp[q][s].y, v[q][s].y);
        r[q][s].x = fmaf(-as, e[q][s].x, r[q][s].x);
        r[q][s].y = fmaf(-as, e[q][s].y, r[q][s].y);
        part[s] += cnorm(r[q][s]);
      }
    }
    const float rnx = sum4_16_owned(part);
    const float beta = upd ? rnx * __fdividef(1.f, rn) : 0.f;
    if (upd) rn = rnx;
    if (step && !down_own && (lane & 3) == 0) {  // the exact tracker's history
      hist[(sy_own * Kmax + (k - 1)) * 2 + 0] = alpha;
      hist[(sy_own * Kmax + (k - 1)) * 2 + 1] = beta;
    }
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float bs = __shfl_sync(0xffffffffu, beta, (lane & 16) + 4 * s);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        pp[q][s].x = fmaf(bs, pp[q][s].x, r[q][s].x);
        pp[q][s].y = fmaf(bs, pp[q][s].y, r[q][s].y);
      }
      *reinterpret_cast<float4*>(Ps + (4 * h + s) * kPStr + u0) =
          make_float4(pp[0][s].x, pp[0][s].y, pp[1][s].x, pp[1][s].y);
    }
    __syncwarp();
  }
  // ------------------------------------------------ per-system epilogue
  if (live_own && (lane & 3) == 0) {
    if (down_own) zout[St * UP + (sy_own - S)] = make_float2(broke ? 1.f : 0.f, 0.f);
    else sys_st[sy_own] = broke ? 1 : 0;
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + 4 * h + s;
    if (sy >= nsys) continue;
    const float4 vv = make_float4(v[0][s].x, v[0][s].y, v[1][s].x, v[1][s].y);
    if (sy >= S) *reinterpret_cast<float4*>(zout + (sy - S) * UP + u0) = vv;  // for precode_q_kernel
    else *reinterpret_cast<float4*>(Ps + (4 * h + s) * kPStr + u0) = vv;     // v_K over its own p row
  }
}

// Persistent tiled-CG kernel (exact tracker, U = 32): 4 warps, 4 CTAs per SM;
// the workspace span / transmit-vector double buffer of block32_kernel.
__global__ void __launch_bounds__(32 * kTWarps, 4) block32t_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  WsOffsets W;
  W.plan(UP, S, p.K, true, p.fx, p.zs);
  const uint32_t span = static_cast<uint32_t>(W.z) * 8u, tbytes = static_cast<uint32_t>(St * U) * 8u;
  Block32TSmem L;
  L.plan(S, St, Kmax, static_cast<int>(span));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  const int nt = blockDim.x, nw = nt >> 5;
  const int tid = threadIdx.x, warp = tid >> 5;
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto bufp = [&](long i) { return smem + L.buf + (i & 1) * L.bufb; };
  auto issue = [&](long i) {
    const long lsc = blockIdx.x + i * gridDim.x;
    unsigned char* dst = bufp(i);
    fence_proxy_async();  // generic reads of this buffer (two subcarriers ago) before the async write
    mbar_expect_tx(bar + (i & 1), span + tbytes);
    bulk_g2s(dst, p.ws + lsc * W.stride, span, bar + (i & 1));
    if (St > 0) bulk_g2s(dst + L.tb, p.T + (p.sc_base + lsc) * St * U, tbytes, bar + (i & 1));
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  if (tid == 0 && n_local > 0) issue(0);
  for (long i = 0; i < n_local; ++i) {
    if (tid == 0 && i + 1 < n_local) issue(i + 1);
    mbar_wait(bar + (i & 1), static_cast<uint32_t>((i >> 1) & 1));
    const long lsc = blockIdx.x + i * gridDim.x;
    const long sc = p.sc_base + lsc;
    const float2* wsb = reinterpret_cast<const float2*>(bufp(i));  // smem copy of the ws span
    const float2* Ts = reinterpret_cast<const float2*>(bufp(i) + L.tb);
    float2* zout = p.ws + lsc * W.stride + W.z;
    for (int base = warp * kTSpw; base < nsys; base += nw * kTSpw)
      block32t_cg_exact(p, wsb + W.mf, Ts, base, wsb + W.g, Ps + base * kPStr, hist, sys_st, zout);
    if (S > 0) {
      __syncthreads();
      moments_tail<UP>(p, wsb, W, sc, Kmax, hist, Ps, sys_st, nt,
                       reinterpret_cast<double*>(smem + L.msh), kPStr, L.msh_doubles);
    }
    __syncthreads();  // buffer i & 1 and the per-subcarrier scratch are free
  }
}

// ---------------------------------------------------------------------------
// Register-tiled CG with the approximate tracker (uplink only: cfg2).  Same
// lane layout as block32t_cg_exact -- a warp runs 8 systems, lane L owns user
// rows 2 (L & 15), + 1 of the 4 systems of its half -- with Eq. (11)'s
// diagonal recursion (detect.cpp:409-427) per (row, system) in registers.
// The system's owner lanes apply the freeze / breakdown rules and form
// alpha, beta and the recursion's two per-system scalars c1 = alpha_k
// (1 + beta_{k-1}) / alpha_{k-1}, c2 = alpha_k beta_{k-2} / alpha_{k-2}
// (detect.cpp:350-358); four shuffles per system hand them out.  alpha
// travels negated when the system does not update (alpha = 1 by the
// reference's rule, but v and r stay put), so no fifth value is needed.
struct Block32ASmem {
  int bar, buf, bufb, ps, total;
  __host__ __device__ static int align(int x) { return (x + 127) & ~127; }
  __host__ __device__ void plan(int S, int span) {
    int o = 0;
    bar = o; o = align(o + 16);
    bufb = align(span);
    buf = o; o = align(o + 2 * bufb);
    ps = o; o = align(o + (S + kTSpw - 1) / kTSpw * kTSpw * kPStr * 8);
    total = o;
  }
};

__device__ __forceinline__ void block32a_cg(const KernelParams& p, long sc, const float2* mfsrc,
                                            int base, const float2* Gs, float2* Ps) {
  constexpr int UP = 32, NS = 4;
  const int S = p.S, U = p.U, K = p.K;
  const int lane = threadIdx.x & 31;
  const int h = lane >> 4, u0 = 2 * (lane & 15);
  const float reg = p.rho_inv_u;
  const float gd[2] = {Gs[u0 * UP + u0].x, Gs[(u0 + 1) * UP + u0 + 1].x};
  float2 v[2][NS], r[2][NS], pp[2][NS];
  float f0[2][NS], f1[2][NS], f2[2][NS];
  float nrm[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + 4 * h + s;
    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sy < S) b = *reinterpret_cast<const float4*>(mfsrc + sy * UP + u0);
    v[0][s] = v[1][s] = make_float2(0.f, 0.f);
    r[0][s] = pp[0][s] = make_float2(b.x, b.y);
    r[1][s] = pp[1][s] = make_float2(b.z, b.w);
    *reinterpret_cast<float4*>(Ps + (4 * h + s) * kPStr + u0) = b;
    nrm[s] = cnorm(r[0][s]) + cnorm(r[1][s]);
#pragma unroll
    for (int q = 0; q < 2; ++q) f0[q][s] = f1[q][s] = f2[q][s] = 0.f;
  }
  // this lane's system (owner of its scalar work): (L >> 2) & 3 of half h
  const int my = (lane >> 2) & 3, sy_own = base + 4 * h + my;
  const bool live_own = sy_own < S;
  float rn = sum4_16_owned(nrm);
  const float rn0 = rn;
  bool broke = false;
  float ia1 = 1.f, ia2 = 1.f, bm1 = 0.f, bm2 = 0.f;  // 1 / alpha and beta of the last two iterations
  const float2* Pg = Ps + 4 * h * kPStr;  // this half's four p rows
  __syncwarp();
  for (int k = 1; k <= K; ++k) {
    unsigned long long a[2][NS], b[2][NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a[0][s] = a[1][s] = b[0][s] = b[1][s] = 0ull;
#pragma unroll 2
    for (int j = 0; j < UP; j += 2) {
      const float4 g0 = *reinterpret_cast<const float4*>(Gs + j * UP + u0);
      const float4 g1 = *reinterpret_cast<const float4*>(Gs + (j + 1) * UP + u0);
      const unsigned long long g00 = f2pack(g0.x, -g0.y), g01 = f2pack(g0.z, -g0.w);
      const unsigned long long g10 = f2pack(g1.x, -g1.y), g11 = f2pack(g1.z, -g1.w);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj = *reinterpret_cast<const ulonglong2*>(Pg + s * kPStr + j);
        const unsigned long long x0 = f2dup_lo(pj.x), y0 = f2dup_hi(pj.x);
        const unsigned long long x1 = f2dup_lo(pj.y), y1 = f2dup_hi(pj.y);
        ffma2(a[0][s], g00, x0);
        ffma2(b[0][s], g00, y0);
        ffma2(a[1][s], g01, x0);
        ffma2(b[1][s], g01, y0);
        ffma2(a[0][s], g10, x1);
        ffma2(b[0][s], g10, y1);
        ffma2(a[1][s], g11, x1);
        ffma2(b[1][s], g11, y1);
      }
    }
    float2 e[2][NS];
    float part[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      part[s] = 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float2 A = f2unpack(a[q][s]), B = f2unpack(b[q][s]);
        e[q][s].x = fmaf(reg, pp[q][s].x, A.x - B.y);
        e[q][s].y = fmaf(reg, pp[q][s].y, A.y + B.x);
        part[s] += pp[q][s].x * e[q][s].x + pp[q][s].y * e[q][s].y;  // Re p^H e
      }
    }
    const float curv = sum4_16_owned(part);
    // owner lanes: solvers.cpp:21-27 freeze, :55-57 breakdown
    const bool frozen = !(rn > 1e-28f * rn0);
    const bool go = live_own && !frozen && !broke;
    if (go && curv < 1e-30f) broke = true;
    const bool upd = go && !broke;
    const float irn = __fdividef(1.f, rn);
    const float alpha = upd ? rn * __fdividef(1.f, curv) : 1.f;
    const float c1 = alpha * (1.f + bm1) * ia1, c2 = alpha * bm2 * ia2;
    const float a_sgn = upd ? alpha : -alpha;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float as = __shfl_sync(0xffffffffu, a_sgn, (lane & 16) + 4 * s);
      const float ae = as > 0.f ? as : 0.f;
      part[s] = 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        v[q][s].x = fmaf(ae, pp[q][s].x, v[q][s].x);
        v[q][s].y = fmaf(ae, pp[q][s].y, v[q][s].y);
        r[q][s].x = fmaf(-ae, e[q][s].x, r[q][s].x);
        r[q][s].y = fmaf(-ae, e[q][s].y, r[q][s].y);
        part[s] += cnorm(r[q][s]);
      }
      // Eq. (11) on the diagonal (detect.cpp:409-427); k = 1: L_1 = alpha_1
      const float al = fabsf(as);
      const float c1s = __shfl_sync(0xffffffffu, c1, (lane & 16) + 4 * s);
      const float c2s = __shfl_sync(0xffffffffu, c2, (lane & 16) + 4 * s);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float nk = f0[q][s] + (c1s - al * (gd[q] + reg)) * (f0[q][s] - f1[q][s]) -
                         c2s * (f1[q][s] - f2[q][s]);
        f2[q][s] = f1[q][s];
        f1[q][s] = f0[q][s];
        f0[q][s] = k == 1 ? al : nk;
      }
    }
    const float rnx = sum4_16_owned(part);
    const float beta = upd ? rnx * irn : 0.f;
    ia2 = ia1;
    ia1 = upd ? curv * irn : 1.f;
    bm2 = bm1;
    bm1 = beta;
    if (upd) rn = rnx;
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float bs = __shfl_sync(0xffffffffu, beta, (lane & 16) + 4 * s);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        pp[q][s].x = fmaf(bs, pp[q][s].x, r[q][s].x);
        pp[q][s].y = fmaf(bs, pp[q][s].y, r[q][s].y);
      }
      *reinterpret_cast<float4*>(Ps + (4 * h + s) * kPStr + u0) =
          make_float4(pp[0][s].x, pp[0][s].y, pp[1][s].x, pp[1][s].y);
    }
    __syncwarp();
  }
  // ------------- outputs: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
  const float rho_row[2] = {gd[0] / p.n0, gd[1] / p.n0};  // the same for every vector of the subcarrier
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int sy = base + 4 * h + s;
    const bool ok = __shfl_sync(0xffffffffu, broke ? 0 : 1, (lane & 16) + 4 * s) != 0;
    if (sy >= S) continue;
    if (p.status && (lane & 15) == 0) p.status[sc * S + sy] = ok ? 0 : 1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int u = u0 + q;
      if (u >= U) continue;
      const long o = (sc * S + sy) * static_cast<long>(U) + u;
      const float2 xh = ok ? v[q][s] : make_float2(0.f, 0.f);
      const float mu_u = ok ? f0[q][s] * gd[q] : 0.f;
      const float rho_u = ok ? rho_row[q] : 0.f;
      if (p.xhat) p.xhat[o] = xh;
      if (p.mu) p.mu[o] = mu_u;
      if (p.rho) p.rho[o] = rho_u;
      if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
    }
  }
}

// Persistent tiled-CG kernel, approximate tracker, uplink only (U = 32):
// ceil(S / 8) warps per CTA (cfg2: 2), the workspace span (G, matched
// filters) double-buffered by cp.async.bulk as in block32t_kernel.  Held to
// 168 registers (no spills; at 128 the tracker state spilled and the kernel
// lost to the pairs kernel).
__global__ void __launch_bounds__(32 * kTWarps, 3) block32a_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.S;
  WsOffsets W;
  W.plan(UP, S, p.K, false, false, 0);
  const uint32_t span = static_cast<uint32_t>(W.z) * 8u;
  Block32ASmem L;
  L.plan(S, static_cast<int>(span));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  const int nw = blockDim.x >> 5;
  const int tid = threadIdx.x, warp = tid >> 5;
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto bufp = [&](long i) { return smem + L.buf + (i & 1) * L.bufb; };
  auto issue = [&](long i) {
    const long lsc = blockIdx.x + i * gridDim.x;
    fence_proxy_async();  // generic reads of this buffer (two subcarriers ago) before the async write
    mbar_expect_tx(bar + (i & 1), span);
    bulk_g2s(bufp(i), p.ws + lsc * W.stride, span, bar + (i & 1));
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  if (tid == 0 && n_local > 0) issue(0);
  for (long i = 0; i < n_local; ++i) {
    if (tid == 0 && i + 1 < n_local) issue(i + 1);
    mbar_wait(bar + (i & 1), static_cast<uint32_t>((i >> 1) & 1));
    const long sc = p.sc_base + blockIdx.x + i * gridDim.x;
    const float2* wsb = reinterpret_cast<const float2*>(bufp(i));
    for (int base = warp * kTSpw; base < S; base += nw * kTSpw)
      block32a_cg(p, sc, wsb + W.mf, base, wsb + W.g, Ps + base * kPStr);
    __syncthreads();  // buffer i & 1 is free
  }
}

template <bool EXACT>
__device__ __forceinline__ void block32_cg(const KernelParams& p, long sc, const float2* mfsrc,
                                           const float2* Ts, int base, const float2* Gs,
                                           float2* Ps, float* hist, float2* Vs, uint8_t* sys_st,
                                           float2* zout) {
  constexpr int UP = 32, NS = kBlkNS;
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  const int lane = threadIdx.x & 31;
  const float gdiag = Gs[lane * UP + lane].x;
  int sys[NS], iters[NS];
  bool live[NS], down[NS], broke[NS];
  float reg[NS], rn[NS], rn0[NS];
  float2 v[NS], r[NS], pp[NS];
  float f0[NS], f1[NS], f2[NS], ia1[NS], ia2[NS], bm1[NS], bm2[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sys[s] = base + s;
    live[s] = sys[s] < nsys;
    down[s] = sys[s] >= S;
    reg[s] = down[s] ? p.rho_inv_d : p.rho_inv_u;
    iters[s] = live[s] ? (down[s] ? p.Kt : p.K) : 0;
    float2 b = make_float2(0.f, 0.f);
    if (live[s] && lane < U)
      b = down[s] ? Ts[(sys[s] - S) * U + lane] : mfsrc[sys[s] * UP + lane];
    v[s] = make_float2(0.f, 0.f);
    r[s] = b;
    pp[s] = b;
    Ps[s * UP + lane] = b;
    rn[s] = cnorm(b);
    broke[s] = false;
    ia1[s] = ia2[s] = 1.f;
    bm1[s] = bm2[s] = 0.f;
    f0[s] = f1[s] = f2[s] = 0.f;
  }
  warp_sum4(rn);
#pragma unroll
  for (int s = 0; s < NS; ++s) rn0[s] = rn[s];
  __syncwarp();
  for (int k = 1; k <= Kmax; ++k) {
    // e = (G + reg I) p on the packed pipe; G[u][j] = conj(G[j][u])
    unsigned long long a0[NS], b0[NS], a1[NS], b1[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) a0[s] = b0[s] = a1[s] = b1[s] = 0ull;
#pragma unroll 4
    for (int j = 0; j < UP; j += 2) {
      const float2 gj0 = Gs[j * UP + lane], gj1 = Gs[(j + 1) * UP + lane];
      const unsigned long long g0 = f2pack(gj0.x, -gj0.y), g1 = f2pack(gj1.x, -gj1.y);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const ulonglong2 pj = *reinterpret_cast<const ulonglong2*>(Ps + s * UP + j);
        ffma2(a0[s], g0, f2dup_lo(pj.x));
        ffma2(b0[s], g0, f2dup_hi(pj.x));
        ffma2(a1[s], g1, f2dup_lo(pj.y));
        ffma2(b1[s], g1, f2dup_hi(pj.y));
      }
    }
    float2 e[NS];
    float curv[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float2 A0 = f2unpack(a0[s]), B0 = f2unpack(b0[s]);
      const float2 A1 = f2unpack(a1[s]), B1 = f2unpack(b1[s]);
      e[s].x = (A0.x - B0.y) + (A1.x - B1.y);
      e[s].y = (B0.x + A0.y) + (B1.x + A1.y);
      e[s].x = fmaf(reg[s], pp[s].x, e[s].x);
      e[s].y = fmaf(reg[s], pp[s].y, e[s].y);
      curv[s] = pp[s].x * e[s].x + pp[s].y * e[s].y;  // Re p^H e
    }
    warp_sum4(curv);
    float alpha[NS], beta[NS], rnx[NS];
    bool upd[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool step = k <= iters[s];
      const bool frozen = !(rn[s] > 1e-28f * rn0[s]);  // solvers.cpp:21,25-27
      const bool go = step && !frozen && !broke[s];
      if (go && curv[s] < 1e-30f) broke[s] = true;  // solvers.cpp:55-57
      upd[s] = go && !broke[s];
      alpha[s] = upd[s] ? __fdividef(rn[s], curv[s]) : 1.f;
      beta[s] = 0.f;
      if (upd[s]) {
        v[s].x = fmaf(alpha[s], pp[s].x, v[s].x);
        v[s].y = fmaf(alpha[s], pp[s].y, v[s].y);
        r[s].x = fmaf(-alpha[s], e[s].x, r[s].x);
        r[s].y = fmaf(-alpha[s], e[s].y, r[s].y);
      }
      rnx[s] = cnorm(r[s]);
    }
    warp_sum4(rnx);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      float ia = 1.f;  // 1 / alpha
      if (upd[s]) {
        const float irn = __fdividef(1.f, rn[s]);
        beta[s] = rnx[s] * irn;
        ia = curv[s] * irn;
        rn[s] = rnx[s];
        pp[s].x = fmaf(beta[s], pp[s].x, r[s].x);
        pp[s].y = fmaf(beta[s], pp[s].y, r[s].y);
      }
      if (k <= iters[s]) {
        if (!down[s]) {
          if (EXACT) {
            if (lane == 0) {
              hist[(sys[s] * Kmax + (k - 1)) * 2 + 0] = alpha[s];
              hist[(sys[s] * Kmax + (k - 1)) * 2 + 1] = beta[s];
            }
          } else {
            // Eq. (11) on the diagonal (detect.cpp:409-427); k = 1: L_1 = alpha_1
            const float c1 = alpha[s] * (1.f + bm1[s]) * ia1[s];
            const float c2 = alpha[s] * bm2[s] * ia2[s];
            const float nk = f0[s] + (c1 - alpha[s] * (gdiag + reg[s])) * (f0[s] - f1[s]) -
                             c2 * (f1[s] - f2[s]);
            const float nf = k == 1 ? alpha[s] : nk;
            f2[s] = f1[s];
            f1[s] = f0[s];
            f0[s] = nf;
          }
        }
        ia2[s] = ia1[s]; ia1[s] = ia;
        bm2[s] = bm1[s]; bm1[s] = beta[s];
      }
    }
    __syncwarp();  // every lane's matvec reads of Ps are done
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (upd[s]) Ps[s * UP + lane] = pp[s];
    __syncwarp();
  }
  // ------------------------------------------------ per-system epilogue
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (!live[s]) continue;
    if (down[s]) {  // v_K and the breakdown flag for precode_q_kernel
      const int ts = sys[s] - S;
      zout[ts * UP + lane] = v[s];
      if (lane == 0) zout[St * UP + ts] = make_float2(broke[s] ? 1.f : 0.f, 0.f);
      continue;
    }
    if (EXACT && lane == 0) sys_st[sys[s]] = broke[s] ? 1 : 0;
    if (EXACT) {
      Vs[sys[s] * UP + lane] = v[s];
      continue;
    }
    if constexpr (!EXACT) {
      // approx uplink: mu = Ltilde G_ii, rho = G_ii / N0 (detect.cpp:435-441)
      if (lane < U) {
        const long o = (sc * S + sys[s]) * static_cast<long>(U) + lane;
        const bool ok = !broke[s];
        const float2 xh = ok ? v[s] : make_float2(0.f, 0.f);
        const float mu_u = ok ? f0[s] * gdiag : 0.f;
        const float rho_u = ok ? gdiag / p.n0 : 0.f;
        if (p.xhat) p.xhat[o] = xh;
        if (p.mu) p.mu[o] = mu_u;
        if (p.rho) p.rho[o] = rho_u;
        if (p.llr) store_llrs_fast(xh, mu_u, rho_u, p.bits, p.llr + o * p.bits);
        if (p.status && lane == 0) p.status[sc * S + sys[s]] = ok ? 0 : 1;
      }
    }
  }
}

// Persistent solve kernel: subcarriers blockIdx.x, + gridDim.x, ...; the
// next one's workspace span and transmit vectors are bulk-copied into the
// other buffer while the current one is solved.
template <bool EXACT>
__global__ void __launch_bounds__(256, 2) block32_kernel(const KernelParams p) {
  constexpr int UP = 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.S, St = p.St, U = p.U;
  const int nsys = S + St;
  const int Kmax = p.K > p.Kt ? p.K : p.Kt;
  WsOffsets W;
  W.plan(UP, S, p.K, EXACT, p.fx, p.zs);
  const uint32_t span = static_cast<uint32_t>(W.z) * 8u, tbytes = static_cast<uint32_t>(St * U) * 8u;
  Block32Smem L;
  L.plan(S, St, Kmax, EXACT, static_cast<int>(span));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float2* Ps = reinterpret_cast<float2*>(smem + L.ps);
  float2* Vs = reinterpret_cast<float2*>(smem + L.vs);
  float* hist = reinterpret_cast<float*>(smem + L.hist);
  uint8_t* sys_st = reinterpret_cast<uint8_t*>(smem + L.sys_st);
  const int nt = blockDim.x, nw = nt >> 5;
  const int tid = threadIdx.x, warp = tid >> 5;
  const long n_local = p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto bufp = [&](long i) { return smem + L.buf + (i & 1) * L.bufb; };
  auto issue = [&](long i) {
    const long lsc = blockIdx.x + i * gridDim.x;
    unsigned char* dst = bufp(i);
    fence_proxy_async();  // generic reads of this buffer (two subcarriers ago) before the async write
    mbar_expect_tx(bar + (i & 1), span + tbytes);
    bulk_g2s(dst, p.ws + lsc * W.stride, span, bar + (i & 1));
    if (St > 0) bulk_g2s(dst + L.tb, p.T + (p.sc_base + lsc) * St * U, tbytes, bar + (i & 1));
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  if (tid == 0 && n_local > 0) issue(0);
  for (long i = 0; i < n_local; ++i) {
    if (tid == 0 && i + 1 < n_local) issue(i + 1);
    mbar_wait(bar + (i & 1), static_cast<uint32_t>((i >> 1) & 1));
    const long lsc = blockIdx.x + i * gridDim.x;
    const long sc = p.sc_base + lsc;
    const float2* wsb = reinterpret_cast<const float2*>(bufp(i));  // smem copy of the ws span
    const float2* Ts = reinterpret_cast<const float2*>(bufp(i) + L.tb);
    float2* zout = p.ws + lsc * W.stride + W.z;
    for (int base = warp * kBlkNS; base < nsys; base += nw * kBlkNS) {
      if constexpr (EXACT)
        block32_cg_exact(p, wsb + W.mf, Ts, base, wsb + W.g, Ps + base * UP, hist, Vs, sys_st, zout);
      else
        block32_cg<EXACT>(p, sc, wsb + W.mf, Ts, base, wsb + W.g, Ps + base * UP, hist, Vs, sys_st,
                          zout);
    }
    if (EXACT && S > 0) {
      __syncthreads();
      moments_tail<UP>(p, wsb, W, sc, Kmax, hist, Vs, sys_st, nt,
                       reinterpret_cast<double*>(smem + L.msh));
    }
    __syncthreads();  // buffer i & 1 and the per-subcarrier scratch are free
  }
}

// Precoder (precode.cpp:22-71) for the transmit vectors solved by
// block32_kernel (B <= 256, natural H_u layout, U = 32): one 256-thread CTA
// per subcarrier, several resident per SM so one CTA's loads overlap the
// others' math and stores.  The subcarrier's H (64 KB) arrives as two 2-D
// TMA tensor tiles (users 0-15 and 16-31: 128-byte rows, SWIZZLE_128B) on
// two mbarriers, v_K + status slots (4 KB) as one bulk copy on the first,
// so the first half's products start while the second half lands and no
// thread issues a load.  Register tile per thread: 4 antenna rows
// (rb + 64 i) x 4 vectors; warp w takes vectors 4 (w mod 4) .. + 3 and row
// block rb = (w / 4) * 32 + lane, so an LDS.128 phase of 8 lanes reads 8 rows
// with distinct (row mod 8) -- under the 128-byte swizzle (chunk c of row r
// at c ^ (r mod 8)) 8 distinct bank groups -- and the v_K reads are
// warp-wide broadcasts: 8 loads per 64 FFMA2.  q_b = sum_u H_u[b][u] v_u
// (precode.cpp:69 with H_d = H_u^H) on packed accumulators
// (a += (h.x, h.y) v.x, b += (h.x, h.y) v.y, q = (a.x - b.y, a.y + b.x));
// gain = ||q|| by a fixed-order reduction (a thread's 4 rows, warp_sum4
// over the lanes, the two row halves), s = q / gain, zero_input when the
// gain vanishes (precode.cpp:22-36); q and s leave from registers as
// coalesced 256-byte warp stores (streaming, evict-first).
struct PrecodeQSmem {
  static constexpr int NTH = 256;
  int bar, h, z, gpart, total;
  __host__ __device__ static int zbytes(int St) { return ((St * 33 + 1) & ~1) * 8; }
  __host__ __device__ void plan(int B, int St) {
    bar = 0;
    h = 1024;  // 128B-swizzled tiles: 1024-byte aligned
    z = h + 2 * B * 128;
    gpart = z + ((zbytes(St) + 127) & ~127);
    total = gpart + 4 * 16 * 4 + 1024;  // + slack to align the base
  }
};

template <int MINB>
__global__ void __launch_bounds__(256, MINB) precode_q_kernel(const KernelParams p,
                                                               const __grid_constant__ CUtensorMap tmH) {
  constexpr int UP = 32, TR = 4, TV = 4;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int St = p.St, B = p.B;
  WsOffsets W;
  W.plan(UP, p.S, p.K, p.exact != 0, p.fx != 0, p.zs);
  PrecodeQSmem L;
  L.plan(B, St);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  float* gpart = reinterpret_cast<float*>(smem + L.gpart);  // [2 row halves][16 vectors]
  float* ginv = gpart + 2 * 16;                               // [16] 1/gain, [16] flags
  const long lsc = blockIdx.x;
  const long sc = p.sc_base + lsc;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    const uint32_t zb = static_cast<uint32_t>(PrecodeQSmem::zbytes(St));
    const int row = static_cast<int>(sc * B);
    mbar_expect_tx(bar, static_cast<uint32_t>(B) * 128u + zb);
    bulk_g2s(smem + L.z, p.ws + lsc * W.stride + W.z, zb, bar);
    tma_load_2d(smem + L.h, &tmH, 0, row, bar);
    mbar_expect_tx(bar + 1, static_cast<uint32_t>(B) * 128u);
    tma_load_2d(smem + L.h + B * 128, &tmH, 32, row, bar + 1);
  }
  __syncthreads();  // barrier init visible
  const float2* Zs = reinterpret_cast<const float2*>(smem + L.z);
  const int tb = warp & 3, half = warp >> 2, rb = half * 32 + lane;
  for (int t0 = 0; t0 < St; t0 += 16) {
    const int nv = St - t0 < 16 ? St - t0 : 16;  // vectors of this pass
    unsigned long long qa[TR][TV], qb[TR][TV];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < TV; ++j) qa[r][j] = qb[r][j] = 0ull;
    // vectors past St read the pass's first one (results discarded)
    const float2* vb = Zs + (t0 + (tb * TV < nv ? tb * TV : 0)) * UP;
    const int vlast = nv - 1 - tb * TV;  // vectors j > vlast of this thread are past St
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      mbar_wait(bar + hh, 0);
      const unsigned char* ht = smem + L.h + hh * B * 128;
#pragma unroll 2
      for (int c = 0; c < 8; ++c) {
        ulonglong2 h[TR], v[TV];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
          const int row = rb + 64 * r;
          h[r] = *reinterpret_cast<const ulonglong2*>(ht + (row < B ? row : 0) * 128 + ((c ^ (row & 7)) << 4));
        }
        const int u = hh * 16 + 2 * c;
#pragma unroll
        for (int j = 0; j < TV; ++j)
          v[j] = *reinterpret_cast<const ulonglong2*>(vb + (j <= vlast ? j : 0) * UP + u);
#pragma unroll
        for (int r = 0; r < TR; ++r)
#pragma unroll
          for (int j = 0; j < TV; ++j) {
            ffma2(qa[r][j], h[r].x, f2dup_lo(v[j].x));
            ffma2(qb[r][j], h[r].x, f2dup_hi(v[j].x));
            ffma2(qa[r][j], h[r].y, f2dup_lo(v[j].y));
            ffma2(qb[r][j], h[r].y, f2dup_hi(v[j].y));
          }
      }
    }
    float2 q[TR][TV];
    float nrm[TV];
#pragma unroll
    for (int j = 0; j < TV; ++j) {
      nrm[j] = 0.f;
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        const float2 A = f2unpack(qa[r][j]), Bq = f2unpack(qb[r][j]);
        q[r][j] = make_float2(A.x - Bq.y, A.y + Bq.x);
        if (rb + 64 * r < B) nrm[j] += cnorm(q[r][j]);  // rows in a fixed order
      }
    }
    warp_sum4(nrm);
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < TV; ++j) gpart[half * 16 + tb * TV + j] = nrm[j];
    __syncthreads();
    if (tid < nv) {
      const int ts = t0 + tid;
      const float n2 = gpart[tid] + gpart[16 + tid];  // fixed order
      const bool ok = Zs[St * UP + ts].x == 0.f;
      const float g = sqrtf(n2);
      const bool zero = ok && !(g > 0.f);
      ginv[tid] = (ok && !zero) ? 1.f / g : 0.f;
      ginv[16 + tid] = ok ? 1.f : 0.f;
      if (p.gain) p.gain[sc * St + ts] = (ok && !zero) ? g : 0.f;
      if (p.pstatus) p.pstatus[sc * St + ts] = ok ? (zero ? 2 : 0) : 1;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TV; ++j) {
      const int t = tb * TV + j;
      if (t >= nv) continue;
      const float inv = ginv[t];
      const bool ok = ginv[16 + t] != 0.f;
      const long ob = (sc * St + t0 + t) * static_cast<long>(B);
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        const int row = rb + 64 * r;
        if (row >= B) continue;
        if (p.q) __stcs(p.q + ob + row, ok ? q[r][j] : make_float2(0.f, 0.f));
        if (p.s_out) __stcs(p.s_out + ob + row, cscale(inv, q[r][j]));
      }
    }
    __syncthreads();  // gpart / ginv reused by the next pass
  }
}

}  // namespace cgm
