// cgm_tc.cuh -- the channel kernel (K1) on the 5th-generation tensor cores.
//
// Per subcarrier, G = H^H H and the matched filter H^H Y are ONE real GEMM:
// with X = [H | Y] viewed as real numbers (row b = antenna, columns
// (u, re/im) then (s, re/im)), D = X_H^T X is a 64 x (64 + 2S) product over
// the B antennas and
//     G[u][j]  = (D[2u][2j]    + D[2u+1][2j+1],  D[2u][2j+1]    - D[2u+1][2j])
//     MF[u][s] = (D[2u][64+2s] + D[2u+1][65+2s], D[2u][65+2s]   - D[2u+1][64+2s]).
// Both operands are read straight from the natural [b][column] layout as
// MN-major SWIZZLE_128B tiles (no transpose).  FP32 accuracy from bf16
// tensor cores: every element is split x = p0 + p1 + p2 (three bf16 pieces,
// exact to 2^-27) and D = sum of the six products p_a p_b with a + b <= 2
// (the dropped terms are < 2^-24 relative).  The p0 p0 product accumulates
// in its own TMEM accumulator (K/16 steps), the five correction products in
// a second one; the epilogue adds them in round-to-nearest FP32.  Measured
// (tools/microbench/umma_probe.cu): error below an FP32 FMA chain; a single
// accumulator loses ~3 bits to the tensor core's truncating accumulation.
//
// Roles (one CTA per SM, persistent over subcarriers):
//   warp NWK     TMA producer: 64-antenna k-blocks of H and Y, bulk copies
//                into a staging ring (cp.async.bulk + mbarrier complete_tx)
//   warp NWK+1   MMA issuer (one thread): tcgen05.mma kind::f16 M=64,
//                N=64+ceil8(2S), 6 passes x 4 k-steps per k-block; commits
//                free the piece slot / publish the accumulator
//   warps 0..NWK-1  workers: split staging -> bf16 pieces (double-buffered
//                slots), then the epilogue of the previous subcarrier
//                (tcgen05.ld, G with an exact Hermitian mirror, MF)
// TMEM: 2 subcarrier buffers x {p0p0, corrections} x 128 columns = 512.
//
// Replaces gram_regularized (linalg.cpp:59-101) and matvec_adjoint
// (linalg.cpp:116-126) on the detect path (detect.cpp:188-196); writes the
// same workspace as channel_kernel, so solve_kernel is unchanged.
#pragma once

#include <cuda_bf16.h>

#include "cgm_split.cuh"

namespace cgm {
namespace tc {

constexpr int UPT = 32;            // users (M = 2U = 64 real rows)
constexpr int KB = 64;             // antennas per k-block
constexpr int ATOM = KB * 128;     // one SW128 column block: 64 rows x 64 bf16
constexpr int PIECE = 2 * ATOM;    // H columns (atom 0) + Y columns (atom 1)
constexpr int PSLOT = 3 * PIECE;   // the three bf16 pieces of one k-block
constexpr int NPS = 2;             // piece slots (max; RING of the kernel uses 1 or 2)
constexpr int TMEM_COLS = 512;     // 2 subcarrier buffers (RING = 2); RING = 1 uses 256
constexpr int GPS = UPT + 1;       // padded G row stride (float2) in smem
constexpr int MAX_STG = 4;

// ------------------------------------------------------------- tcgen05 PTX
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// arrives on `bar` once every previously issued MMA of this thread completed
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Shared-memory matrix descriptor: SWIZZLE_128B, LBO = stride between
// 64-column atoms (MN direction), SBO = stride between 8-row groups (K).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) |  // sm_100 version
         (2ull << 61);                                                          // SWIZZLE_128B
}
// Instruction descriptor: kind::f16 with bf16 A/B, FP32 D, both MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16_mn(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-uniform issue: the whole warp runs the issue loop (descriptors stay
// in uniform registers) and one elected lane executes the instruction --
// a single divergent thread needs ~2x the clocks per MMA to build and move
// its descriptors (tools/microbench/umma_probe.cu: 92.7 vs 48.2 clk for
// M64 x N96 x K16).
__device__ __forceinline__ void mma_bf16_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 TMEM lanes (this warp's quarter) x 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr)
      : "memory");
}
// 16x32bx2 shape for the M = 64 accumulator layout (rows in lanes 0-15 of
// each quarter): threads 0-15 read their row at columns [c, c+8), threads
// 16-31 the same rows at [c + off, c + off + 8).  `off` is an immediate.
template <int OFF>
__device__ __forceinline__ void tmem_ld8_x2_imm(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr), "n"(OFF)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8_x2(uint32_t taddr, int off, uint32_t (&v)[8]) {
  switch (off) {  // warp-uniform
    case 32: tmem_ld8_x2_imm<32>(taddr, v); break;
    case 40: tmem_ld8_x2_imm<40>(taddr, v); break;
    case 48: tmem_ld8_x2_imm<48>(taddr, v); break;
    case 56: tmem_ld8_x2_imm<56>(taddr, v); break;
    default: tmem_ld8_x2_imm<64>(taddr, v); break;
  }
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// x = p0 + p1 + p2 (bf16, round-to-nearest at each step; the differences
// are exact in FP32), 8 consecutive columns -> one 16-byte chunk per piece
__device__ __forceinline__ void split8(const float (&x)[8], uint4& o0, uint4& o1, uint4& o2) {
  uint32_t a[4], b[4], c[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(x[2 * t], x[2 * t + 1]);
    const float2 f0 = __bfloat1622float2(h0);
    const float r0 = __fsub_rn(x[2 * t], f0.x), r1 = __fsub_rn(x[2 * t + 1], f0.y);
    const __nv_bfloat162 h1 = __floats2bfloat162_rn(r0, r1);
    const float2 f1 = __bfloat1622float2(h1);
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(__fsub_rn(r0, f1.x), __fsub_rn(r1, f1.y));
    a[t] = *reinterpret_cast<const uint32_t*>(&h0);
    b[t] = *reinterpret_cast<const uint32_t*>(&h1);
    c[t] = *reinterpret_cast<const uint32_t*>(&h2);
  }
  o0 = make_uint4(a[0], a[1], a[2], a[3]);
  o1 = make_uint4(b[0], b[1], b[2], b[3]);
  o2 = make_uint4(c[0], c[1], c[2], c[3]);
}

// Shared-memory plan (offsets from a 1024-aligned base).
struct Smem {
  int pieces, stage, stage_bytes, nstg, gp, bar, total;
  __host__ __device__ static int align(int x, int a) { return (x + a - 1) / a * a; }
  // ring = piece slots and TMEM subcarrier buffers (2: one CTA per SM
  // double-buffers; 1: half the shared memory, two CTAs per SM)
  __host__ __device__ void plan(int S, int nstage, int ring = NPS) {
    int o = 0;
    pieces = o;
    o += ring * PSLOT;
    stage_bytes = align(KB * UPT * 8 + KB * S * 8, 128);
    nstg = nstage;
    stage = o;
    o += nstg * stage_bytes;
    gp = o;
    o = align(o + UPT * GPS * 8, 128);
    bar = o;
    o += 16 * 8 + 16 + 16;  // 16 mbarriers, TMEM base, misc
    total = align(o, 128) + 1024;  // + alignment slack of the dynamic base
  }
};

// True when the tensor-core kernel handles this problem (natural layout,
// U = 32, whole 64-antenna k-blocks, at most 32 vectors per subcarrier).
__host__ __device__ inline bool supported(int U, int B, int S, int use_tma) {
  return use_tma && U == UPT && B > 0 && (B % KB) == 0 && S >= 0 && 2 * S <= 64;
}

}  // namespace tc

// Warp roles.  NSP > 0 (specialised): [0, NEP) epilogue, [NEP, NEP+NSP)
// split.  NSP == 0 (unified): warps [0, NEP) split subcarrier i, then run
// the epilogue of subcarrier i-1 while the tensor core works on i.  Then
// the TMA producer warp and the MMA warp.  k1_pair carries the staging depth.
// 18 warps = 5 on two of the SM's four sub-partitions, each with a 16 K
// register file: 96 registers per thread is the most a CTA of this size can
// have (__maxnreg__(112) compiles without the specialised instantiation's
// 72 / 120 bytes of spills but cannot launch).
template <int NEP, int NSP, int RING = 2>
__global__ void __launch_bounds__(32 * (NEP + NSP + 2), 3 - RING) channel_tc_kernel(const KernelParams p) {
  using namespace tc;
  constexpr int UP = UPT;
  constexpr bool UNIFIED = NSP == 0;
  constexpr int NTE = 32 * NEP;                      // epilogue threads
  constexpr int NTS = 32 * (UNIFIED ? NEP : NSP);    // split threads
  constexpr int SPLIT0 = UNIFIED ? 0 : NEP;          // first split warp
  constexpr int WPROD = NEP + NSP, WMMA = NEP + NSP + 1;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  tc::Smem L;
  L.plan(p.S, p.k1_pair, RING);
  WsOffsets W;
  W.plan(UP, p.S, p.K, p.exact != 0, p.fx != 0, p.zs);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = p.S, B = p.B, nkb = B / KB, nstg = L.nstg;
  const int ny = S > 0 ? ((2 * S + 7) & ~7) : 0;  // Y columns fed to the MMA (zero padded)
  const int N = 64 + ny;
  const long n_local =
      p.n_sc > blockIdx.x ? (p.n_sc - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = bars + MAX_STG;
  uint64_t* pcs_full = bars + 2 * MAX_STG;
  uint64_t* pcs_empty = pcs_full + NPS;
  uint64_t* acc_full = pcs_empty + NPS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  constexpr uint32_t TCOLS = RING == 2 ? TMEM_COLS : 256;
  if (warp == 0) tmem_alloc(tmem_slot, TCOLS);
  if (tid == 0) {
    for (int s = 0; s < nstg; ++s) {
      mbar_init(stg_full + s, 1);
      mbar_init(stg_empty + s, NTS / 32);
    }
    for (int s = 0; s < NPS; ++s) {
      mbar_init(pcs_full + s, NTS / 32);
      mbar_init(pcs_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, NEP);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ------------------------------------------------ split of one subcarrier
  long pq = 0;        // piece-slot uses so far
  int stg_s = 0;      // staging slot
  uint32_t sph = 0;   // its phase parity
  auto split_sc = [&](long i) {
    const int st = tid - SPLIT0 * 32;  // 0 .. NTS-1
    const int nyc = ny / 8;            // Y chunks (8 columns) per antenna row
    int lg = 0;
    while ((1 << lg) < nyc) ++lg;
    constexpr int HPT = KB * 8 / NTS;  // H chunks per thread
    static_assert(KB * 8 % NTS == 0, "H chunks must divide evenly");
    for (int kb = 0; kb < nkb; ++kb, ++pq) {
      mbar_wait(stg_full + stg_s, sph);
      const int ps = static_cast<int>(pq % RING);
      if (pq >= RING) mbar_wait(pcs_empty + ps, static_cast<uint32_t>(((pq / RING) - 1) & 1));
      const float* Hst = reinterpret_cast<const float*>(smem + L.stage + stg_s * L.stage_bytes);
      const float* Yst = Hst + KB * UP * 2;
      unsigned char* slot = smem + L.pieces + ps * PSLOT;
      {
        // H: 64 rows x 8 chunks, Y: 64 rows x nyc chunks; a thread's chunks
        // are loaded together (latency overlap), then split
        // a thread's 32-byte chunk is two LDS.128; lanes 4-7 of every
        // 8-lane phase read the halves in the opposite order, so a phase
        // covers 8 distinct 16-byte bank groups (was 2-way conflicted)
        const bool hswap = (lane >> 2) & 1;
        float hx[HPT][8];
#pragma unroll
        for (int r = 0; r < HPT; ++r) {
          const int it = st + r * NTS, k = it >> 3, j = it & 7;
          const float* src = Hst + k * 64 + j * 8;
          const float4 a0 = *reinterpret_cast<const float4*>(src + (hswap ? 4 : 0));
          const float4 b0 = *reinterpret_cast<const float4*>(src + (hswap ? 0 : 4));
          const float4 a = hswap ? b0 : a0, b = hswap ? a0 : b0;
          hx[r][0] = a.x; hx[r][1] = a.y; hx[r][2] = a.z; hx[r][3] = a.w;
          hx[r][4] = b.x; hx[r][5] = b.y; hx[r][6] = b.z; hx[r][7] = b.w;
        }
        const int ycount = KB << lg;
        float yx[8];
        int yk = 0, yj = 0;
        const bool ylive = st < ycount && (st & ((1 << lg) - 1)) < nyc;
        if (ylive && nyc == 4 && (S & 1) == 0) {
          // 4 chunks per Y row (S = 13..16; 16-byte aligned rows for even S):
          // lanes 0-3 / 4-7 of a phase take rows r and r + 4 -- distinct
          // swizzled chunks for the piece stores (j ^ (k mod 8)) -- and read
          // their halves in opposite orders (distinct bank groups)
          const int t = st & 31;
          yk = (st >> 5) * 8 + 4 * ((t >> 2) & 1) + (t >> 3);
          yj = t & 3;
          const float* src = Yst + yk * 2 * S + yj * 8;
          const int c0 = yj * 8;
          float4 h0 = make_float4(0.f, 0.f, 0.f, 0.f), h1 = h0;
          if (hswap) {
            if (c0 + 4 < 2 * S) h1 = *reinterpret_cast<const float4*>(src + 4);
            h0 = *reinterpret_cast<const float4*>(src);
          } else {
            h0 = *reinterpret_cast<const float4*>(src);
            if (c0 + 4 < 2 * S) h1 = *reinterpret_cast<const float4*>(src + 4);
          }
          yx[0] = h0.x; yx[1] = h0.y; yx[2] = h0.z; yx[3] = h0.w;
          yx[4] = h1.x; yx[5] = h1.y; yx[6] = h1.z; yx[7] = h1.w;
        } else if (ylive) {
          yk = st >> lg;
          yj = st & ((1 << lg) - 1);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int col = yj * 8 + 2 * t;
            float2 v = make_float2(0.f, 0.f);
            if (col < 2 * S) v = *reinterpret_cast<const float2*>(Yst + yk * 2 * S + col);
            yx[2 * t] = v.x;
            yx[2 * t + 1] = v.y;
          }
        }
#pragma unroll
        for (int r = 0; r < HPT; ++r) {
          const int it = st + r * NTS, k = it >> 3, j = it & 7;
          uint4 o0, o1, o2;
          split8(hx[r], o0, o1, o2);
          const int off = k * 128 + ((j ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(slot + off) = o0;
          *reinterpret_cast<uint4*>(slot + PIECE + off) = o1;
          *reinterpret_cast<uint4*>(slot + 2 * PIECE + off) = o2;
        }
        if (ylive) {
          uint4 o0, o1, o2;
          split8(yx, o0, o1, o2);
          const int off = ATOM + yk * 128 + ((yj ^ (yk & 7)) << 4);
          *reinterpret_cast<uint4*>(slot + off) = o0;
          *reinterpret_cast<uint4*>(slot + PIECE + off) = o1;
          *reinterpret_cast<uint4*>(slot + 2 * PIECE + off) = o2;
        }
        for (int it = st + NTS; it < ycount; it += NTS) {  // more Y chunks than threads
          const int k = it >> lg, j = it & ((1 << lg) - 1);
          if (j >= nyc) continue;
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
          split8(x, o0, o1, o2);
          const int off = ATOM + k * 128 + ((j ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(slot + off) = o0;
          *reinterpret_cast<uint4*>(slot + PIECE + off) = o1;
          *reinterpret_cast<uint4*>(slot + 2 * PIECE + off) = o2;
        }
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
  };

  // ------------------------------------------------ epilogue of one subcarrier
  auto epilogue_sc = [&](long e) {
    float* Gpf = reinterpret_cast<float*>(smem + L.gp);  // [UP][GPS] float2 as floats
    // TMEM column split of the loads: lanes 0-15 read columns [0, hoff),
    // lanes 16-31 [hoff, 2 hoff) of the same accumulator rows
    const int hoff = (N / 2 + 7) & ~7;
    constexpr int CPW = 8 / (NEP / 4);            // max 8-column chunks per warp (hoff <= 64)
    constexpr int CB = CPW < 4 ? CPW : 4;         // chunks per batch of loads
    const int qd = warp & 3;                      // TMEM lane quarter of this warp
    const int m = qd * 16 + (lane & 15);          // accumulator row (M = 64 layout)
    const int u = m >> 1, odd = m & 1;            // user; re (even) / im (odd) row
    const int cbase = lane < 16 ? 0 : hoff;
    const int c_first = (warp >> 2) * 8, c_step = 8 * (NEP / 4);
    const int ab = static_cast<int>(e % RING);
    mbar_wait(acc_full + ab, static_cast<uint32_t>((e / RING) & 1));
    tc_fence_after();
    const long lsc = blockIdx.x + e * gridDim.x;
    float2* ws = p.ws + lsc * W.stride;
    float* mff = reinterpret_cast<float*>(ws + W.mf);
    const uint32_t tq = tmem + ab * 256 + (static_cast<uint32_t>(qd * 32) << 16);
    // TMEM loads in batches of up to 4 chunks (64 registers) in flight, one
    // wait per batch; the accumulator is released after the last batch
#pragma unroll
    for (int c00 = 0; c00 < CPW; c00 += CB) {
      uint32_t vb[CB][8], vs[CB][8];
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const int c0 = c_first + (c00 + c) * c_step;
        if (c0 < hoff) {
          tmem_ld8_x2(tq + c0, hoff, vb[c]);
          tmem_ld8_x2(tq + 128 + c0, hoff, vs[c]);
        }
      }
      tmem_wait_ld();
      if (c00 + CB >= CPW) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);  // accumulators may be overwritten
      }
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const int c0 = c_first + (c00 + c) * c_step;
        if (c0 >= hoff) continue;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float a = __fadd_rn(__uint_as_float(vb[c][2 * t]), __uint_as_float(vs[c][2 * t]));
          const float b =
              __fadd_rn(__uint_as_float(vb[c][2 * t + 1]), __uint_as_float(vs[c][2 * t + 1]));
          const float other = __shfl_xor_sync(0xffffffffu, b, 1);
          // even row 2u: re = D[2u][2j] + D[2u+1][2j+1]; odd row: im = D[2u][2j+1] - D[2u+1][2j]
          const float val = odd ? __fsub_rn(other, a) : __fadd_rn(a, other);
          const int j = (cbase + c0) / 2 + t;  // column pair
          if (j < UP)
            Gpf[(u * GPS + j) * 2 + odd] = val;  // full row; Hermitian fix-up below
          else if (j - UP < S)
            mff[((j - UP) * UP + u) * 2 + odd] = val;
        }
      }
    }
    named_sync(1, NTE);  // G rows complete in smem
    {
      // G = lower triangle + conjugate mirror, real diagonal (exactly Hermitian)
      const float2* Gp2 = reinterpret_cast<const float2*>(Gpf);
      float2* Gw = ws + W.g;
      for (int x = tid; x < UP * UP; x += NTE) {
        const int r = x >> 5, c = x & 31;
        float2 g = Gp2[(c < r ? r : c) * GPS + (c < r ? c : r)];
        if (c > r) g.y = -g.y;
        if (c == r) g.y = 0.f;
        Gw[x] = g;
      }
    }
  };

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
    // whole warp, warp-uniform control flow; one elected lane issues
    const uint32_t idesc = idesc_bf16_mn(64, N);
    const uint64_t dbase = smem_desc(smem_u32(smem + L.pieces), ATOM, 1024);
    long mq = 0;
    for (long i = 0; i < n_local; ++i) {
      const int ab = static_cast<int>(i % RING);
      if (i >= RING) mbar_wait(acc_empty + ab, static_cast<uint32_t>(((i / RING) - 1) & 1));
      tc_fence_after();
      const uint32_t d_big = tmem + ab * 256, d_small = d_big + 128;
      for (int kb = 0; kb < nkb; ++kb, ++mq) {
        const int ps = static_cast<int>(mq % RING);
        mbar_wait(pcs_full + ps, static_cast<uint32_t>((mq / RING) & 1));
        tc_fence_after();
        // descriptor start addresses advance by (byte offset >> 4)
        const uint64_t dslot = dbase + static_cast<uint64_t>((ps * PSLOT) >> 4);
        {
#pragma unroll
          for (int pass = 0; pass < 6; ++pass) {
            // (A piece, B piece) of the six products, p0 p0 first
            constexpr int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
            for (int ks = 0; ks < KB / 16; ++ks) {
              const uint64_t da = dslot + ((pa[pass] * PIECE + ks * 2048) >> 4);
              const uint64_t db = dslot + ((pb[pass] * PIECE + ks * 2048) >> 4);
              if (pass == 0)
                mma_bf16_elect(d_big, da, db, idesc, (kb | ks) ? 1u : 0u);
              else
                mma_bf16_elect(d_small, da, db, idesc, (pass > 1 || kb || ks) ? 1u : 0u);
            }
          }
        }
        tc_commit_elect(pcs_empty + ps);  // piece slot free once these MMAs retire
        __syncwarp();
      }
      tc_commit_elect(acc_full + ab);  // accumulators of subcarrier i complete
      __syncwarp();
    }
  } else if (UNIFIED) {
    // ------------------------------------------------------ unified workers
    for (long i = 0; i <= n_local; ++i) {
      if (i < n_local) split_sc(i);
      if (i > 0) epilogue_sc(i - 1);
    }
  } else if (warp >= NEP) {
    for (long i = 0; i < n_local; ++i) split_sc(i);
  } else {
    for (long e = 0; e < n_local; ++e) epilogue_sc(e);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TCOLS);
}

}  // namespace cgm
