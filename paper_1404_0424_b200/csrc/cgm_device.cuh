// cgm_device.cuh -- device helpers shared by the sm_100a kernels:
// complex64 arithmetic on float2, warp reductions, the TMA bulk-copy
// (cp.async.bulk + mbarrier complete_tx) used to stage each subcarrier's
// contiguous H / Y block into shared memory, and the 4x4 register-tiled
// "conj(X)^T Y" contraction that the Gram, matched filter and Chebyshev
// basis products are all built from.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cgm {

// ------------------------------------------------------------ complex64
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float s, float2 a) { return make_float2(s * a.x, s * a.y); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// Packed FP32x2 (FFMA2) helpers.  One complex MAC is two fma.rn.f32x2,
// (re, im) += (a.x, a.x) * (b.x, b.y) then (re, im) += (-a.y, a.y) * (b.y, b.x)
// -- the same per-component FMA order as four scalar fmaf (bitwise equal
// results) at half the instructions; the broadcast / swapped operands are
// free SASS operand selectors.  As a drop-in inside float2 loops the
// pack/unpack moves cost more than they save (measured), so cfma/cfma_conj
// stay scalar unless CGM_FFMA2_CFMA is defined; the CG kernel
// (cgm_solve32.cuh) keeps packed accumulators and uses ffma2 directly.
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a,
                                      unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
// lane swap / broadcast of a packed float pair (FFMA2 operand shuffles)
__device__ __forceinline__ unsigned long long f2swap_hl(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {hi, lo}; }" : "=l"(r) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long f2dup_lo(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {lo, lo}; }" : "=l"(r) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long f2dup_hi(unsigned long long v) {
  unsigned long long r;
  asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; mov.b64 %0, {hi, hi}; }" : "=l"(r) : "l"(v));
  return r;
}
// acc += a * b
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
#ifndef CGM_FFMA2_CFMA
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
#else
  unsigned long long c = f2pack(acc.x, acc.y);
  ffma2(c, f2pack(a.x, a.x), f2pack(b.x, b.y));
  ffma2(c, f2pack(-a.y, a.y), f2pack(b.y, b.x));
  acc = f2unpack(c);
#endif
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_conj(float2& acc, float2 a, float2 b) {
#ifndef CGM_FFMA2_CFMA
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
#else
  unsigned long long c = f2pack(acc.x, acc.y);
  ffma2(c, f2pack(a.x, a.x), f2pack(b.x, b.y));
  ffma2(c, f2pack(a.y, -a.y), f2pack(b.y, b.x));
  acc = f2unpack(c);
#endif
}
__device__ __forceinline__ float cnorm(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// ------------------------------------------------------------ reductions
// Sum over aligned groups of G lanes (G a power of two <= 32).
template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// Plain arrive (release at CTA scope): the consumer-side "slot free" /
// "data ready" signal of the producer/consumer rings.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier over a subset of warps (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One bulk global->shared copy (bytes % 16 == 0, both addresses 16B aligned)
// completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One 2-D TMA tensor tile (cp.async.bulk.tensor) global->shared through a
// tensor map (__grid_constant__ kernel parameter), completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 16-byte asynchronous global->shared copy (cp.async, L2-only), grouped by
// commit / wait_group: lets every thread place chunks at padded addresses
// (bank-conflict-free row strides) that one bulk copy cannot produce.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Order prior generic-proxy smem accesses before later async-proxy writes
// into the same buffer (buffer reuse across subcarriers).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------ 4x4 tile
// acc[r][c] += sum_{k in [k0,k1)} conj(X[k*ldx + i0 + r]) * Y(k, j0 + c)
// where Y(k, j) = Ys[k*yk + j*yj].  X rows are read as two float4 (i0 % 2 == 0
// and the row 16B aligned); columns of Y with j >= jmax read column jmax-1
// (results discarded by the caller).
template <bool Y_ROW_CONTIG>
__device__ __forceinline__ void tile4x4(float2 (&acc)[4][4], const float2* __restrict__ X, int ldx,
                                        int i0, const float2* __restrict__ Ys, int yk, int yj,
                                        int j0, int jmax, int k0, int k1) {
  int jc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) jc[c] = min(j0 + c, jmax - 1);
#pragma unroll 2
  for (int k = k0; k < k1; ++k) {
    const float4* xr = reinterpret_cast<const float4*>(X + k * ldx + i0);
    const float4 xa = xr[0], xb = xr[1];
    const float2 x[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w),
                         make_float2(xb.x, xb.y), make_float2(xb.z, xb.w)};
    float2 y[4];
    if (Y_ROW_CONTIG) {
      const float4* yr = reinterpret_cast<const float4*>(Ys + k * yk + j0);
      const float4 ya = yr[0], yb = yr[1];
      y[0] = make_float2(ya.x, ya.y);
      y[1] = make_float2(ya.z, ya.w);
      y[2] = make_float2(yb.x, yb.y);
      y[3] = make_float2(yb.z, yb.w);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) y[c] = Ys[k * yk + jc[c] * yj];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) cfma_conj(acc[r][c], x[r], y[c]);
  }
}

// Software-pipelined 4x4 tile: the operands of row k+1 are loaded before the
// 64 FFMAs of row k, so each warp keeps one LDS round trip in flight.
// acc[r][c] += sum_k conj(X[k*ldx + i0 + r]) * Z[k*ldz + j0 + c]; X and Z rows
// 16B aligned (Z columns past the valid range are read and discarded).
__device__ __forceinline__ void tile4x4_pipe(float2 (&acc)[4][4], const float2* __restrict__ X,
                                             int ldx, int i0, const float2* __restrict__ Z,
                                             int ldz, int j0, int k0, int k1) {
  const float4* xp = reinterpret_cast<const float4*>(X + k0 * ldx + i0);
  const float4* zp = reinterpret_cast<const float4*>(Z + k0 * ldz + j0);
  const int xs = ldx / 2, zs = ldz / 2;  // float4 strides
  // packed FP32x2 accumulators: conj(x) y = y * x.x + swap(y) * (x.y, -x.y),
  // the same two roundings per component in the same order as cfma_conj
  // (bitwise-equal results) at half the FMA-pipe instructions
  unsigned long long pk[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) pk[r][c] = f2pack(acc[r][c].x, acc[r][c].y);
  auto fma_row = [&](const float4& xa, const float4& xb, const float4& za, const float4& zb) {
    const float2 x[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w),
                         make_float2(xb.x, xb.y), make_float2(xb.z, xb.w)};
    const unsigned long long y[4] = {f2pack(za.x, za.y), f2pack(za.z, za.w), f2pack(zb.x, zb.y),
                                     f2pack(zb.z, zb.w)};
    unsigned long long ys[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) ys[c] = f2swap_hl(y[c]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const unsigned long long ax = f2pack(x[r].x, x[r].x), ay = f2pack(x[r].y, -x[r].y);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ffma2(pk[r][c], y[c], ax);
        ffma2(pk[r][c], ys[c], ay);
      }
    }
  };
  int k = k0;
  // two rows per trip: both rows' operands are in flight before the FMAs
  for (; k + 2 <= k1; k += 2) {
    const float4 xa0 = xp[0], xb0 = xp[1], za0 = zp[0], zb0 = zp[1];
    const float4 xa1 = xp[xs], xb1 = xp[xs + 1], za1 = zp[zs], zb1 = zp[zs + 1];
    xp += 2 * xs;
    zp += 2 * zs;
    fma_row(xa0, xb0, za0, zb0);
    fma_row(xa1, xb1, za1, zb1);
  }
  if (k < k1) fma_row(xp[0], xp[1], zp[0], zp[1]);
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = f2unpack(pk[r][c]);
}

// acc[r][c] += sum_k conj(X[k*ldx + i0 + r]) * Z[k*ldz + j0 + c], r, c < 2.
// X rows 16B aligned; Z rows 16B aligned when Z_VEC (else 2 scalar loads,
// columns >= jmax clamped).  Neighbouring lanes share either the X or the Z
// pair, so the loads are broadcasts or contiguous (no bank conflicts).
template <bool Z_VEC>
__device__ __forceinline__ void tile2x2(float2 (&acc)[2][2], const float2* __restrict__ X, int ldx,
                                        int i0, const float2* __restrict__ Z, int ldz, int j0,
                                        int jmax, int k0, int k1) {
  const int j1 = min(j0 + 1, jmax - 1);
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const float4 xa = *reinterpret_cast<const float4*>(X + k * ldx + i0);
    float4 za;
    if (Z_VEC) {
      za = *reinterpret_cast<const float4*>(Z + k * ldz + j0);
    } else {
      const float2 z0 = Z[k * ldz + j0], z1 = Z[k * ldz + j1];
      za = make_float4(z0.x, z0.y, z1.x, z1.y);
    }
    const float2 x0 = make_float2(xa.x, xa.y), x1 = make_float2(xa.z, xa.w);
    const float2 y0 = make_float2(za.x, za.y), y1 = make_float2(za.z, za.w);
    cfma_conj(acc[0][0], x0, y0);
    cfma_conj(acc[0][1], x0, y1);
    cfma_conj(acc[1][0], x1, y0);
    cfma_conj(acc[1][1], x1, y1);
  }
}

}  // namespace cgm
