// cgm_harness.cu -- the coded uplink BLER trial, restructured for the GPU
// (SURVEY.md section 8(f) rows 1-2).
//
// The reference's run_uplink_trial (sim.cpp:147-203) detects every
// (OFDM symbol, subcarrier) vector with its own detect_cg call and decodes on
// the CPU.  Here a batch of trials is one pipeline:
//   device per (trial, user) frame: info bits from Rng(key).fork(1).fork(u)
//          (sim.cpp:110-118), the rate-5/6 punctured K = 7 convolutional
//          code (each coded bit a parity of a 7-bit window: parallel) and the
//          Fisher-Yates interleaver from Rng(key).fork(4).fork(u) (sequential,
//          one thread per codeword) (coding.cpp:70-159, restated), Gray labels
//          (constellation.cpp:88-99);
//          Rayleigh channel per subcarrier from Rng(key).fork(2).fork(sc) and
//          y = H x + n with noise from Rng(key).fork(3).fork(sym*N_sc + sc)
//          (sim.cpp:162-180, channel.cpp:10-30); ONE batched detect_cg over
//          all subcarriers of all trials (S = OFDM symbols sharing H);
//          LLR stream -> deinterleave (coding.cpp:161-168); soft max-log
//          Viterbi, one warp per codeword, FP64 metrics with the reference's
//          tie rule (coding.cpp:100-147); block errors per trial.
// A trial whose detection breaks down is flagged and counts no errors, as
// the reference's early return (sim.cpp:183-188).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cgmimo_b200.h"
#include "cgm_rng.cuh"

struct cgm_ctx;
extern "C" int cgm_internal_fail(cgm_ctx* ctx, int code, const char* msg);
extern "C" int cgm_internal_device(cgm_ctx* ctx, void** stream, int* sms, long** launches);

namespace {

using namespace cgm_rng;

constexpr int kTail = 6;
constexpr unsigned kGenA = 0133, kGenB = 0171;
// puncturing keeps A at period steps 0,1,3 and B at 0,2,4 (coding.cpp:96-103)

__host__ __device__ __forceinline__ unsigned parity(unsigned w) {
#ifdef __CUDA_ARCH__
  return __popc(w) & 1u;
#else
  return __builtin_popcount(w) & 1u;
#endif
}

// ---------------------------------------------------------------- host side
struct Plan {
  int bps = 0, n_sym = 0;
  long coded = 0, info = 0;
};

// sim.cpp:38-51: the fewest OFDM symbols whose coded length is a multiple of 6
bool plan_frame(int n_sc, int bps, Plan& p) {
  p.bps = bps;
  for (int s = 1; s <= 6; ++s)
    if ((static_cast<long>(n_sc) * bps * s) % 6 == 0) {
      p.n_sym = s;
      break;
    }
  if (!p.n_sym) return false;
  p.coded = static_cast<long>(n_sc) * bps * p.n_sym;
  const long total = p.coded / 6 * 5;
  if (total <= kTail) return false;
  p.info = total - kTail;
  return true;
}

// ------------------------------------------------------------ device side
// H of every (trial, subcarrier): rayleigh_channel from Rng(key_t).fork(2).fork(sc)
__global__ void gen_channel_trials(float2* H, int B, int U, int n_sc, long n_tot,
                                   const uint64_t* keys) {
  const long per = static_cast<long>(B) * U;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < per * n_tot;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long g = idx / per, e = idx - g * per;
    const long t = g / n_sc, sc = g - t * n_sc;
    const uint64_t key = fork_key(fork_key(keys[t], 2), static_cast<uint64_t>(sc));
    const double2 v = gauss_pair(key, static_cast<uint64_t>(e), sqrt(0.5));
    H[idx] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

// y = H x + n per (trial, subcarrier, symbol); x from the frames' labels,
// n from Rng(key_t).fork(3).fork(sym * n_sc + sc) (sim.cpp:176-180)
__global__ void gen_received_trials(float2* Y, const float2* H, const uint8_t* labels, int B,
                                    int U, int n_sc, int S, int bits, double n0, long n_tot,
                                    const uint64_t* keys) {
  extern __shared__ double2 xs[];
  for (long inst = blockIdx.x; inst < n_tot * S; inst += gridDim.x) {
    const long g = inst / S;
    const int sym = static_cast<int>(inst - g * S);
    const long t = g / n_sc, sc = g - t * n_sc;
    for (int u = threadIdx.x; u < U; u += blockDim.x) xs[u] = qam_point(labels[inst * U + u], bits);
    __syncthreads();
    const uint64_t nk =
        fork_key(fork_key(keys[t], 3), static_cast<uint64_t>(sym) * n_sc + static_cast<uint64_t>(sc));
    const float2* h = H + g * static_cast<long>(B) * U;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      double re = 0.0, im = 0.0;
      for (int u = 0; u < U; ++u) {
        const float2 hv = h[b * U + u];
        re += static_cast<double>(hv.x) * xs[u].x - static_cast<double>(hv.y) * xs[u].y;
        im += static_cast<double>(hv.x) * xs[u].y + static_cast<double>(hv.y) * xs[u].x;
      }
      const double2 nz = gauss_pair(nk, static_cast<uint64_t>(b), sqrt(0.5 * n0));
      Y[(g * B + b) * S + sym] = make_float2(static_cast<float>(re + nz.x), static_cast<float>(im + nz.y));
    }
    __syncthreads();
  }
}

// Downlink transmit vectors t of every (trial, subcarrier, symbol): the
// frames' constellation points (sim.cpp:233-236), T layout [g][sym][u]
__global__ void gen_transmit_trials(float2* T, const uint8_t* labels, int bits, long n) {
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const double2 x = qam_point(labels[idx], bits);
    T[idx] = make_float2(static_cast<float>(x.x), static_cast<float>(x.y));
  }
}

// detect::compute_llrs (detect.cpp:57-86) in FP64 for the downlink genie
// demapper: z = xhat / mu, I-axis bits then Q-axis bits, per axis bit p the
// nearest amplitude with bit p = 0 vs 1, rho * (d0 - d1), clip +-64
__device__ void llrs_fp64(double zr, double zi, double rho, int bits, float* out) {
  const int half = bits / 2;
  const unsigned levels = 1u << half;
  const double scale = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
  if (rho < 0.0) rho = 0.0;
  for (int axis = 0; axis < 2; ++axis) {
    const double z = axis == 0 ? zr : zi;
    for (int p = 0; p < half; ++p) {
      double d0 = INFINITY, d1 = INFINITY;
      for (unsigned g = 0; g < levels; ++g) {
        const double amp = (2.0 * gray_decode(g) - (levels - 1.0)) * scale;
        const double d = (z - amp) * (z - amp);
        if ((g >> (half - 1 - p)) & 1u) d1 = d < d1 ? d : d1;
        else d0 = d < d0 ? d : d0;
      }
      double v = rho * (d0 - d1);
      v = v < -64.0 ? -64.0 : (v > 64.0 ? 64.0 : v);
      out[axis * half + p] = static_cast<float>(v);
    }
  }
}

// Downlink receive side of run_downlink_trial (sim.cpp:248-266): z = H_d s
// with H_d = H^H, y_u = z_u + n_u (n_u = next_gaussian pair u of
// Rng(key_t).fork(3).fork(sym * n_sc + sc)), genie gain z_u / t_u, LLRs of
// y_u / gain at rho = |gain|^2 / N0, zeros below |gain|^2 < 1e-24.
__global__ void downlink_receive(float* llr, const float2* H, const float2* Sx,
                                 const uint8_t* labels, int B, int U, int n_sc, int S, int bits,
                                 double n0, long n_tot, const uint64_t* keys) {
  extern __shared__ double2 sv[];
  const double sd = sqrt(0.5 * n0);
  for (long inst = blockIdx.x; inst < n_tot * S; inst += gridDim.x) {
    const long g = inst / S;
    const int sym = static_cast<int>(inst - g * S);
    const long t = g / n_sc, sc = g - t * n_sc;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const float2 v = Sx[inst * B + b];
      sv[b] = make_double2(v.x, v.y);
    }
    __syncthreads();
    const uint64_t nk =
        fork_key(fork_key(keys[t], 3), static_cast<uint64_t>(sym) * n_sc + static_cast<uint64_t>(sc));
    const float2* h = H + g * static_cast<long>(B) * U;
    for (int u = threadIdx.x; u < U; u += blockDim.x) {
      double zr = 0.0, zi = 0.0;  // sum_b conj(H[b][u]) s_b
      for (int b = 0; b < B; ++b) {
        const float2 hv = h[b * U + u];
        zr += static_cast<double>(hv.x) * sv[b].x + static_cast<double>(hv.y) * sv[b].y;
        zi += static_cast<double>(hv.x) * sv[b].y - static_cast<double>(hv.y) * sv[b].x;
      }
      // cplx(sd * g(), sd * g()) at sim.cpp:252: the two draws are unsequenced
      // constructor arguments; g++ (the reference's compiler) evaluates them
      // right to left, so the real part gets the pair's SECOND variate
      const double2 nz = gauss_pair(nk, static_cast<uint64_t>(u), sd);
      const double yr = zr + nz.y, yi = zi + nz.x;
      const double2 x = qam_point(labels[inst * U + u], bits);
      const double xn = x.x * x.x + x.y * x.y;  // gain = z / t
      const double gr = (zr * x.x + zi * x.y) / xn, gi = (zi * x.x - zr * x.y) / xn;
      const double g2 = gr * gr + gi * gi;
      float* o = llr + inst * static_cast<long>(U) * bits + u * bits;
      if (g2 < 1e-24) {
        for (int b = 0; b < bits; ++b) o[b] = 0.f;
      } else {  // y / gain
        const double qr = (yr * gr + yi * gi) / g2, qi = (yi * gr - yr * gi) / g2;
        llrs_fp64(qr, qi, g2 / n0, bits, o);
      }
    }
    __syncthreads();
  }
}

// LLR stream of user u (index (sym * n_sc + sc) * bps + b, sim.cpp:194-196)
// -> coded-bit order through the interleaver (coding.cpp:161-168)
__global__ void deinterleave_llrs(double* coded, const float* llr, const int32_t* perm, int U,
                                  int n_sc, int S, int bps, long coded_len, long n_cw) {
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < n_cw * coded_len;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long cw = idx / coded_len, j = idx - cw * coded_len;
    const long t = cw / U;
    const int u = static_cast<int>(cw - t * U);
    const long sidx = j / bps;
    const int b = static_cast<int>(j - sidx * bps);
    const long sym = sidx / n_sc, sc = sidx - sym * n_sc;
    const long g = t * n_sc + sc;
    const float v = llr[((g * S + sym) * U + u) * bps + b];
    coded[cw * coded_len + perm[cw * coded_len + j]] = static_cast<double>(v);
  }
}

// ---- frames on the device (sim.cpp:110-118, coding.cpp:70-159)
// info bit i of codeword (t, u): Rng(key_t).fork(1).fork(u).next_u64() & 1
__global__ void frame_info(uint8_t* info, long info_len, int U, long n_cw, const uint64_t* keys) {
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < n_cw * info_len;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long cw = idx / info_len, i = idx - cw * info_len;
    const long t = cw / U;
    const uint64_t bk = fork_key(fork_key(keys[t], 1), static_cast<uint64_t>(cw - t * U));
    info[idx] = static_cast<uint8_t>(draw(bk, static_cast<uint64_t>(i) + 1) & 1u);
  }
}

// Fisher-Yates of codeword (t, u) with Rng(key_t).fork(4).fork(u).next_unit
// (coding.cpp:149-157): sequential per codeword, one thread each.  The swap
// chain is latency bound, so the permutation lives in shared memory (16-bit
// entries, `per` codewords per block) and is copied out once at the end.
__global__ void frame_perm(int32_t* perm, long n, int U, long n_cw, int per, const uint64_t* keys) {
  extern __shared__ uint16_t ps[];
  const long cw0 = blockIdx.x * static_cast<long>(per);
  const int nloc = static_cast<int>(n_cw - cw0 < per ? n_cw - cw0 : per);
  for (long i = threadIdx.x; i < nloc * n; i += blockDim.x) ps[i] = static_cast<uint16_t>(i % n);
  __syncthreads();
  if (threadIdx.x < nloc) {
    const long cw = cw0 + threadIdx.x;
    const long t = cw / U;
    const uint64_t key = fork_key(fork_key(keys[t], 4), static_cast<uint64_t>(cw - t * U));
    uint16_t* p = ps + threadIdx.x * n;
    uint64_t ctr = 0;
    for (long i = n; i-- > 1;) {
      const double un = unit(draw(key, ++ctr));
      long j = static_cast<long>(un * static_cast<double>(i + 1));
      if (j > i) j = i;
      const uint16_t a = p[i];
      p[i] = p[j];
      p[j] = a;
    }
  }
  __syncthreads();
  for (long i = threadIdx.x; i < nloc * n; i += blockDim.x) perm[cw0 * n + i] = ps[i];
}

// The same without the 16-bit / shared-memory limits (long frames)
__global__ void frame_perm_global(int32_t* perm, long n, int U, long n_cw, const uint64_t* keys) {
  const long cw = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (cw >= n_cw) return;
  const long t = cw / U;
  const uint64_t key = fork_key(fork_key(keys[t], 4), static_cast<uint64_t>(cw - t * U));
  int32_t* p = perm + cw * n;
  for (long i = 0; i < n; ++i) p[i] = static_cast<int32_t>(i);
  uint64_t ctr = 0;
  for (long i = n; i-- > 1;) {
    const double un = unit(draw(key, ++ctr));
    long j = static_cast<long>(un * static_cast<double>(i + 1));
    if (j > i) j = i;
    const int32_t a = p[i];
    p[i] = p[j];
    p[j] = a;
  }
}

// coded bit c of a codeword (the 6 punctured bits of a 5-step period are
// t0A t0B t1A t2B t3A t4B): parity of the generator over the 7-bit window
// (u_t, u_{t-1}, ..., u_{t-6}); tail and t < 0 inputs are 0
__device__ __forceinline__ unsigned coded_bit(const uint8_t* in, long info_len, long c) {
  const long p = c / 6;
  const int r = static_cast<int>(c - p * 6);
  const int dt = r == 0 ? 0 : r - 1;
  const long t = p * 5 + dt;
  unsigned word = 0;
#pragma unroll
  for (int k = 0; k <= kTail; ++k) {
    const long tk = t - k;
    const unsigned bit = (tk >= 0 && tk < info_len) ? (in[tk] & 1u) : 0u;
    word |= bit << (kTail - k);
  }
  const bool stream_b = (r == 1) || (r == 3) || (r == 5);
  return parity(word & (stream_b ? kGenB : kGenA));
}

// Gray label of symbol sidx of codeword (t, u): interleaved bits
// [sidx*bps, +bps) = coded[perm[...]], MSB first (constellation.cpp:88-99)
__global__ void frame_labels(uint8_t* labels, const uint8_t* info, const int32_t* perm,
                             long info_len, long coded_len, int bps, int n_sc, int S, int U,
                             long n_cw) {
  const long n_sym_cw = coded_len / bps;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < n_cw * n_sym_cw;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long cw = idx / n_sym_cw, sidx = idx - cw * n_sym_cw;
    const long t = cw / U;
    const int u = static_cast<int>(cw - t * U);
    const uint8_t* in = info + cw * info_len;
    const int32_t* pm = perm + cw * coded_len;
    unsigned lab = 0;
    for (int b = 0; b < bps; ++b) lab = (lab << 1) | coded_bit(in, info_len, pm[sidx * bps + b]);
    const long sym = sidx / n_sc, sc = sidx - sym * n_sc;
    labels[((t * n_sc + sc) * S + sym) * U + u] = static_cast<uint8_t>(lab);
  }
}

// Soft max-log Viterbi (coding.cpp:90-147), one warp per codeword.  Lane k
// owns next states k (input 0) and k + 32 (input 1); both are reached from
// states 2k and 2k+1.  FP64 path metrics; ties keep the lower predecessor
// (the reference visits states in ascending order with a strict '>').
// The add-compare-select chain is latency bound, so nothing else sits on it:
// the punctured LLRs of the next 32 periods (192 doubles) are loaded into
// registers one chunk ahead and staged through shared memory; the decision
// words of 32 steps (two 32-bit ballots per step: which predecessor) are held
// one per lane and written as one coalesced 256-byte store.  Traceback from
// the terminated all-zero state walks 32 steps at a time through shuffles of
// a prefetched block of decision words; the decoded bits come out one per
// lane, so the comparison with the info bits is coalesced too.
constexpr int kVitWarps = 4;
constexpr int kChunkPeriods = 32;                 // 160 trellis steps
constexpr int kChunkLlrs = kChunkPeriods * 6;     // 192 doubles, 6 per lane

__global__ void __launch_bounds__(32 * kVitWarps) viterbi_decode(
    const double* coded, const uint8_t* info, uint2* dec, uint8_t* err, uint8_t* out,
    long coded_len, long info_len, long n_cw) {
  __shared__ double stage[kVitWarps][kChunkLlrs];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long cw = blockIdx.x * static_cast<long>(kVitWarps) + wib;
  if (cw >= n_cw) return;
  const long total = info_len + kTail;  // = 5 * coded_len / 6
  const long n_periods = coded_len / 6;
  const double* L = coded + cw * coded_len;
  uint2* D = dec + cw * total;
  double* sl = stage[wib];
  // branch metric of (pred 2k+q, input u) = (+-la) + (+-lb) with the signs of
  // its output bits (a, b) -- the reference's bm[(a << 1) | b] table
  // (coding.cpp:114-116) -- formed as fma(lb, sb, la * sa): the product by
  // +-1 is exact, so it rounds once, exactly like the table's addition.  (An
  // indexed bm[4] table would live in local memory: lane-dependent index.)
  double sa[2][2], sb[2][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned word = (static_cast<unsigned>(u) << kTail) | static_cast<unsigned>(2 * lane + q);
      sa[q][u] = parity(word & kGenA) ? 1.0 : -1.0;
      sb[q][u] = parity(word & kGenB) ? 1.0 : -1.0;
    }
  const double ninf = -static_cast<double>(INFINITY);
  double m0 = lane == 0 ? 0.0 : ninf;  // state lane
  double m1 = ninf;                    // state lane + 32
  const int src0 = (2 * lane) & 31, src1 = (2 * lane + 1) & 31;
  const bool upper = lane >= 16;
  double pre[6];
  auto fetch = [&](long chunk) {
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      const long i = chunk * kChunkLlrs + r * 32 + lane;
      pre[r] = i < coded_len ? L[i] : 0.0;
    }
  };
  fetch(0);
  uint2 mine = make_uint2(0u, 0u);
  for (long p = 0; p < n_periods; ++p) {
    const int pc = static_cast<int>(p % kChunkPeriods);
    if (pc == 0) {  // stage this chunk, prefetch the next
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 6; ++r) sl[r * 32 + lane] = pre[r];
      __syncwarp();
      fetch(p / kChunkPeriods + 1);
    }
    const double* q = sl + pc * 6;
    // punctured positions inside a period: A at 0,2,4 (steps 0,1,3); B at
    // 1,3,5 (steps 0,2,4) (coding.cpp:96-103)
    const double lv[6] = {q[0], q[1], q[2], q[3], q[4], q[5]};
#pragma unroll
    for (int ph = 0; ph < 5; ++ph) {
      const long tt = p * 5 + ph;
      constexpr int offA[5] = {0, 2, -1, 4, -1};
      constexpr int offB[5] = {1, -1, 3, -1, 5};
      const double la = offA[ph] >= 0 ? lv[offA[ph] < 0 ? 0 : offA[ph]] : 0.0;
      const double lb = offB[ph] >= 0 ? lv[offB[ph] < 0 ? 0 : offB[ph]] : 0.0;
      // metrics of states 2k and 2k+1 (lane (2k)&31, half (2k)>>5)
      const double a0 = __shfl_sync(0xffffffffu, m0, src0), a1 = __shfl_sync(0xffffffffu, m1, src0);
      const double b0 = __shfl_sync(0xffffffffu, m0, src1), b1 = __shfl_sync(0xffffffffu, m1, src1);
      const double p0 = upper ? a1 : a0, p1 = upper ? b1 : b0;
      const double bm00 = fma(lb, sb[0][0], la * sa[0][0]), bm10 = fma(lb, sb[1][0], la * sa[1][0]);
      const double bm01 = fma(lb, sb[0][1], la * sa[0][1]), bm11 = fma(lb, sb[1][1], la * sa[1][1]);
      const double c00 = p0 + bm00, c10 = p1 + bm10;
      const bool d0 = c10 > c00;
      const double n0 = d0 ? c10 : c00;
      // next state lane + 32 (input 1) is not reachable in the tail
      const double c01 = p0 + bm01, c11 = p1 + bm11;
      const bool d1 = c11 > c01;
      const double n1 = tt < info_len ? (d1 ? c11 : c01) : ninf;
      const unsigned w0 = __ballot_sync(0xffffffffu, d0), w1 = __ballot_sync(0xffffffffu, d1);
      const int slot = static_cast<int>(tt & 31);
      if (lane == slot) mine = make_uint2(w0, w1);
      if (slot == 31 || tt == total - 1) {
        const long i = (tt & ~31L) + lane;
        if (i <= tt) D[i] = mine;
      }
      m0 = n0;
      m1 = n1;
    }
  }
  __syncwarp();
  // traceback, 32 steps per block, next block's words prefetched
  const long nblk = (total + 31) / 32;
  unsigned state = 0;
  bool bad = false;
  uint2 cur = (nblk - 1) * 32 + lane < total ? D[(nblk - 1) * 32 + lane] : make_uint2(0u, 0u);
  for (long blk = nblk - 1; blk >= 0; --blk) {
    const uint2 nxt = blk > 0 ? D[(blk - 1) * 32 + lane] : make_uint2(0u, 0u);
    const int top = static_cast<int>(total - 1 - blk * 32 < 31 ? total - 1 - blk * 32 : 31);
    unsigned myu = 0;
    for (int j = top; j >= 0; --j) {
      const unsigned w = __shfl_sync(0xffffffffu, (state >> 5) ? cur.y : cur.x, j);
      const unsigned pick = (w >> (state & 31)) & 1u;
      if (lane == j) myu = state >> 5;
      state = ((state & 31u) << 1) | pick;
    }
    const long tt = blk * 32 + lane;
    if (tt < info_len) {
      if (info) bad |= myu != (info[cw * info_len + tt] & 1u);
      if (out) out[cw * info_len + tt] = static_cast<uint8_t>(myu);
    }
    cur = nxt;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (err && lane == 0) err[cw] = bad ? 1 : 0;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// run_uplink_trial / run_downlink_trial (sim.cpp:147-275) for a batch of trials
int run_trials(cgm_ctx* ctx, bool downlink, int method, int B, int U, int n_sc, int qam_bits,
               int K, int tracker, double snr_db, long n_trials, const uint64_t* trial_keys,
               uint32_t* user_errors, uint8_t* breakdown) {
  const char* who = downlink ? "cgm_downlink_trials" : "cgm_uplink_trials";
  void* stv = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &stv, &sms, &launches)) return CGM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stv);
  if (B < 1 || U < 1 || U > B || n_sc < 1 || n_trials < 0 || !trial_keys || !user_errors ||
      (qam_bits != 2 && qam_bits != 4 && qam_bits != 6))
    return cgm_internal_fail(ctx, CGM_EINVAL, (std::string(who) + ": bad arguments").c_str());
  if (n_trials == 0) return CGM_OK;
  // CGMIMO_HARNESS_TIMING=1: phase timings on stderr (pipeline study)
  const bool timing = std::getenv("CGMIMO_HARNESS_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_start = now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(st);
    const auto t = now();
    std::fprintf(stderr, "harness %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_start).count());
    t_start = t;
  };
  Plan pl;
  if (!plan_frame(n_sc, qam_bits, pl))
    return cgm_internal_fail(ctx, CGM_EINVAL, (std::string(who) + ": frame does not fit the code").c_str());
  const int S = pl.n_sym, bps = pl.bps;
  // channel.cpp:44-52: N0 = U / SNR uplink (per receive antenna), 1 / SNR downlink
  const double n0 = (downlink ? 1.0 : static_cast<double>(U)) / std::pow(10.0, snr_db / 10.0);
  const long n_tot = n_trials * n_sc, n_cw = n_trials * U;
  // ---- device buffers (stream-ordered: the pool keeps them across calls)
  const long total_steps = pl.info + kTail;
  void *dH = nullptr, *dY = nullptr, *dLab = nullptr, *dLlr = nullptr, *dSt = nullptr,
       *dKeys = nullptr, *dInfo = nullptr, *dPerm = nullptr, *dCoded = nullptr, *dDec = nullptr,
       *dErr = nullptr, *dT = nullptr;
  auto cleanup = [&] {
    for (void* q : {dH, dY, dLab, dLlr, dSt, dKeys, dInfo, dPerm, dCoded, dDec, dErr, dT})
      if (q) cudaFreeAsync(q, st);
  };
  cudaError_t e = cudaSuccess;
  {  // keep freed blocks in the stream-ordered pool between sweep batches
    // (the default threshold 0 hands them back to the driver at every sync)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 8ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  auto A = [&](void** q, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(q, bytes > 0 ? bytes : 16, st);
  };
  A(&dH, static_cast<size_t>(n_tot) * B * U * 8);
  A(&dY, static_cast<size_t>(n_tot) * B * S * 8);
  A(&dLab, static_cast<size_t>(n_tot) * S * U);
  A(&dLlr, static_cast<size_t>(n_tot) * S * U * bps * 4);
  A(&dSt, static_cast<size_t>(n_tot) * S);
  A(&dKeys, static_cast<size_t>(n_trials) * 8);
  A(&dInfo, static_cast<size_t>(n_cw) * pl.info);
  A(&dPerm, static_cast<size_t>(n_cw) * pl.coded * 4);
  A(&dCoded, static_cast<size_t>(n_cw) * pl.coded * 8);
  A(&dDec, static_cast<size_t>(n_cw) * total_steps * 8);
  A(&dErr, static_cast<size_t>(n_cw));
  if (downlink) A(&dT, static_cast<size_t>(n_tot) * S * U * 8);
  if (e != cudaSuccess) {
    cleanup();
    return cgm_internal_fail(ctx, CGM_ENOMEM, (std::string(who) + ": device allocation").c_str());
  }
  cudaMemcpyAsync(dKeys, trial_keys, static_cast<size_t>(n_trials) * 8, cudaMemcpyHostToDevice, st);
  mark("alloc+keys");
  auto grid = [&](long work) {
    return static_cast<unsigned>(std::max<long>(1, std::min<long>((work + 255) / 256, 32L * sms)));
  };
  // ---- frames on the device
  frame_info<<<grid(n_cw * pl.info), 256, 0, st>>>(static_cast<uint8_t*>(dInfo), pl.info, U, n_cw,
                                                  static_cast<uint64_t*>(dKeys));
  {
    // codewords per block: spread over the SMs, within 220 KB of 16-bit entries
    const long fit = (220L * 1024) / (pl.coded * 2);
    const long per = std::min<long>({32L, fit, (n_cw + sms - 1) / sms});
    if (pl.coded <= 65536 && per >= 1) {
      const size_t sm = static_cast<size_t>(per * pl.coded * 2);
      cudaFuncSetAttribute(frame_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
      frame_perm<<<static_cast<unsigned>((n_cw + per - 1) / per), 128, sm, st>>>(
          static_cast<int32_t*>(dPerm), pl.coded, U, n_cw, static_cast<int>(per),
          static_cast<uint64_t*>(dKeys));
    } else {
      frame_perm_global<<<static_cast<unsigned>((n_cw + 31) / 32), 32, 0, st>>>(
          static_cast<int32_t*>(dPerm), pl.coded, U, n_cw, static_cast<uint64_t*>(dKeys));
    }
  }
  frame_labels<<<grid(n_cw * (pl.coded / bps)), 256, 0, st>>>(
      static_cast<uint8_t*>(dLab), static_cast<uint8_t*>(dInfo), static_cast<int32_t*>(dPerm),
      pl.info, pl.coded, bps, n_sc, S, U, n_cw);
  *launches += 3;
  mark("frames");
  gen_channel_trials<<<grid(n_tot * B * U), 256, 0, st>>>(static_cast<float2*>(dH), B, U, n_sc,
                                                         n_tot, static_cast<uint64_t*>(dKeys));
  int rc = CGM_OK;
  if (!downlink) {
    gen_received_trials<<<static_cast<unsigned>(std::min<long>(n_tot * S, 32L * sms)), 128,
                          U * sizeof(double2), st>>>(
        static_cast<float2*>(dY), static_cast<float2*>(dH), static_cast<uint8_t*>(dLab), B, U, n_sc,
        S, bps, n0, n_tot, static_cast<uint64_t*>(dKeys));
    *launches += 2;
    e = cudaGetLastError();
    mark("channel+y");
    // ---- ONE batched detection over every subcarrier of every trial
    if (e == cudaSuccess)
      rc = cgm_detect(ctx, method, B, U, n_tot, S, static_cast<float*>(dH), static_cast<float*>(dY),
                      1.0 / n0, n0, 1.0, qam_bits, K, tracker, nullptr, nullptr, nullptr,
                      static_cast<float*>(dLlr), static_cast<uint8_t*>(dSt), CGM_DEVICE_POINTERS);
  } else {
    gen_transmit_trials<<<grid(n_tot * S * U), 256, 0, st>>>(
        static_cast<float2*>(dT), static_cast<uint8_t*>(dLab), bps, n_tot * S * U);
    *launches += 2;
    e = cudaGetLastError();
    mark("channel+t");
    // ---- ONE batched precode over every (symbol, subcarrier) of every
    // trial; H_d = H^H from the uplink-layout draws (sim.cpp:223); the
    // transmit vectors s land in dY (same size)
    if (e == cudaSuccess)
      rc = cgm_precode(ctx, method, B, U, n_tot, S, static_cast<float*>(dH), static_cast<float*>(dT),
                       1.0 / n0, K, nullptr, static_cast<float*>(dY), nullptr,
                       static_cast<uint8_t*>(dSt), CGM_DEVICE_POINTERS | CGM_HD_UPLINK_LAYOUT);
    if (rc == CGM_OK) {
      downlink_receive<<<static_cast<unsigned>(std::min<long>(n_tot * S, 32L * sms)), 64,
                         B * sizeof(double2), st>>>(
          static_cast<float*>(dLlr), static_cast<float2*>(dH), static_cast<float2*>(dY),
          static_cast<uint8_t*>(dLab), B, U, n_sc, S, bps, n0, n_tot, static_cast<uint64_t*>(dKeys));
      ++*launches;
      e = cudaGetLastError();
    }
  }
  mark("detect");
  if (e == cudaSuccess && rc == CGM_OK) {
    deinterleave_llrs<<<grid(n_cw * pl.coded), 256, 0, st>>>(
        static_cast<double*>(dCoded), static_cast<float*>(dLlr), static_cast<int32_t*>(dPerm), U,
        n_sc, S, bps, pl.coded, n_cw);
    viterbi_decode<<<static_cast<unsigned>((n_cw + kVitWarps - 1) / kVitWarps), 32 * kVitWarps, 0, st>>>(
        static_cast<double*>(dCoded), static_cast<uint8_t*>(dInfo), static_cast<uint2*>(dDec),
        static_cast<uint8_t*>(dErr), nullptr, pl.coded, pl.info, n_cw);
    *launches += 2;
    e = cudaGetLastError();
  }
  mark("decode");
  std::vector<uint8_t> errs(static_cast<size_t>(n_cw)), stat(static_cast<size_t>(n_tot * S));
  if (e == cudaSuccess && rc == CGM_OK) {
    e = cudaMemcpyAsync(errs.data(), dErr, errs.size(), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(stat.data(), dSt, stat.size(), cudaMemcpyDeviceToHost, st);
  }
  cleanup();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  mark("d2h+free");
  if (rc != CGM_OK) return rc;
  if (e != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, cudaGetErrorString(e));
  for (uint8_t v : stat)
    if (v & 4u)  // NotPositiveDefinite / domain_error propagate out of run_point in the reference
      return cgm_internal_fail(ctx, CGM_EINVAL, (std::string(who) + ": solver input not positive definite").c_str());
  for (long t = 0; t < n_trials; ++t) {
    bool broke = false;
    for (long i = t * n_sc * S; i < (t + 1) * n_sc * S; ++i) broke |= (stat[i] & 1u) != 0;
    uint32_t ue = 0;
    for (int u = 0; u < U; ++u) ue += errs[t * U + u];
    user_errors[t] = broke ? 0u : ue;
    if (breakdown) breakdown[t] = broke ? 1 : 0;
  }
  return CGM_OK;
}

}  // namespace

extern "C" {

int cgm_uplink_trials(cgm_ctx* ctx, int B, int U, int n_sc, int qam_bits, int K, int tracker,
                      double snr_db, long n_trials, const uint64_t* trial_keys,
                      uint32_t* user_errors, uint8_t* breakdown) {
  return run_trials(ctx, false, CGM_METHOD_CG, B, U, n_sc, qam_bits, K, tracker, snr_db, n_trials,
                    trial_keys, user_errors, breakdown);
}

int cgm_sweep_trials(cgm_ctx* ctx, int direction, int method, int B, int U, int n_sc,
                     int qam_bits, int iters, int tracker, double snr_db, long n_trials,
                     const uint64_t* trial_keys, uint32_t* user_errors, uint8_t* breakdown) {
  if (direction != 1 && direction != 2)
    return cgm_internal_fail(ctx, CGM_EINVAL, "cgm_sweep_trials: direction must be 1 (uplink) or 2 (downlink)");
  if (method < CGM_METHOD_CHOLESKY || method > CGM_METHOD_NEUMANN)
    return cgm_internal_fail(ctx, CGM_EINVAL, "cgm_sweep_trials: unknown method");
  return run_trials(ctx, direction == 2, method, B, U, n_sc, qam_bits, iters,
                    direction == 2 ? CGM_TRACKER_APPROX : tracker, snr_db, n_trials, trial_keys,
                    user_errors, breakdown);
}

int cgm_downlink_trials(cgm_ctx* ctx, int B, int U, int n_sc, int qam_bits, int K,
                        double snr_db, long n_trials, const uint64_t* trial_keys,
                        uint32_t* user_errors, uint8_t* breakdown) {
  return run_trials(ctx, true, CGM_METHOD_CG, B, U, n_sc, qam_bits, K, CGM_TRACKER_APPROX, snr_db,
                    n_trials, trial_keys, user_errors, breakdown);
}

int cgm_viterbi_decode(cgm_ctx* ctx, const double* llrs, long coded_len, long n_cw,
                       uint8_t* info_out) {
  void* stv = nullptr;
  int sms = 0;
  long* launches = nullptr;
  if (cgm_internal_device(ctx, &stv, &sms, &launches)) return CGM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stv);
  if (coded_len % 6 != 0 || coded_len / 6 * 5 <= kTail || n_cw < 0 || !llrs || !info_out)
    return cgm_internal_fail(ctx, CGM_EINVAL, "cgm_viterbi_decode: coded length must be 6k with 5k > 6");
  if (n_cw == 0) return CGM_OK;
  const long info_len = coded_len / 6 * 5 - kTail, total = info_len + kTail;
  void *dL = nullptr, *dD = nullptr, *dO = nullptr;
  cudaError_t e = cudaMalloc(&dL, static_cast<size_t>(n_cw * coded_len) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dD, static_cast<size_t>(n_cw * total) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dO, static_cast<size_t>(n_cw * info_len));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dL, llrs, static_cast<size_t>(n_cw * coded_len) * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    viterbi_decode<<<static_cast<unsigned>((n_cw + kVitWarps - 1) / kVitWarps), 32 * kVitWarps, 0, st>>>(
        static_cast<double*>(dL), nullptr, static_cast<uint2*>(dD), nullptr,
        static_cast<uint8_t*>(dO), coded_len, info_len, n_cw);
    ++*launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(info_out, dO, static_cast<size_t>(n_cw * info_len), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (void* q : {dL, dD, dO})
    if (q) cudaFree(q);
  if (e != cudaSuccess) return cgm_internal_fail(ctx, CGM_ECUDA, cudaGetErrorString(e));
  return CGM_OK;
}

// Rng(seed).fork(direction).fork(point).fork(trial) -- the trial streams of
// run_uplink_sweep (direction 1) / run_downlink_sweep (2) (sim.cpp:378-380)
uint64_t cgm_sweep_trial_key(uint64_t seed, int direction, long point, long trial) {
  return fork_key(fork_key(fork_key(seed, static_cast<uint64_t>(direction)), static_cast<uint64_t>(point)),
                  static_cast<uint64_t>(trial));
}

}  // extern "C"
