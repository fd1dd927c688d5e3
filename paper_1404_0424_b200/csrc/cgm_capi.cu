// cgm_capi.cu -- host runtime behind include/cgmimo_b200.h: contexts and
// streams, argument validation with the reference's error semantics,
// template dispatch of the fused subcarrier kernel, the chunked host-buffer
// pipeline (H2D / kernel / D2H overlapped on two streams) and the seeded
// device input generators.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the entry points are resolved at run time

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cgmimo_b200.h"
#include "cgm_alt.cuh"
#include "cgm_basis.cuh"
#include "cgm_precode_small.cuh"
#include "cgm_uplink_small.cuh"
#include "cgm_rows32.cuh"
#include "cgm_solve32.cuh"
#include "cgm_tc.cuh"

struct cgm_ctx {
  int device = 0;
  int sms = 0;
  int max_smem = 0;
  cudaStream_t user_stream = nullptr;
  // host-buffer pipeline: copy-in, compute and copy-out streams over a ring
  // of kHostSets device buffer sets (events: in done, compute done, out done)
  static constexpr int kHostSets = 3;
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t hev[kHostSets][3] = {};
  void* ws[kHostSets] = {nullptr, nullptr, nullptr};
  size_t ws_bytes[kHostSets] = {0, 0, 0};
  float* tscratch = nullptr;
  size_t tscratch_bytes = 0;
  long launches = 0;
  int policy = 0;  // 0 split K1+K2 path (production), 1 single fused kernel (A/B)
  // optional per-kernel event timing (bench roofline): pairs of events per launch
  int profiling = 0;
  // overlapped split path: channel kernel of chunk c+1 runs concurrently with
  // the solve kernel of chunk c (two internal streams, two workspace halves)
  cudaStream_t ov[2] = {nullptr, nullptr};
  cudaEvent_t ov_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // start, done1[2], done2[2]
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_log;  // kind, (start, stop)
  size_t ev_next = 0;
  // per kernel: dynamic shared memory already granted, occupancy per (threads, smem)
  struct KernInfo {
    const void* fn;
    int smem_set, nt, smem, occ;
  };
  std::vector<KernInfo> kinfo;
  std::string err;
};

namespace {

// Record a timing event pair around one kernel launch when profiling is on.
cudaEvent_t prof_event(cgm_ctx* ctx) {
  if (ctx->ev_next == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_next++];
}

// Environment overrides (A/B switches for the kernel variants; read per call
// so tests can flip them inside one process).
const char* env(const char* name) { return std::getenv(name); }

int fail(cgm_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CGM_CUDA(ctx, call)                                                        \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(ctx, CGM_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                             \
  } while (0)

// cudaFuncSetAttribute + occupancy query, cached per context: the two calls
// cost tens of microseconds per launch otherwise (host-bound small batches).
template <class F>
int kern_prep(cgm_ctx* ctx, F* fn, int nt, int smem, int* occ) {
  const void* key = reinterpret_cast<const void*>(fn);
  cgm_ctx::KernInfo* ki = nullptr;
  for (auto& k : ctx->kinfo)
    if (k.fn == key) ki = &k;
  if (!ki) {
    ctx->kinfo.push_back({key, -1, -1, -1, 0});
    ki = &ctx->kinfo.back();
  }
  if (smem > ki->smem_set) {
    CGM_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ki->smem_set = smem;
  }
  if (occ) {
    if (ki->nt != nt || ki->smem != smem) {
      int o = 0;
      CGM_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, nt, smem));
      ki->nt = nt;
      ki->smem = smem;
      ki->occ = o;
    }
    *occ = ki->occ;
  }
  return CGM_OK;
}

#define CGM_PREP(ctx, fn, nt, smem, occ)               \
  do {                                                 \
    const int rc_ = kern_prep(ctx, fn, nt, smem, occ); \
    if (rc_) return rc_;                               \
  } while (0)

unsigned gray_decode(unsigned g) {
  unsigned m = g;
  for (unsigned s = g >> 1; s != 0; s >>= 1) m ^= s;
  return m;
}

// Axis amplitude subsets of Gray square QAM, constellation.cpp:75-84.
cgm::AxisTables make_axis_tables() {
  cgm::AxisTables t;
  std::memset(&t, 0, sizeof t);
  for (int q = 0; q < 3; ++q) {
    const int half = q + 1;
    const unsigned levels = 1u << half;
    const double scale = 1.0 / std::sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
    int n0[3] = {0, 0, 0}, n1[3] = {0, 0, 0};
    for (unsigned k = 0; k < levels; ++k)
      t.lv[q][k] = static_cast<float>((2.0 * k - (levels - 1.0)) * scale);
    for (unsigned g = 0; g < levels; ++g) {
      const double amp = (2.0 * gray_decode(g) - (levels - 1.0)) * scale;
      for (int p = 0; p < half; ++p) {
        if ((g >> (half - 1 - p)) & 1u) t.a1[q][p][n1[p]++] = static_cast<float>(amp);
        else t.a0[q][p][n0[p]++] = static_cast<float>(amp);
      }
    }
  }
  return t;
}

int up_of(int U) { return U <= 8 ? 8 : U <= 16 ? 16 : U <= 32 ? 32 : 64; }

struct Launch {
  int smem = 0;
  int grid = 0;
  int t_in_smem = 1;
};

template <int UP, int NT, bool EXACT>
int plan_and_launch(cgm_ctx* ctx, cgm::KernelParams& p, cudaStream_t st) {
  const int Kmax = std::max(p.K, p.Kt);
  cgm::Smem<UP> L;
  p.t_in_smem = 1;
  L.plan(p.B, p.S, p.St, Kmax, EXACT, 1);
  if (L.total > ctx->max_smem) {
    p.t_in_smem = 0;
    L.plan(p.B, p.S, p.St, Kmax, EXACT, 0);
  }
  if (L.total > ctx->max_smem)
    return fail(ctx, CGM_EINVAL,
                "per-subcarrier working set %d B exceeds shared memory (%d B): reduce B or S",
                L.total, ctx->max_smem);
  if (p.use_tma == 2) p.use_tma = 0;  // the fused A/B kernel stages Y by bulk copy only
  auto kern = cgm::subcarrier_kernel<UP, NT, EXACT>;
  int occ = 0;
  CGM_PREP(ctx, kern, NT, L.total, &occ);
  if (occ < 1) return fail(ctx, CGM_EINVAL, "kernel does not fit on an SM (smem %d)", L.total);
  long grid = std::min<long>(p.n_sc, static_cast<long>(occ) * ctx->sms);
  if (grid < 1) grid = 1;
  if (EXACT && !p.t_in_smem) {
    const size_t need = static_cast<size_t>(grid) * Kmax * UP * UP * sizeof(float2);
    if (need > ctx->tscratch_bytes) {
      if (ctx->tscratch) cudaFree(ctx->tscratch);
      ctx->tscratch = nullptr;
      ctx->tscratch_bytes = 0;
      CGM_CUDA(ctx, cudaMalloc(&ctx->tscratch, need));
      ctx->tscratch_bytes = need;
    }
    p.tscratch = ctx->tscratch;
  }
  kern<<<static_cast<unsigned>(grid), NT, L.total, st>>>(p);
  CGM_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return CGM_OK;
}

// Split path (cgm_split.cuh): K1 channel kernel + K2 solve kernel per chunk
// of subcarriers; the chunk is sized so the K1->K2 workspace (and the H that
// the precoder re-reads) stays resident in the 126 MB L2.
template <int UP, bool EXACT>
int launch_split(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  const int Kmax = std::max(p.K, p.Kt);
  // K1: persistent, two TMA stages (prefetch one subcarrier ahead)
  cgm::K1Split sp;
  sp.plan(UP, p.B, p.S);
  // exact tracker, U = 32 / 64: the Chebyshev basis products run in their
  // own kernel (cgm_basis.cuh), so the channel kernel needs no basis buffers;
  // CGMIMO_BASIS=inline keeps them in the channel kernel
  bool basis_ext = false;
  if constexpr (EXACT && (UP == 32 || UP == 64)) {
    const char* e = env("CGMIMO_BASIS");
    basis_ext = p.S > 0 && p.K > 0 && !(e && std::strcmp(e, "inline") == 0) &&
                cgm::BasisGeo<UP>::SMEM <= ctx->max_smem;
  }
  p.basis_ext = basis_ext ? 1 : 0;
  // one vector per subcarrier (cfg4): the basis kernel also does the
  // extraction and the LLRs (basis_kernel<UP, true>), run after the CG; the
  // workspace carries the CG history instead of T_1..T_K.  CGMIMO_FX=0 keeps
  // the materialised basis; forced solve variants keep it too.
  {
    const char* fxe = env("CGMIMO_FX");
    p.fx = (basis_ext && p.S == 1 && p.St == 0 && !env("CGMIMO_SOLVE") &&
            !(fxe && std::strcmp(fxe, "0") == 0)) ? 1 : 0;
  }
  // fx with U = 32, opt-in (CGMIMO_FXFUSED=1): one warp per subcarrier does
  // Gram + matched filter + CG (fused_rows32_approx_kernel<16, true>) in place
  // of the tensor-core channel kernel and the CG kernel -- measured slower on
  // cfg4a (1.54 ms against 1.21 + 0.21 ms, K = 2)
  bool fxfused = false;
  int fx_smem = 0;
  if constexpr (EXACT && UP == 32) {
    const char* e = env("CGMIMO_FXFUSED");
    const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
    cgm::FusedSmem FL;
    FL.plan(p.B, p.S);
    fxfused = p.fx && p.U == 32 && p.S <= 16 && !p.hd_layout && (p.B % 2) == 0 && (al & 15u) == 0 &&
              FL.total <= ctx->max_smem && e && std::strcmp(e, "1") == 0;
    fx_smem = FL.total;
    if (fxfused) p.fx = 2;  // G rows not exactly Hermitian: the basis kernel symmetrises
  }
  const bool k1_basis = EXACT && !basis_ext;
  cgm::K1Smem<UP> L1;
  L1.plan(p.B, p.S, k1_basis, 2);
  if (L1.total > ctx->max_smem) {  // very large B: single stage
    sp.nstage = 1;
    L1.plan(p.B, p.S, k1_basis, 1);
  }
  p.k1_pair = sp.nstage;
  p.k1_spl = sp.spl;
  p.k1_wpp = sp.wpp;
  int nt1 = 32 * sp.wpp;
  cgm::K2Smem<UP> L2;
  L2.plan(p.B, p.S, p.St, Kmax, EXACT);
  if (L1.total > ctx->max_smem || L2.total > ctx->max_smem)
    return fail(ctx, CGM_EINVAL,
                "per-subcarrier working set (%d / %d B) exceeds shared memory (%d B)", L1.total,
                L2.total, ctx->max_smem);
  cgm::WsOffsets W;
  W.plan(UP, p.S, p.K, EXACT, p.fx);
  void (*k1)(cgm::KernelParams) = cgm::channel_kernel<UP, EXACT>;
  void (*k2)(cgm::KernelParams) = cgm::solve_kernel<UP, EXACT>;
  int smem2 = L2.total;
  int smem1 = L1.total;
  // U = 32, natural layout, whole 64-antenna blocks: Gram + matched filter on
  // the tensor cores (cgm_tc.cuh); CGMIMO_CHANNEL=ffma keeps the FFMA kernel
  bool use_tc = false;
  if constexpr (UP == 32) {
    const char* force = env("CGMIMO_CHANNEL");
    // the tensor-core kernel stages Y per 64-antenna block (64 S complex,
    // always a 16-byte multiple), so odd S is fine there (cfg4: S = 1)
    const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
    const int tc_tma = (!p.hd_layout && p.U == UP && (al & 15u) == 0) ? 1 : 0;
    if (cgm::tc::supported(p.U, p.B, p.S, tc_tma) && !(force && std::strcmp(force, "ffma") == 0)) {
      cgm::tc::Smem T;
      int nstg = 3;
      T.plan(p.S, EXACT, nstg);
      if (T.total > ctx->max_smem) T.plan(p.S, EXACT, nstg = 2);
      if (T.total <= ctx->max_smem) {
        use_tc = true;
        p.k1_pair = nstg;
        smem1 = T.total;
        // epilogue / split warps (CGMIMO_TC_WARPS=EP,SP; SP = 0: the same
        // warps do both).  Measured best (tools/microbench/tc_bench.cu and
        // bench.py, cfg2: 16 unified 37.9 us vs 8 + 8 specialised 39.4 us):
        // approx 16 unified; exact 8 unified for few vectors per subcarrier
        // (cfg4a: 2.28 vs 2.37 ms for 8 + 8), 8 + 8 specialised for many
        // (cfg5, S = 16: 15.7 vs 16.1 ms per step)
        int nep = EXACT ? 8 : 16, nsp = (EXACT && p.S >= 8) ? 8 : 0;
        if (const char* w = env("CGMIMO_TC_WARPS")) std::sscanf(w, "%d,%d", &nep, &nsp);
        if (nep == 16 && nsp == 0)
          k1 = cgm::channel_tc_kernel<EXACT, 16, 0>;
        else if (nep == 4 && nsp == 8)
          k1 = cgm::channel_tc_kernel<EXACT, 4, 8>;
        else if (nep == 8 && nsp == 8)
          k1 = cgm::channel_tc_kernel<EXACT, 8, 8>;
        else
          k1 = cgm::channel_tc_kernel<EXACT, 8, 0>, nep = 8, nsp = 0;
        nt1 = 32 * (nep + nsp + 2);
      }
    }
  }
  // K2: lane-per-row kernel by default; CGMIMO_SOLVE=tiles selects the
  // block-tiled FFMA2 CG (cgm_solve32.cuh, U = 32, >= 8 systems), which
  // issues ~25% fewer instructions but measured slower on cfg2 / cfg5 (lower
  // occupancy: 50 vs 43 us on cfg2); CGMIMO_SOLVE_TS=2|4
  bool use_s32 = false;
  int ts2 = 2;
  if constexpr (UP == 32) {
    const char* force = env("CGMIMO_SOLVE");
    if (const char* t = env("CGMIMO_SOLVE_TS")) ts2 = std::atoi(t) == 4 ? 4 : 2;
    cgm::S32Smem T2;
    T2.plan(p.B, p.S, p.St, Kmax, EXACT, ts2);
    if (p.S + p.St >= 8 && T2.total <= ctx->max_smem && force && std::strcmp(force, "tiles") == 0) {
      use_s32 = true;
      k2 = ts2 == 4 ? cgm::solve32_kernel<EXACT, 4> : cgm::solve32_kernel<EXACT, 2>;
      smem2 = T2.total;
    }
  }
  // persistent K2 with the next subcarrier's G + MF prefetched: measured
  // faster with many systems per subcarrier (cfg5, S + St = 32: 14.4 vs
  // 15.7 ms) and slower with few (cfg2 45.8 vs 43.3 us, cfg4 +13-40%: the
  // static subcarrier split loses the hardware's dynamic balancing), so on
  // from 24 systems; CGMIMO_SOLVE=pf / nopf force it either way
  bool use_pf = false;
  {
    const char* force = env("CGMIMO_SOLVE");
    const bool want = force ? std::strcmp(force, "pf") == 0
                            : (p.S + p.St >= 24);
    if (!use_s32 && want) {
      const int need = 128 + 2 * cgm::k2_pre_bytes(UP, p.S) + L2.total;
      if (need <= ctx->max_smem) {
        use_pf = true;
        k2 = cgm::solve_kernel_pf<UP, EXACT>;
        smem2 = need;
      }
    }
  }
  // U = 32: Gram row in registers, packed FFMA2 matvec (cgm_rows32.cuh).
  // Default for uplink-only calls (St = 0): one warp per (subcarrier, system
  // pair), approximate (cfg2 43.4 -> 35.2 us) or exact tracker with the
  // extraction inside the warp; CGMIMO_SOLVE=rows selects the CTA-per-
  // subcarrier form (any systems, CTA-wide tails), CGMIMO_SOLVE=lanes the
  // lane-per-row kernel
  bool use_rows = false, use_pairs = false;
  int rows_ns = 2;  // systems per warp of the pairs kernels
  bool rows_pf = false;
  if constexpr (UP == 32) {
    const char* force = env("CGMIMO_SOLVE");
    // uplink + precoding on the same channels (cfg5): the CTA-per-subcarrier
    // rows kernel with 8 warps (11.6 vs 12.7 ms for the persistent lane kernel)
    const bool cta = force ? std::strcmp(force, "rows") == 0 : (p.S > 0 && p.St > 0);
    if (!use_s32 && !force && p.St == 0 && p.K <= cgm::kMaxK) {
      use_rows = use_pairs = true;
      use_pf = false;
      k2 = EXACT ? cgm::solve_rows32_exact_pairs_kernel : cgm::solve_rows32_pairs_kernel<2>;
      smem2 = 0;
      if (!EXACT && env("CGMIMO_ROWS_NS") && std::atoi(env("CGMIMO_ROWS_NS")) == 4) {
        k2 = cgm::solve_rows32_pairs_kernel<4>;
        rows_ns = 4;
      } else if (!EXACT && env("CGMIMO_ROWS_NS") && std::atoi(env("CGMIMO_ROWS_NS")) == 1) {
        k2 = cgm::solve_rows32_pairs_kernel<1>;
        rows_ns = 1;
      } else if (!EXACT && env("CGMIMO_ROWS_PF") && std::atoi(env("CGMIMO_ROWS_PF")) == 1) {
        k2 = cgm::solve_rows32_pairs_pf_kernel;  // persistent, next item prefetched
        rows_pf = true;
        smem2 = 4 * (32 * 32 + 6 * 32) * 8;
      }
    } else if (!use_s32 && cta) {
      cgm::Rows32Smem R;
      R.plan(p.B, p.S, p.St, Kmax, EXACT);
      if (R.total <= ctx->max_smem) {
        use_rows = true;
        use_pf = false;
        k2 = cgm::solve_rows32_kernel<EXACT>;
        smem2 = R.total;
      }
    }
  }
  CGM_PREP(ctx, k2, 32, smem2, nullptr);
  // exact tracker, U = 32 / 64: the Chebyshev basis products in their own
  // kernel (cgm_basis.cuh) instead of the channel kernel's epilogue;
  // CGMIMO_BASIS=inline keeps them in the channel kernel
  void (*kb)(cgm::KernelParams) = nullptr;
  int nb_t = 0, nb_smem = 0, nb_spc = 1;
  if constexpr (EXACT && (UP == 32 || UP == 64)) {
    if (basis_ext) {
      using BG = cgm::BasisGeo<UP>;
      kb = p.fx ? cgm::basis_kernel<UP, true> : cgm::basis_kernel<UP, false>;
      nb_t = BG::NT;
      nb_smem = BG::SMEM;
      nb_spc = BG::SPC;
      CGM_PREP(ctx, kb, nb_t, nb_smem, nullptr);
    }
  }
  int occ1 = 0;
  CGM_PREP(ctx, k1, nt1, smem1, &occ1);
  if (occ1 < 1) return fail(ctx, CGM_EINVAL, "channel kernel does not fit on an SM");
  if (use_tc) occ1 = 1;  // one CTA (and all 512 TMEM columns) per SM
  // K2 block: enough lane groups for every system at once (>= UP threads
  // for the exact extraction), at most 8 warps
  using GE = cgm::K2Geo<UP>;
  const int nsys = p.S + p.St;
  int nw2 = (nsys + GE::GPW * GE::NS - 1) / (GE::GPW * GE::NS);
  if (EXACT) nw2 = std::max(nw2, std::max(4, UP / 32));
  nw2 = std::max(1, std::min(8, nw2));
  if (use_s32) nw2 = ((nsys + ts2 - 1) / ts2 * 8 + 31) / 32;  // 8 threads per tile, whole warps
  if (use_rows) {
    nw2 = (p.S + p.St) >= 16 ? 8 : 2;
    if (const char* e = env("CGMIMO_ROWS_WARPS")) nw2 = std::max(1, std::min(8, std::atoi(e)));
  }
  long g2cap = 1L << 40;
  if (use_pf) {
    int occ2 = 0;
    CGM_PREP(ctx, k2, 32 * nw2, smem2, &occ2);
    g2cap = static_cast<long>(std::max(occ2, 1)) * ctx->sms;
  }
  // chunk so that workspace + channel (+ Y) of a chunk fit comfortably in L2
  const size_t per_sc = static_cast<size_t>(W.stride) * 8 + static_cast<size_t>(p.B) * p.U * 8 +
                        static_cast<size_t>(p.B) * p.S * 8;
  long chunk = static_cast<long>((80ull << 20) / std::max<size_t>(per_sc, 1));
  chunk = std::max<long>(chunk, static_cast<long>(ctx->sms) * occ1);
  // external basis: the basis products need several full waves per launch
  // more than they need the workspace in L2 (T_1..T_K then round-trips HBM)
  if (kb) chunk = std::max<long>(chunk, static_cast<long>(ctx->sms) * 32);
  chunk = std::min(chunk, p.n_sc);
  // overlap K1(c+1) with K2(c): at least `ovl` chunks (CGMIMO_OVERLAP_CHUNKS,
  // default 1 = off: measured slower on cfg2/cfg3/cfg5)
  int ovl = 1;
  if (const char* e = env("CGMIMO_OVERLAP_CHUNKS")) ovl = std::max(1, std::atoi(e));
  const long min_chunk = static_cast<long>(ctx->sms) * occ1;
  if (ovl > 1 && p.n_sc >= 2 * min_chunk)
    chunk = std::min(chunk, std::max(min_chunk, (p.n_sc + ovl - 1) / ovl));
  const long total = p.n_sc;
  const bool overlap = chunk < total && ovl > 1;
  const size_t ws_half = static_cast<size_t>(chunk) * W.stride * sizeof(float2);
  const size_t ws_need = ws_half * (overlap ? 2 : 1);
  if (ws_need > ctx->tscratch_bytes) {
    if (ctx->tscratch) cudaFree(ctx->tscratch);
    ctx->tscratch = nullptr;
    ctx->tscratch_bytes = 0;
    CGM_CUDA(ctx, cudaMalloc(&ctx->tscratch, ws_need));
    ctx->tscratch_bytes = ws_need;
  }
  cudaStream_t s1 = st, s2 = st;
  if (overlap) {
    if (!ctx->ov[0]) {
      for (int i = 0; i < 2; ++i) CGM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->ov[i], cudaStreamNonBlocking));
      for (int i = 0; i < 5; ++i) CGM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ov_ev[i], cudaEventDisableTiming));
    }
    s1 = ctx->ov[0];
    s2 = ctx->ov[1];
    CGM_CUDA(ctx, cudaEventRecord(ctx->ov_ev[0], st));  // order after prior work on st
    CGM_CUDA(ctx, cudaStreamWaitEvent(s1, ctx->ov_ev[0], 0));
    CGM_CUDA(ctx, cudaStreamWaitEvent(s2, ctx->ov_ev[0], 0));
  }
  long ci = 0;
  for (long c0 = 0; c0 < total; c0 += chunk, ++ci) {
    const long n = std::min(chunk, total - c0);
    const int half = overlap ? static_cast<int>(ci & 1) : 0;
    p.ws = reinterpret_cast<float2*>(reinterpret_cast<char*>(ctx->tscratch) + half * ws_half);
    p.sc_base = c0;
    p.n_sc = n;
    const long g1 = std::max<long>(1, std::min<long>(n, static_cast<long>(occ1) * ctx->sms));
    if (overlap && ci >= 2)  // K2 of chunk ci-2 has released this workspace half
      CGM_CUDA(ctx, cudaStreamWaitEvent(s1, ctx->ov_ev[3 + half], 0));
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
    if (ctx->profiling) {
      e0 = prof_event(ctx);
      e1 = prof_event(ctx);
      e2 = prof_event(ctx);
      e3 = prof_event(ctx);
      cudaEventRecord(e0, s1);
    }
    if (fxfused) {
      auto kf = cgm::fused_rows32_approx_kernel<16, EXACT>;
      CGM_PREP(ctx, kf, 32, fx_smem, nullptr);
      kf<<<static_cast<unsigned>(n), 32, fx_smem, s1>>>(p);
    } else {
      k1<<<static_cast<unsigned>(g1), nt1, smem1, s1>>>(p);
    }
    CGM_CUDA(ctx, cudaGetLastError());
    if (ctx->profiling) cudaEventRecord(e1, s1);
    if (kb && !p.fx) {
      cudaEvent_t b0 = nullptr, b1 = nullptr;
      if (ctx->profiling) {
        b0 = prof_event(ctx);
        b1 = prof_event(ctx);
        cudaEventRecord(b0, s1);
      }
      kb<<<static_cast<unsigned>((n + nb_spc - 1) / nb_spc), nb_t, nb_smem, s1>>>(p);
      CGM_CUDA(ctx, cudaGetLastError());
      if (ctx->profiling) {
        cudaEventRecord(b1, s1);
        ctx->ev_log.push_back({3, {b0, b1}});
      }
      ctx->launches += 1;
    }
    if (overlap) {
      CGM_CUDA(ctx, cudaEventRecord(ctx->ov_ev[1 + half], s1));
      CGM_CUDA(ctx, cudaStreamWaitEvent(s2, ctx->ov_ev[1 + half], 0));
    }
    if (ctx->profiling) cudaEventRecord(e2, s2);
    if (fxfused)
      ;  // the CG ran inside the fused kernel
    else if (use_pairs && rows_pf)  // persistent: four CTAs per SM
      k2<<<static_cast<unsigned>(std::min<long>((n * ((p.S + 1) / 2) + 3) / 4, 4L * ctx->sms)), 128,
           smem2, s2>>>(p);
    else if (use_pairs)  // 4 warps per CTA, one (subcarrier, system pair) per warp
      k2<<<static_cast<unsigned>((n * ((p.S + rows_ns - 1) / rows_ns) + 3) / 4), 128, 0, s2>>>(p);
    else
      k2<<<static_cast<unsigned>(std::min(n, g2cap)), 32 * nw2, smem2, s2>>>(p);
    CGM_CUDA(ctx, cudaGetLastError());
    if (ctx->profiling) {
      cudaEventRecord(e3, s2);
      ctx->ev_log.push_back({1, {e0, e1}});
      ctx->ev_log.push_back({2, {e2, e3}});
    }
    if (kb && p.fx) {  // basis + extraction after the CG
      cudaEvent_t b0 = nullptr, b1 = nullptr;
      if (ctx->profiling) {
        b0 = prof_event(ctx);
        b1 = prof_event(ctx);
        cudaEventRecord(b0, s2);
      }
      kb<<<static_cast<unsigned>((n + nb_spc - 1) / nb_spc), nb_t, nb_smem, s2>>>(p);
      CGM_CUDA(ctx, cudaGetLastError());
      if (ctx->profiling) {
        cudaEventRecord(b1, s2);
        ctx->ev_log.push_back({3, {b0, b1}});
      }
      ctx->launches += 1;
    }
    if (overlap) CGM_CUDA(ctx, cudaEventRecord(ctx->ov_ev[3 + half], s2));
    ctx->launches += 2;
  }
  if (overlap) {  // the caller's stream waits for both internal streams
    CGM_CUDA(ctx, cudaEventRecord(ctx->ov_ev[0], s1));
    CGM_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ov_ev[0], 0));
    CGM_CUDA(ctx, cudaEventRecord(ctx->ov_ev[0], s2));
    CGM_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ov_ev[0], 0));
  }
  return CGM_OK;
}

template <int UP>
int dispatch_split(cgm_ctx* ctx, cgm::KernelParams& p, bool exact, cudaStream_t st) {
  return exact ? launch_split<UP, true>(ctx, p, st) : launch_split<UP, false>(ctx, p, st);
}

template <int UP, int NT>
int dispatch_exact(cgm_ctx* ctx, cgm::KernelParams& p, bool exact, cudaStream_t st) {
  return exact ? plan_and_launch<UP, NT, true>(ctx, p, st)
               : plan_and_launch<UP, NT, false>(ctx, p, st);
}

// Cholesky / CGLS / Neumann detection and precoding (cgm_alt.cuh): one CTA
// per subcarrier, persistent over the chunk.
int launch_alt(cgm_ctx* ctx, cgm::KernelParams& p, cudaStream_t st) {
  cgm::alt::AltSmem L;
  L.plan(p.B, p.U, p.St > 0 ? p.St : p.S, p.method);
  const size_t smem = static_cast<size_t>(L.total) * sizeof(float2);
  if (smem > static_cast<size_t>(ctx->max_smem))
    return fail(ctx, CGM_EINVAL, "B = %d, U = %d: %zu bytes of shared memory per subcarrier exceed %d",
                p.B, p.U, smem, ctx->max_smem);
  auto k = p.method == cgm::alt::kCholesky ? cgm::alt::alt_kernel<cgm::alt::kCholesky>
           : p.method == cgm::alt::kCgls   ? cgm::alt::alt_kernel<cgm::alt::kCgls>
                                           : cgm::alt::alt_kernel<cgm::alt::kNeumann>;
  int occ = 0;
  CGM_PREP(ctx, k, cgm::alt::NT, static_cast<int>(smem), &occ);
  const long grid = std::max<long>(1, std::min<long>(p.n_sc, static_cast<long>(std::max(occ, 1)) * ctx->sms));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, st);
  }
  k<<<static_cast<unsigned>(grid), cgm::alt::NT, smem, st>>>(p);
  CGM_CUDA(ctx, cudaGetLastError());
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    ctx->ev_log.push_back({2, {e0, e1}});
  }
  ++ctx->launches;
  return CGM_OK;
}

// Fused small-U CG precoder (cgm_precode_small.cuh): pure precode calls with
// H_d in the reference layout, U <= 16.  CGMIMO_PRECODE=split keeps the
// channel + solve pair.
template <int UP>
int launch_precode_small(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  cgm::PrecodeSmallSmem L;
  L.plan(UP, p.B, p.St);
  auto k = cgm::precode_small_kernel<UP>;
  int occ = 0;
  CGM_PREP(ctx, k, cgm::PrecodeSmallGeo<UP>::NT, L.total, &occ);
  const long grid = std::max<long>(1, std::min<long>(p.n_sc, static_cast<long>(std::max(occ, 1)) * ctx->sms));
  p.use_tma = ((p.B % 2) == 0 && (reinterpret_cast<uintptr_t>(p.H) & 15u) == 0) ? 1 : 0;
  p.sc_base = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, st);
  }
  k<<<static_cast<unsigned>(grid), cgm::PrecodeSmallGeo<UP>::NT, L.total, st>>>(p);
  CGM_CUDA(ctx, cudaGetLastError());
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    ctx->ev_log.push_back({2, {e0, e1}});
  }
  ++ctx->launches;
  return CGM_OK;
}

// Fully fused U = 32 approximate-tracker detector (one warp per subcarrier,
// cgm_rows32.cuh): Gram + matched filters + every system's CG in one kernel.
// Opt-in (CGMIMO_FUSED=1): measured 111 us on cfg2 against 67 us for the
// tensor-core channel kernel + pairs solve kernel -- eight warps per SM
// leave the fourteen sequential CG chains of a subcarrier latency-exposed.
bool fused_rows32_ok(cgm_ctx* ctx, const cgm::KernelParams& p, bool exact) {
  if (exact || p.U != 32 || p.St != 0 || p.S < 1 || p.S > 16 || p.hd_layout || (p.B % 2) != 0)
    return false;
  const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
  if (al & 15u) return false;
  const char* e = env("CGMIMO_FUSED");
  if (!(e && std::strcmp(e, "1") == 0)) return false;
  cgm::FusedSmem L;
  L.plan(p.B, p.S);
  return L.total <= ctx->max_smem;
}

int launch_fused_rows32(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  cgm::FusedSmem L;
  L.plan(p.B, p.S);
  auto k = cgm::fused_rows32_approx_kernel<16>;
  CGM_PREP(ctx, k, 32, L.total, nullptr);
  p.sc_base = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, st);
  }
  k<<<static_cast<unsigned>(p.n_sc), 32, L.total, st>>>(p);
  CGM_CUDA(ctx, cudaGetLastError());
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    ctx->ev_log.push_back({2, {e0, e1}});
  }
  ++ctx->launches;
  return CGM_OK;
}

// Fused small-U CG detector (cgm_uplink_small.cuh): uplink-only calls with
// U <= 16, one warp per subcarrier.  CGMIMO_UPSMALL=split keeps the pair.
bool uplink_small_ok(cgm_ctx* ctx, const cgm::KernelParams& p, bool exact) {
  if (!(p.St == 0 && p.S >= 1 && !p.hd_layout && p.U <= 16 && p.K >= 1 && p.K <= cgm::kMaxK))
    return false;
  const char* e = env("CGMIMO_UPSMALL");
  if (e && std::strcmp(e, "split") == 0) return false;
  cgm::UpSmallSmem L;
  L.plan(up_of(p.U), p.B, p.U, p.S, p.K, exact);
  return L.total <= ctx->max_smem;
}

template <int UP, bool EXACT>
int launch_uplink_small(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  cgm::UpSmallSmem L;
  L.plan(UP, p.B, p.U, p.S, p.K, EXACT);
  auto k = cgm::uplink_small_kernel<UP, EXACT>;
  int occ = 0;
  CGM_PREP(ctx, k, 32, L.total, &occ);
  const long grid = std::max<long>(1, std::min<long>(p.n_sc, static_cast<long>(std::max(occ, 1)) * ctx->sms));
  const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
  p.use_tma = ((p.B * p.U) % 2 == 0 && (p.B * p.S) % 2 == 0 && (al & 15u) == 0) ? 1 : 0;
  p.sc_base = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, st);
  }
  k<<<static_cast<unsigned>(grid), 32, L.total, st>>>(p);
  CGM_CUDA(ctx, cudaGetLastError());
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    ctx->ev_log.push_back({2, {e0, e1}});
  }
  ++ctx->launches;
  return CGM_OK;
}

bool precode_small_ok(cgm_ctx* ctx, const cgm::KernelParams& p) {
  if (!(p.S == 0 && p.St > 0 && p.hd_layout && p.U <= 16 && p.B <= 512 && p.B >= 4 && p.B % 2 == 0))
    return false;
  const char* e = env("CGMIMO_PRECODE");
  if (e && std::strcmp(e, "split") == 0) return false;
  cgm::PrecodeSmallSmem L;
  L.plan(up_of(p.U), p.B, p.St);
  return L.total <= ctx->max_smem;
}

int launch(cgm_ctx* ctx, cgm::KernelParams& p, bool exact, cudaStream_t st) {
  if (p.n_sc <= 0) return CGM_OK;
  if (p.method != cgm::alt::kCg) return launch_alt(ctx, p, st);
  const int UP = up_of(p.U);
  if (ctx->policy == 0 && fused_rows32_ok(ctx, p, exact)) return launch_fused_rows32(ctx, p, st);
  if (ctx->policy == 0 && uplink_small_ok(ctx, p, exact)) {
    if (UP == 8) return exact ? launch_uplink_small<8, true>(ctx, p, st) : launch_uplink_small<8, false>(ctx, p, st);
    return exact ? launch_uplink_small<16, true>(ctx, p, st) : launch_uplink_small<16, false>(ctx, p, st);
  }
  if (ctx->policy == 0 && precode_small_ok(ctx, p))
    return UP == 8 ? launch_precode_small<8>(ctx, p, st) : launch_precode_small<16>(ctx, p, st);
  const uintptr_t a = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
  // 1: H and Y by bulk copy; 2 (odd S, channel_kernel only): H by bulk copy,
  // the padded Y rows by the threads
  p.use_tma = (!p.hd_layout && p.U == UP && (p.B % 2) == 0 && (a & 15u) == 0)
                  ? ((p.S % 2) == 0 ? 1 : 2) : 0;
  if (ctx->policy == 0) {
    switch (UP) {
      case 8: return dispatch_split<8>(ctx, p, exact, st);
      case 16: return dispatch_split<16>(ctx, p, exact, st);
      case 32: return dispatch_split<32>(ctx, p, exact, st);
      default: return dispatch_split<64>(ctx, p, exact, st);
    }
  }
  switch (UP) {
    case 8: return dispatch_exact<8, 128>(ctx, p, exact, st);
    case 16: return dispatch_exact<16, 128>(ctx, p, exact, st);
    case 32: return dispatch_exact<32, 288>(ctx, p, exact, st);
    default: return dispatch_exact<64, 320>(ctx, p, exact, st);
  }
}

// ------------------------------------------------------------ validation
struct Job {
  int B = 0, U = 0, S = 0, St = 0, K = 0, Kt = 0, bits = 0, tracker = 0;
  int method = cgm::alt::kCg;
  long n_sc = 0;
  double rho_u = 1, n0 = 1, es = 1, rho_d = 1;
  bool hd_layout = false;
  const float *H = nullptr, *Y = nullptr, *T = nullptr;
  float *xhat = nullptr, *mu = nullptr, *rho = nullptr, *llr = nullptr;
  uint8_t* status = nullptr;
  float *q = nullptr, *s = nullptr, *gain = nullptr;
  uint8_t* pstatus = nullptr;
};

int validate(cgm_ctx* ctx, const Job& j) {
  if (!ctx) return CGM_EINVAL;
  if (j.n_sc < 0) return fail(ctx, CGM_EINVAL, "n_sc must be >= 0");
  if (j.B < 1 || j.U < 1) return fail(ctx, CGM_EINVAL, "B and U must be >= 1");
  if (j.U > 64) return fail(ctx, CGM_EINVAL, "U = %d > 64 is not supported", j.U);
  if (j.S < 0 || j.St < 0 || j.S + j.St > cgm::kMaxSys)
    return fail(ctx, CGM_EINVAL, "vectors per subcarrier must be in [0, %d]", cgm::kMaxSys);
  if (j.S > 0) {
    // detect.cpp:186-188
    if (!(j.rho_u > 0.0 && j.n0 > 0.0 && j.es > 0.0))
      return fail(ctx, CGM_EINVAL, "detect_cg: bad parameters (rho_u, N0, Es must be > 0)");
    if (j.K < 1) return fail(ctx, CGM_EINVAL, "detect: need at least one iteration / series term");
    if (j.K > (j.method == cgm::alt::kCg ? cgm::kMaxK : 256))
      return fail(ctx, CGM_EINVAL, "K = %d is above the supported maximum", j.K);
    if (j.bits != 2 && j.bits != 4 && j.bits != 6)
      return fail(ctx, CGM_EINVAL, "qam_bits must be 2, 4 or 6");
    if (j.tracker != CGM_TRACKER_EXACT && j.tracker != CGM_TRACKER_APPROX)
      return fail(ctx, CGM_EINVAL, "unknown tracker %d", j.tracker);
    if (!j.H || !j.Y) return fail(ctx, CGM_EINVAL, "H and Y are required");
  }
  if (j.St > 0) {
    // precode.cpp:59-60, solvers.cpp:39-40
    if (!(j.rho_d > 0.0)) return fail(ctx, CGM_EINVAL, "precode_cg: rho_d must be positive");
    if (j.Kt < 1) return fail(ctx, CGM_EINVAL, "precode: need at least one iteration / series term");
    if (j.Kt > (j.method == cgm::alt::kCg ? cgm::kMaxK : 256))
      return fail(ctx, CGM_EINVAL, "K = %d is above the supported maximum", j.Kt);
    if (!j.H || !j.T) return fail(ctx, CGM_EINVAL, "H and T are required");
  }
  return CGM_OK;
}

cgm::KernelParams params_of(const Job& j, long n_sc) {
  cgm::KernelParams p;
  std::memset(&p, 0, sizeof p);
  p.H = reinterpret_cast<const float2*>(j.H);
  p.Y = reinterpret_cast<const float2*>(j.Y);
  p.T = reinterpret_cast<const float2*>(j.T);
  p.xhat = reinterpret_cast<float2*>(j.xhat);
  p.mu = j.mu;
  p.rho = j.rho;
  p.llr = j.llr;
  p.status = j.status;
  p.q = reinterpret_cast<float2*>(j.q);
  p.s_out = reinterpret_cast<float2*>(j.s);
  p.gain = j.gain;
  p.pstatus = j.pstatus;
  p.n_sc = n_sc;
  p.B = j.B;
  p.U = j.U;
  p.S = j.S;
  p.St = j.St;
  p.K = j.S > 0 ? j.K : 0;
  p.Kt = j.St > 0 ? j.Kt : 0;
  p.bits = j.bits > 0 ? j.bits : 2;
  p.hd_layout = j.hd_layout ? 1 : 0;
  p.rho_inv_u = j.S > 0 ? static_cast<float>(1.0 / j.rho_u) : 0.f;
  p.rho_inv_d = j.St > 0 ? static_cast<float>(1.0 / j.rho_d) : 0.f;
  p.n0 = static_cast<float>(j.n0);
  if (const char* dbg = env("CGMIMO_DEBUG_WS")) p.debug = std::atoi(dbg);
  p.es = static_cast<float>(j.es);
  p.method = j.method;
  return p;
}

bool is_exact(const Job& j) { return j.S > 0 && j.tracker == CGM_TRACKER_EXACT; }

// Per-subcarrier byte counts of each array (host pipeline).
struct Sizes {
  size_t h, y, t, xhat, mu, rho, llr, st, q, s, gain, pst;
  size_t total() const { return h + y + t + xhat + mu + rho + llr + st + q + s + gain + pst; }
};

Sizes sizes_of(const Job& j) {
  Sizes z;
  z.h = static_cast<size_t>(j.B) * j.U * 8;
  z.y = static_cast<size_t>(j.S) * j.B * 8;
  z.t = static_cast<size_t>(j.St) * j.U * 8;
  z.xhat = j.xhat ? static_cast<size_t>(j.S) * j.U * 8 : 0;
  z.mu = j.mu ? static_cast<size_t>(j.S) * j.U * 4 : 0;
  z.rho = j.rho ? static_cast<size_t>(j.S) * j.U * 4 : 0;
  z.llr = j.llr ? static_cast<size_t>(j.S) * j.U * j.bits * 4 : 0;
  z.st = j.status ? static_cast<size_t>(j.S) : 0;
  z.q = j.q ? static_cast<size_t>(j.St) * j.B * 8 : 0;
  z.s = j.s ? static_cast<size_t>(j.St) * j.B * 8 : 0;
  z.gain = j.gain ? static_cast<size_t>(j.St) * 4 : 0;
  z.pst = j.pstatus ? static_cast<size_t>(j.St) : 0;
  return z;
}

size_t round_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

int run_job(cgm_ctx* ctx, const Job& j, unsigned flags) {
  int rc = validate(ctx, j);
  if (rc) return rc;
  CGM_CUDA(ctx, cudaSetDevice(ctx->device));
  if (j.n_sc == 0) return CGM_OK;
  if (flags & CGM_DEVICE_POINTERS) {
    cgm::KernelParams p = params_of(j, j.n_sc);
    return launch(ctx, p, is_exact(j), ctx->user_stream);
  }
  // ---------------- host buffers: chunked three-stream pipeline
  // chunk i uses buffer set i % kHostSets: H2D on pipe[0] (after the set's
  // previous D2H), kernels on pipe[1], D2H on pipe[2].  The host->device
  // copies run back to back and overlap the device->host copies of earlier
  // chunks (PCIe is full duplex); CGMIMO_HOST_CHUNKS sets the chunk count.
  constexpr int NB = cgm_ctx::kHostSets;
  const Sizes z = sizes_of(j);
  const size_t per_sc = z.total() + 16 * 12;
  const size_t budget = 192ull << 20;  // per buffer set
  long chunk = static_cast<long>(std::max<size_t>(1, budget / std::max<size_t>(per_sc, 1)));
  chunk = std::min(chunk, j.n_sc);
  // up to 8 chunks of at least ~8 MB each: small batches are bound by the
  // per-chunk API calls, not by the copy overlap (cfg1, 9.4 MB: one chunk
  // 4.1 M vec/s against 3.2 M with eight)
  const size_t total_bytes = per_sc * static_cast<size_t>(j.n_sc);
  int nch = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, total_bytes / (8ull << 20))));
  if (const char* e = env("CGMIMO_HOST_CHUNKS")) nch = std::max(1, std::atoi(e));
  const long min_chunk = std::max<long>(1, ctx->sms);  // keep each launch >= one wave
  if (j.n_sc >= 2 * min_chunk)
    chunk = std::min(chunk, std::max(min_chunk, (j.n_sc + nch - 1) / nch));
  const int nsets = static_cast<int>(std::min<long>(NB, (j.n_sc + chunk - 1) / chunk));
  for (int b = 0; b < nsets; ++b) {
    size_t need = 0;
    const size_t parts[12] = {z.h, z.y, z.t, z.xhat, z.mu, z.rho, z.llr, z.st, z.q, z.s, z.gain, z.pst};
    for (size_t x : parts) need += round_up(x * chunk);
    if (need > ctx->ws_bytes[b]) {
      if (ctx->ws[b]) cudaFree(ctx->ws[b]);
      ctx->ws[b] = nullptr;
      ctx->ws_bytes[b] = 0;
      CGM_CUDA(ctx, cudaMalloc(&ctx->ws[b], need));
      ctx->ws_bytes[b] = need;
    }
    for (int k = 0; k < 3; ++k)
      if (!ctx->hev[b][k]) CGM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->hev[b][k], cudaEventDisableTiming));
  }
  cudaStream_t s_in = ctx->pipe[0], s_comp = ctx->pipe[1], s_out = ctx->pipe[2];
  auto H8 = reinterpret_cast<const char*>(j.H);
  auto Y8 = reinterpret_cast<const char*>(j.Y);
  auto T8 = reinterpret_cast<const char*>(j.T);
  int ci = 0;
  for (long c0 = 0; c0 < j.n_sc; c0 += chunk, ++ci) {
    const long n = std::min(chunk, j.n_sc - c0);
    const int b = ci % nsets;
    char* base = static_cast<char*>(ctx->ws[b]);
    size_t off = 0;
    auto carve = [&](size_t per) -> char* {
      char* p = per ? base + off : nullptr;
      off += round_up(per * chunk);
      return p;
    };
    char* dH = carve(z.h);
    char* dY = carve(z.y);
    char* dT = carve(z.t);
    char* dX = carve(z.xhat);
    char* dMu = carve(z.mu);
    char* dRho = carve(z.rho);
    char* dL = carve(z.llr);
    char* dSt = carve(z.st);
    char* dQ = carve(z.q);
    char* dS = carve(z.s);
    char* dG = carve(z.gain);
    char* dPs = carve(z.pst);
    // ---- copy in (after this set's previous results left the device)
    if (ci >= nsets) CGM_CUDA(ctx, cudaStreamWaitEvent(s_in, ctx->hev[b][2], 0));
    if (z.h) CGM_CUDA(ctx, cudaMemcpyAsync(dH, H8 + z.h * c0, z.h * n, cudaMemcpyHostToDevice, s_in));
    if (z.y) CGM_CUDA(ctx, cudaMemcpyAsync(dY, Y8 + z.y * c0, z.y * n, cudaMemcpyHostToDevice, s_in));
    if (z.t) CGM_CUDA(ctx, cudaMemcpyAsync(dT, T8 + z.t * c0, z.t * n, cudaMemcpyHostToDevice, s_in));
    CGM_CUDA(ctx, cudaEventRecord(ctx->hev[b][0], s_in));
    // ---- compute
    CGM_CUDA(ctx, cudaStreamWaitEvent(s_comp, ctx->hev[b][0], 0));
    Job jd = j;
    jd.H = reinterpret_cast<float*>(dH);
    jd.Y = reinterpret_cast<float*>(dY);
    jd.T = reinterpret_cast<float*>(dT);
    jd.xhat = reinterpret_cast<float*>(dX);
    jd.mu = reinterpret_cast<float*>(dMu);
    jd.rho = reinterpret_cast<float*>(dRho);
    jd.llr = reinterpret_cast<float*>(dL);
    jd.status = reinterpret_cast<uint8_t*>(dSt);
    jd.q = reinterpret_cast<float*>(dQ);
    jd.s = reinterpret_cast<float*>(dS);
    jd.gain = reinterpret_cast<float*>(dG);
    jd.pstatus = reinterpret_cast<uint8_t*>(dPs);
    cgm::KernelParams p = params_of(jd, n);
    rc = launch(ctx, p, is_exact(j), s_comp);
    if (rc) return rc;
    CGM_CUDA(ctx, cudaEventRecord(ctx->hev[b][1], s_comp));
    // ---- copy out
    CGM_CUDA(ctx, cudaStreamWaitEvent(s_out, ctx->hev[b][1], 0));
    auto d2h = [&](void* host, const char* dev, size_t per) -> cudaError_t {
      if (!per) return cudaSuccess;
      return cudaMemcpyAsync(static_cast<char*>(host) + per * c0, dev, per * n,
                             cudaMemcpyDeviceToHost, s_out);
    };
    CGM_CUDA(ctx, d2h(j.xhat, dX, z.xhat));
    CGM_CUDA(ctx, d2h(j.mu, dMu, z.mu));
    CGM_CUDA(ctx, d2h(j.rho, dRho, z.rho));
    CGM_CUDA(ctx, d2h(j.llr, dL, z.llr));
    CGM_CUDA(ctx, d2h(j.status, dSt, z.st));
    CGM_CUDA(ctx, d2h(j.q, dQ, z.q));
    CGM_CUDA(ctx, d2h(j.s, dS, z.s));
    CGM_CUDA(ctx, d2h(j.gain, dG, z.gain));
    CGM_CUDA(ctx, d2h(j.pstatus, dPs, z.pst));
    CGM_CUDA(ctx, cudaEventRecord(ctx->hev[b][2], s_out));
  }
  CGM_CUDA(ctx, cudaStreamSynchronize(s_out));
  CGM_CUDA(ctx, cudaStreamSynchronize(s_comp));
  CGM_CUDA(ctx, cudaStreamSynchronize(s_in));
  return CGM_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* cgm_version(void) { return "cgmimo_b200 0.1 sm_100a"; }

// hooks for cgm_generate.cu (same library, not part of the public header)
int cgm_internal_fail(cgm_ctx* ctx, int code, const char* msg) { return fail(ctx, code, "%s", msg); }
int cgm_internal_device(cgm_ctx* ctx, void** stream, int* sms, long** launches) {
  if (!ctx) return CGM_EINVAL;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, CGM_ECUDA, "cudaSetDevice");
  *stream = ctx->user_stream;
  *sms = ctx->sms;
  *launches = &ctx->launches;
  return CGM_OK;
}

int cgm_ctx_create(int device, cgm_ctx** out) {
  if (!out) return CGM_EINVAL;
  *out = nullptr;
  cgm_ctx* ctx = new cgm_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&ctx->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int major = 0, minor = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (e == cudaSuccess && major != 10) {
    delete ctx;
    return CGM_ECUDA;  // built for sm_100a only
  }
  for (int i = 0; i < 3 && e == cudaSuccess; ++i)
    e = cudaStreamCreateWithFlags(&ctx->pipe[i], cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    const cgm::AxisTables t = make_axis_tables();
    e = cudaMemcpyToSymbol(cgm::c_axis, &t, sizeof t);
  }
  if (e != cudaSuccess) {
    delete ctx;
    return CGM_ECUDA;
  }
  *out = ctx;
  return CGM_OK;
}

int cgm_ctx_destroy(cgm_ctx* ctx) {
  if (!ctx) return CGM_OK;
  cudaSetDevice(ctx->device);
  for (int b = 0; b < cgm_ctx::kHostSets; ++b) {
    if (ctx->ws[b]) cudaFree(ctx->ws[b]);
    for (int k = 0; k < 3; ++k)
      if (ctx->hev[b][k]) cudaEventDestroy(ctx->hev[b][k]);
  }
  for (int i = 0; i < 3; ++i)
    if (ctx->pipe[i]) cudaStreamDestroy(ctx->pipe[i]);
  if (ctx->tscratch) cudaFree(ctx->tscratch);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i)
    if (ctx->ov[i]) cudaStreamDestroy(ctx->ov[i]);
  for (int i = 0; i < 5; ++i)
    if (ctx->ov_ev[i]) cudaEventDestroy(ctx->ov_ev[i]);
  delete ctx;
  return CGM_OK;
}

int cgm_ctx_set_stream(cgm_ctx* ctx, void* stream) {
  if (!ctx) return CGM_EINVAL;
  ctx->user_stream = static_cast<cudaStream_t>(stream);
  return CGM_OK;
}

int cgm_ctx_set_profiling(cgm_ctx* ctx, int on) {
  if (!ctx) return CGM_EINVAL;
  ctx->profiling = on ? 1 : 0;
  ctx->ev_log.clear();
  ctx->ev_next = 0;
  return CGM_OK;
}

int cgm_ctx_kernel_times_ex(cgm_ctx* ctx, double* channel_ms, double* basis_ms, double* solve_ms,
                            long* launches) {
  if (!ctx || !channel_ms || !basis_ms || !solve_ms || !launches) return CGM_EINVAL;
  *channel_ms = *basis_ms = *solve_ms = 0.0;
  *launches = 0;
  for (auto& rec : ctx->ev_log) {
    CGM_CUDA(ctx, cudaEventSynchronize(rec.second.second));
    float ms = 0.f;
    CGM_CUDA(ctx, cudaEventElapsedTime(&ms, rec.second.first, rec.second.second));
    (rec.first == 1 ? *channel_ms : rec.first == 3 ? *basis_ms : *solve_ms) += ms;
    if (rec.first == 1) ++*launches;
  }
  return CGM_OK;
}

int cgm_ctx_kernel_times(cgm_ctx* ctx, double* channel_ms, double* solve_ms, long* launches) {
  double basis = 0.0;
  const int rc = cgm_ctx_kernel_times_ex(ctx, channel_ms, &basis, solve_ms, launches);
  if (rc == CGM_OK) *channel_ms += basis;  // basis products counted with the channel stage
  return rc;
}

int cgm_ctx_set_kernel_policy(cgm_ctx* ctx, int policy) {
  if (!ctx || policy < 0 || policy > 1) return CGM_EINVAL;
  ctx->policy = policy;
  return CGM_OK;
}

int cgm_synchronize(cgm_ctx* ctx) {
  if (!ctx) return CGM_EINVAL;
  CGM_CUDA(ctx, cudaSetDevice(ctx->device));
  CGM_CUDA(ctx, cudaStreamSynchronize(ctx->user_stream));
  return CGM_OK;
}

const char* cgm_last_error(const cgm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

long cgm_kernel_launches(const cgm_ctx* ctx) { return ctx ? ctx->launches : 0; }

int cgm_detect_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* H, const float* Y,
                  double rho_u, double n0, double es, int qam_bits, int K, int tracker,
                  float* xhat, float* mu, float* rho, float* llr, uint8_t* status,
                  unsigned flags) {
  Job j;
  j.B = B; j.U = U; j.n_sc = n_sc; j.S = S; j.H = H; j.Y = Y;
  j.rho_u = rho_u; j.n0 = n0; j.es = es; j.bits = qam_bits; j.K = K; j.tracker = tracker;
  j.xhat = xhat; j.mu = mu; j.rho = rho; j.llr = llr; j.status = status;
  if (S < 1) return fail(ctx, CGM_EINVAL, "detect_cg: S must be >= 1");
  return run_job(ctx, j, flags);
}

int cgm_precode_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* Hd,
                   const float* T, double rho_d, int K, float* q, float* s, float* gain,
                   uint8_t* status, unsigned flags) {
  Job j;
  j.B = B; j.U = U; j.n_sc = n_sc; j.St = S; j.H = Hd; j.T = T; j.rho_d = rho_d; j.Kt = K;
  j.hd_layout = !(flags & CGM_HD_UPLINK_LAYOUT);
  j.q = q; j.s = s; j.gain = gain; j.pstatus = status;
  if (S < 1) return fail(ctx, CGM_EINVAL, "precode_cg: S must be >= 1");
  return run_job(ctx, j, flags);
}

int cgm_detect(cgm_ctx* ctx, int method, int B, int U, long n_sc, int S, const float* H,
               const float* Y, double rho_u, double n0, double es, int qam_bits, int iters,
               int tracker, float* xhat, float* mu, float* rho, float* llr, uint8_t* status,
               unsigned flags) {
  if (method < CGM_METHOD_CHOLESKY || method > CGM_METHOD_NEUMANN)
    return fail(ctx, CGM_EINVAL, "unknown method %d", method);
  if (method == CGM_METHOD_CHOLESKY) iters = 1;  // no iteration count (detect.cpp:122-125)
  if (method != CGM_METHOD_CG) tracker = CGM_TRACKER_APPROX;
  Job j;
  j.method = method;
  j.B = B; j.U = U; j.n_sc = n_sc; j.S = S; j.H = H; j.Y = Y;
  j.rho_u = rho_u; j.n0 = n0; j.es = es; j.bits = qam_bits; j.K = iters; j.tracker = tracker;
  j.xhat = xhat; j.mu = mu; j.rho = rho; j.llr = llr; j.status = status;
  if (S < 1) return fail(ctx, CGM_EINVAL, "detect: S must be >= 1");
  return run_job(ctx, j, flags);
}

int cgm_precode(cgm_ctx* ctx, int method, int B, int U, long n_sc, int S, const float* Hd,
                const float* T, double rho_d, int iters, float* q, float* s, float* gain,
                uint8_t* status, unsigned flags) {
  if (method < CGM_METHOD_CHOLESKY || method > CGM_METHOD_NEUMANN)
    return fail(ctx, CGM_EINVAL, "unknown method %d", method);
  if (method == CGM_METHOD_CHOLESKY) iters = 1;  // precode_explicit (precode.cpp:45-54)
  Job j;
  j.method = method;
  j.B = B; j.U = U; j.n_sc = n_sc; j.St = S; j.H = Hd; j.T = T; j.rho_d = rho_d; j.Kt = iters;
  j.hd_layout = !(flags & CGM_HD_UPLINK_LAYOUT);
  j.q = q; j.s = s; j.gain = gain; j.pstatus = status;
  if (S < 1) return fail(ctx, CGM_EINVAL, "precode: S must be >= 1");
  return run_job(ctx, j, flags);
}

int cgm_detect_precode_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* H,
                          const float* Y, double rho_u, double n0, double es, int qam_bits,
                          int K, int tracker, float* xhat, float* mu, float* rho, float* llr,
                          uint8_t* status, int St, const float* T, double rho_d, int Kt,
                          float* q, float* s, float* gain, uint8_t* pstatus, unsigned flags) {
  Job j;
  j.B = B; j.U = U; j.n_sc = n_sc; j.S = S; j.H = H; j.Y = Y;
  j.rho_u = rho_u; j.n0 = n0; j.es = es; j.bits = qam_bits; j.K = K; j.tracker = tracker;
  j.xhat = xhat; j.mu = mu; j.rho = rho; j.llr = llr; j.status = status;
  j.St = St; j.T = T; j.rho_d = rho_d; j.Kt = Kt;
  j.q = q; j.s = s; j.gain = gain; j.pstatus = pstatus;
  if (S < 1 || St < 1) return fail(ctx, CGM_EINVAL, "detect_precode_cg: S and St must be >= 1");
  return run_job(ctx, j, flags);
}


// ---------------------------------------------------------------- multi-GPU
struct cgm_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

namespace {
// NCCL through dlopen: the library loads (and single-GPU use works) where
// NCCL is absent; in a torch process the already-loaded libnccl is reused.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}
}  // namespace

#define CGM_NCCL(ctx, call)                                                                 \
  do {                                                                                      \
    const ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                                  \
      return fail(ctx, CGM_ENCCL, "%s: %s", #call, nccl_api().GetErrorString(r_));           \
  } while (0)

int cgm_comm_unique_id(unsigned char id[128]) {
  if (!id) return CGM_EINVAL;
  NcclApi& n = nccl_api();
  if (!n.ok) return CGM_ENCCL;
  ncclUniqueId uid;
  if (n.GetUniqueId(&uid) != ncclSuccess) return CGM_ENCCL;
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &uid, sizeof uid);
  return CGM_OK;
}

int cgm_comm_create(cgm_ctx* ctx, int nranks, int rank, const unsigned char id[128],
                    cgm_comm** out) {
  if (!ctx || !out || !id) return CGM_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(ctx, CGM_EINVAL, "cgm_comm_create: rank %d of %d", rank, nranks);
  NcclApi& n = nccl_api();
  if (!n.ok) return fail(ctx, CGM_ENCCL, "libnccl.so.2 not available");
  CGM_CUDA(ctx, cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  cgm_comm* c = new cgm_comm();
  const ncclResult_t r = n.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(ctx, CGM_ENCCL, "ncclCommInitRank: %s", n.GetErrorString(r));
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return CGM_OK;
}

int cgm_comm_destroy(cgm_comm* comm) {
  if (!comm) return CGM_OK;
  if (comm->comm && nccl_api().ok) nccl_api().CommDestroy(comm->comm);
  delete comm;
  return CGM_OK;
}

int cgm_gather(cgm_ctx* ctx, cgm_comm* comm, const void* send, const size_t* counts, void* recv,
               int root) {
  if (!ctx || !comm || !counts) return CGM_EINVAL;
  if (root < 0 || root >= comm->nranks)
    return fail(ctx, CGM_EINVAL, "cgm_gather: root %d of %d ranks", root, comm->nranks);
  NcclApi& n = nccl_api();
  CGM_CUDA(ctx, cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->user_stream;
  if (comm->rank == root) {
    if (!recv) return fail(ctx, CGM_EINVAL, "cgm_gather: root needs a receive buffer");
    size_t off = 0;
    CGM_NCCL(ctx, n.GroupStart());
    for (int r = 0; r < comm->nranks; ++r) {
      char* dst = static_cast<char*>(recv) + off;
      if (counts[r] > 0) {
        if (r == root) {
          const cudaError_t e = cudaMemcpyAsync(dst, send, counts[r], cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess) {
            n.GroupEnd();
            return fail(ctx, CGM_ECUDA, "cgm_gather: %s", cudaGetErrorString(e));
          }
        } else {
          const ncclResult_t rr = n.Recv(dst, counts[r], ncclInt8, r, comm->comm, st);
          if (rr != ncclSuccess) {
            n.GroupEnd();
            return fail(ctx, CGM_ENCCL, "ncclRecv: %s", n.GetErrorString(rr));
          }
        }
      }
      off += counts[r];
    }
    CGM_NCCL(ctx, n.GroupEnd());
  } else if (counts[comm->rank] > 0) {
    CGM_NCCL(ctx, n.GroupStart());
    const ncclResult_t rs = n.Send(send, counts[comm->rank], ncclInt8, root, comm->comm, st);
    if (rs != ncclSuccess) {
      n.GroupEnd();
      return fail(ctx, CGM_ENCCL, "ncclSend: %s", n.GetErrorString(rs));
    }
    CGM_NCCL(ctx, n.GroupEnd());
  }
  return CGM_OK;
}

}  // extern "C"
