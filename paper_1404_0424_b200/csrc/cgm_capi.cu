// cgm_capi.cu -- host runtime behind include/cgmimo_b200.h: contexts and
// streams, argument validation with the reference's error semantics,
// template dispatch of the fused subcarrier kernel, the chunked host-buffer
// pipeline (H2D / kernel / D2H overlapped on two streams) and the seeded
// device input generators.
#include <cuda.h>  // CUtensorMap types only (the encoder comes from cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>
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
#include "cgm_block32.cuh"
#include "cgm_moments.cuh"
#include "cgm_precode_small.cuh"
#include "cgm_uplink_small.cuh"
#include "cgm_tc64.cuh"
#include "cgm_rows32.cuh"
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
  float* tscratch = nullptr;  // split-path workspace (grown, never freed while the context lives)
  size_t tscratch_bytes = 0;
  std::vector<void*> retired;  // outgrown workspaces (possibly referenced by captured graphs)
  long launches = 0;
  int policy = 0;  // kernel-variant switches (kPol*), 0 = production defaults
  int host_chunks = 0;  // CGMIMO_HOST_CHUNKS, read once at context creation
  size_t host_set_bytes = 384ull << 20;  // host pipeline: device bytes per buffer set (CGMIMO_HOST_SET_MB)
  size_t chunk_bytes = 1024ull << 20;  // split-path chunk budget (CGMIMO_CHUNK_MB)
  // optional per-kernel event timing (bench roofline): pairs of events per launch
  int profiling = 0;
  cudaEvent_t order_ev = nullptr;  // host pipeline: ordered after the context stream's work
  // split path: consecutive chunks alternate between two streams (and two
  // workspace halves), so one chunk's HBM-bound tail kernels overlap the
  // next chunk's compute-bound head kernels
  cudaStream_t chunk_st[2] = {nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[2] = {nullptr, nullptr};
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

// 2-D tensor map of an H_u block [rows][32 complex] for the precoder's TMA
// tiles: FP32 elements, inner extent 64 (one 256-byte antenna row), box
// 32 x B (users 0-15 or 16-31 of all B rows of one subcarrier: 128-byte
// rows), SWIZZLE_128B.  cuTensorMapEncodeTiled is resolved through the
// runtime (no libcuda link).
bool encode_h_tiles(CUtensorMap* m, const float2* H, long rows, int B) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!enc) return false;
  const cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(B)};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(H), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Kernel-variant switches (cgm_ctx_set_kernel_policy): A/B alternatives kept
// for parity tests and measurements, never selected by default.
constexpr int kPolFfmaChannel = 1;  // U = 32: FFMA channel kernel instead of tcgen05
constexpr int kPolSplitSmall = 2;   // U <= 16: channel + solve pair instead of the fused kernels
constexpr int kPolLaneSolve = 4;    // U = 32: lane-per-row solve kernel instead of the row kernels
constexpr int kPolBlockUp = 8;      // U = 32 uplink only: the shared-G block kernel instead of pairs
constexpr int kPolRowsCta = 16;     // U = 32 with transmit vectors: the 8-warp row CTA instead of block
constexpr int kPolPoisonWs = 32;    // test only: fill the workspace with NaN before every chunk
constexpr int kPolTileMoments = 64; // U = 32, FP32 moments: the 4x4-tile CTA kernel instead of warp rows
constexpr int kPolSerialChunks = 128;  // split path: every chunk on the call's stream (no two-stream overlap)
constexpr int kPolUntiledCg = 256;     // cfg5 block CG: lane-per-row 8-warp kernel instead of the tiled one
constexpr int kPolPairsCg = 512;       // cfg2 (approximate, uplink only): warp-per-pair kernel instead of the tiled block CG

// Device workspace of the split path.  A call captured into a CUDA graph
// bakes in this pointer, so a larger call never frees it: the old buffer
// is retired (kept until the context is destroyed) and the new one grown by
// at least 1.5x (graphs replayed after a larger call).
int ensure_ws(cgm_ctx* ctx, size_t need) {
  if (need <= ctx->tscratch_bytes) return CGM_OK;
  const size_t want = std::max(need, ctx->tscratch_bytes + ctx->tscratch_bytes / 2);
  void* p = nullptr;
  CGM_CUDA(ctx, cudaMalloc(&p, want));
  if (ctx->tscratch) ctx->retired.push_back(ctx->tscratch);
  ctx->tscratch = static_cast<float*>(p);
  ctx->tscratch_bytes = want;
  return CGM_OK;
}

// one timed launch: CUDA events around it on `st` when profiling (kind 1
// channel, 2 solve, 3 exact-tracker moments, 4 the separate precoder kernel)
template <class F>
int timed(cgm_ctx* ctx, cudaStream_t st, int kind, F&& go) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profiling) {
    e0 = prof_event(ctx);
    e1 = prof_event(ctx);
    cudaEventRecord(e0, st);
  }
  go();
  CGM_CUDA(ctx, cudaGetLastError());
  if (ctx->profiling) {
    cudaEventRecord(e1, st);
    ctx->ev_log.push_back({kind, {e0, e1}});
  }
  ++ctx->launches;
  return CGM_OK;
}

// Split path, per chunk of subcarriers:
//   K1 channel kernel   G = H^H H (+ rho^-1 I in the CG), matched filters
//                       (tcgen05 for U = 32 natural layout, FFMA otherwise)
//   KM moments kernel   exact tracker only: (c, d) and the row moments
//                       D_k[i] of the Chebyshev basis (cgm_moments.cuh)
//   K2 solve kernel     CG + tracker extraction + LLRs (+ precoder tail)
// The chunk is sized so the workspace, H (re-read by the precoder tail) and
// Y of a chunk stay resident in the 126 MB L2 between the kernels.
template <int UP, bool EXACT>
int launch_split(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  const int Kmax = std::max(p.K, p.Kt);
  p.exact = EXACT ? 1 : 0;
  // one vector per subcarrier: the CG runs before the moments kernel, which
  // then does the per-vector extraction itself (moments_kernel<..., FX>) --
  // except for U = 32 with K <= 6, where the warp-per-subcarrier row-moment
  // kernel (FP32 moment table) and the pairs kernel's extraction are faster
  // (cfg4a K = 4: 2.66 -> see DESIGN s12)
  const bool rows_moments = UP == 32 && p.K <= cgm::kLaneK && !(ctx->policy & kPolTileMoments);
  p.fx = (EXACT && p.S == 1 && p.St == 0 && !rows_moments) ? 1 : 0;
  // ------------------------------------------------------------------ K1
  cgm::K1Split sp;
  sp.plan(UP, p.B, p.S);
  cgm::K1Smem<UP> L1;
  L1.plan(p.B, p.S, 2);
  if (L1.total > ctx->max_smem) {  // very large B: single stage
    sp.nstage = 1;
    L1.plan(p.B, p.S, 1);
  }
  p.k1_pair = sp.nstage;
  p.k1_spl = sp.spl;
  p.k1_wpp = sp.wpp;
  int nt1 = 32 * sp.wpp, smem1 = L1.total;
  void (*k1)(cgm::KernelParams) = cgm::channel_kernel<UP, EXACT>;
  bool use_tc = false;
  if constexpr (UP == 32) {
    // the tensor-core kernel stages Y per 64-antenna block (64 S complex,
    // always a 16-byte multiple), so odd S is fine there (cfg4: S = 1)
    const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
    const int tc_tma = (!p.hd_layout && p.U == UP && (al & 15u) == 0) ? 1 : 0;
    if (cgm::tc::supported(p.U, p.B, p.S, tc_tma) && !(ctx->policy & kPolFfmaChannel)) {
      cgm::tc::Smem T;
      int nstg = 4;  // staging depth: 4 / 3 / 2 as shared memory allows (cfg2 channel 0.430 -> 0.417 ms from 3 to 4)
      T.plan(p.S, nstg);
      if (T.total > ctx->max_smem) T.plan(p.S, nstg = 3);
      if (T.total > ctx->max_smem) T.plan(p.S, nstg = 2);
      if (T.total <= ctx->max_smem) {
        use_tc = true;
        p.k1_pair = nstg;
        smem1 = T.total;
        // split / epilogue warps, measured (tools/microbench/tc_bench.cu,
        // bench.py): approximate 16 unified (cfg2 37.9 vs 39.4 us for 8 + 8
        // specialised); exact 16 unified for few vectors per subcarrier
        // (cfg4a, 65,536 subcarriers: 0.86 ms against 0.925 for 8 unified and
        // 0.96 for 8 + 8), 8 + 8 specialised from S = 8 on
        if (!EXACT) {
          k1 = cgm::channel_tc_kernel<16, 0>;
          nt1 = 32 * 18;
        } else if (p.S >= 8) {
          k1 = cgm::channel_tc_kernel<8, 8>;
          nt1 = 32 * 18;
        } else {
          k1 = cgm::channel_tc_kernel<16, 0>;
          nt1 = 32 * 18;
        }
      }
    }
  }
  if constexpr (UP == 64) {
    // U = 64 natural layout: the M = 128 tensor-core kernel (cgm_tc64.cuh)
    const uintptr_t al = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
    const int tc_tma = (!p.hd_layout && p.U == UP && (al & 15u) == 0) ? 1 : 0;
    if (cgm::tc64::supported(p.U, p.B, p.S, tc_tma) && !(ctx->policy & kPolFfmaChannel)) {
      cgm::tc64::Smem T;
      int nstg = 3;
      T.plan(p.S, nstg);
      if (T.total > ctx->max_smem) T.plan(p.S, nstg = 2);
      if (T.total <= ctx->max_smem) {
        use_tc = true;
        p.k1_pair = nstg;
        smem1 = T.total;
        k1 = cgm::channel_tc64_kernel;
        nt1 = cgm::tc64::NT;
      }
    }
  }
  int occ1 = 0;
  CGM_PREP(ctx, k1, nt1, smem1, &occ1);
  if (occ1 < 1) return fail(ctx, CGM_EINVAL, "channel kernel does not fit on an SM");
  if (use_tc) occ1 = 1;  // one CTA (and all 512 TMEM columns) per SM
  // ------------------------------------------------------------------ KM
  void (*km)(cgm::KernelParams) = nullptr;
  int nm_t = 0, nm_smem = 0, nm_spc = 1;
  if constexpr (EXACT) {
    if (p.S > 0) {
      using MG = cgm::MomGeo<UP>;
      // moment table: FP32 products up to K = 6, FP64 beyond; FX (one
      // vector per subcarrier): FP32 entrywise sums (cgm_moments.cuh)
      const bool dbl = !p.fx && p.K > 6;
      km = p.fx ? cgm::moments_kernel<UP, float, true>
                : dbl ? cgm::moments_kernel<UP, double> : cgm::moments_kernel<UP, float>;
      nm_smem = dbl ? MG::template smem<double>() : MG::template smem<float>();
      nm_t = MG::NT;
      nm_spc = MG::SPC;
      if constexpr (UP == 32) {
        if (!p.fx && !dbl && !(ctx->policy & kPolTileMoments)) {  // warp per subcarrier
          km = cgm::moments_rows32_kernel;
          nm_smem = cgm::MomRowsSmem::TOTAL;
          nm_t = 32 * cgm::kMrW;
          nm_spc = cgm::kMrW;
        }
      }
      if (nm_smem > ctx->max_smem)
        return fail(ctx, CGM_EINVAL, "exact tracker: %d B of shared memory per moments CTA exceed %d",
                    nm_smem, ctx->max_smem);
      CGM_PREP(ctx, km, nm_t, nm_smem, nullptr);
    }
  }
  // ------------------------------------------------------------------ K2
  // U = 32 (default): the Gram row lives in registers (cgm_rows32.cuh) --
  // uplink only: one warp per (subcarrier, pair of systems) (one system for
  // S = 1), outputs from the warp; with downlink systems: one 8-warp CTA per
  // subcarrier with the precoder tail.  Otherwise the lane-per-row kernel
  // (cgm_split.cuh), persistent with a prefetched workspace from 24
  // systems per subcarrier on.
  cgm::K2Smem<UP> L2;
  L2.plan(p.B, p.S, p.St, Kmax, EXACT);
  if (L2.total > ctx->max_smem)
    return fail(ctx, CGM_EINVAL, "per-subcarrier working set (%d B) exceeds shared memory (%d B)",
                L2.total, ctx->max_smem);
  void (*k2)(cgm::KernelParams) = cgm::solve_kernel<UP, EXACT>;
  int smem2 = L2.total;
  enum { kLanes, kLanesPf, kPairs, kRowsCta, kBlock, kBlockT, kBlockA } mode = kLanes;
  int pair_ns = 2;
  if constexpr (UP == 32) {
    // persistent shared-G block kernel (+ precode_q_kernel for transmit
    // vectors): its bulk copies need 16-byte aligned T rows and H rows
    cgm::WsOffsets WB;
    WB.plan(UP, p.S, p.K, EXACT, p.fx, p.St);
    cgm::Block32Smem BL;
    BL.plan(p.S, p.St, Kmax, EXACT, WB.z * 8);
    const uintptr_t alt = reinterpret_cast<uintptr_t>(p.T) | reinterpret_cast<uintptr_t>(p.H);
    const bool block_ok = BL.total <= ctx->max_smem && p.U == 32 && !p.hd_layout && !p.fx &&
                          (p.St == 0 || (p.B <= 256 && (alt & 15u) == 0));
    if (!(ctx->policy & kPolLaneSolve) && block_ok &&
        (p.St > 0 ? !(ctx->policy & kPolRowsCta) : (ctx->policy & kPolBlockUp) != 0)) {
      mode = kBlock;
      k2 = cgm::block32_kernel<EXACT>;
      smem2 = BL.total;
      p.zs = p.St;  // the transmit vectors' v_K go through the workspace
      if constexpr (EXACT) {
        cgm::Block32TSmem BT;
        BT.plan(p.S, p.St, Kmax, WB.z * 8);
        if (!(ctx->policy & kPolUntiledCg) && BT.total <= ctx->max_smem) {  // register-tiled CG
          mode = kBlockT;
          k2 = cgm::block32t_kernel;
          smem2 = BT.total;
        }
      }
    } else if (!(ctx->policy & kPolLaneSolve)) {
      cgm::Block32ASmem BA;
      BA.plan(p.S, WB.z * 8);
      if (!EXACT && p.St == 0 && p.S >= 2 && p.U == 32 && !(ctx->policy & kPolPairsCg) &&
          BA.total <= ctx->max_smem) {
        // approximate tracker, several vectors per subcarrier (cfg2): the
        // register-tiled block CG, ceil(S / 8) warps per CTA
        mode = kBlockA;
        k2 = cgm::block32a_kernel;
        smem2 = BA.total;
      } else if (p.St == 0) {
        mode = kPairs;
        pair_ns = p.S == 1 ? 1 : 2;
        k2 = pair_ns == 1 ? cgm::solve_rows32_pairs_kernel<EXACT, 1>
                          : cgm::solve_rows32_pairs_kernel<EXACT, 2>;
        smem2 = 0;
      } else {
        cgm::Rows32Smem R;
        R.plan(p.B, p.S, p.St, Kmax, EXACT);
        if (R.total <= ctx->max_smem) {
          mode = kRowsCta;
          k2 = cgm::solve_rows32_kernel<EXACT>;
          smem2 = R.total;
        }
      }
    }
  }
  if (mode == kLanes && p.S + p.St >= 24) {
    const int need = 128 + 2 * cgm::k2_pre_bytes(UP, p.S) + L2.total;
    if (need <= ctx->max_smem) {
      mode = kLanesPf;
      k2 = cgm::solve_kernel_pf<UP, EXACT>;
      smem2 = need;
    }
  }
  CGM_PREP(ctx, k2, 32, smem2, nullptr);
  // K2 block: lanes kernel -- enough lane groups for every system (>= UP
  // threads for the exact extraction), at most 8 warps; row CTA kernel: 8
  // warps from 16 systems on
  using GE = cgm::K2Geo<UP>;
  const int nsys = p.S + p.St;
  int nw2 = (nsys + GE::GPW * GE::NS - 1) / (GE::GPW * GE::NS);
  if (EXACT) nw2 = std::max(nw2, std::max(4, UP / 32));
  nw2 = std::max(1, std::min(8, nw2));
  if (mode == kRowsCta) nw2 = nsys >= 16 ? 8 : 2;
  if (mode == kBlock)  // NS systems per warp
    nw2 = std::min(cgm::kBlkMaxW, (nsys + cgm::kBlkNS - 1) / cgm::kBlkNS);
  if (mode == kBlockT) nw2 = cgm::kTWarps;
  if (mode == kBlockA) nw2 = std::min(cgm::kTWarps, (nsys + cgm::kTSpw - 1) / cgm::kTSpw);
  long g2cap = 1L << 40;
  CUtensorMap tmH{};
  auto pq_kernel = cgm::precode_q_kernel<2>;
  if (mode == kBlock || mode == kBlockT || mode == kBlockA) {  // persistent
    int occ2 = 0;
    CGM_PREP(ctx, k2, 32 * nw2, smem2, &occ2);
    g2cap = static_cast<long>(std::max(occ2, 1)) * ctx->sms;
    if (p.St > 0) {
      cgm::PrecodeQSmem PQ;
      PQ.plan(p.B, p.St);
      if (PQ.total > ctx->max_smem)
        return fail(ctx, CGM_EINVAL, "precoder: %d B of shared memory exceed %d", PQ.total, ctx->max_smem);
      CGM_PREP(ctx, pq_kernel, cgm::PrecodeQSmem::NTH, PQ.total, nullptr);
      if (!encode_h_tiles(&tmH, p.H, p.n_sc * static_cast<long>(p.B), p.B))
        return fail(ctx, CGM_ECUDA, "cuTensorMapEncodeTiled failed for the precoder's H tiles");
    }
  }
  if (mode == kLanesPf) {
    int occ2 = 0;
    CGM_PREP(ctx, k2, 32 * nw2, smem2, &occ2);
    g2cap = static_cast<long>(std::max(occ2, 1)) * ctx->sms;
  }
  // --------------------------------------------------------------- chunks
  cgm::WsOffsets W;
  W.plan(UP, p.S, p.K, EXACT, p.fx, p.zs);
  const size_t per_sc = static_cast<size_t>(W.stride) * 8 + static_cast<size_t>(p.B) * p.U * 8 +
                        static_cast<size_t>(p.B) * p.S * 8;
  long chunk = static_cast<long>(ctx->chunk_bytes / std::max<size_t>(per_sc, 1));
  chunk = std::max<long>(chunk, static_cast<long>(ctx->sms) * occ1);
  // a call that fits one chunk but is large (a GPU's shard of cfg5 at 8 GPUs)
  // still splits in two, so the two chunk streams overlap its kernels
  if (!(ctx->policy & kPolSerialChunks) && p.n_sc <= chunk && p.n_sc >= 32L * ctx->sms)
    chunk = (p.n_sc + 1) / 2;
  chunk = std::min(chunk, p.n_sc);
  // two or more chunks: alternate two streams and workspace halves (fork from
  // and join back into the call's stream; captures into a CUDA graph as a
  // fork/join)
  const bool dual = p.n_sc > chunk && !(ctx->policy & kPolSerialChunks);
  const size_t ws_half = static_cast<size_t>(chunk) * W.stride;  // float2 per workspace half
  const int rc = ensure_ws(ctx, (dual ? 2 : 1) * ws_half * sizeof(float2));
  if (rc) return rc;
  const cudaStream_t call_st = st;
  if (dual) {
    CGM_CUDA(ctx, cudaEventRecord(ctx->fork_ev, call_st));
    for (int k = 0; k < 2; ++k) CGM_CUDA(ctx, cudaStreamWaitEvent(ctx->chunk_st[k], ctx->fork_ev, 0));
  }
  int ci = 0;
  for (long c0 = 0; c0 < p.n_sc; c0 += chunk, ++ci) {
    const long n = std::min(chunk, p.n_sc - c0);
    st = dual ? ctx->chunk_st[ci & 1] : call_st;
    p.ws = reinterpret_cast<float2*>(ctx->tscratch) + (dual ? (ci & 1) * ws_half : 0);
    // poisoned workspace: a kernel reading workspace it did not write first
    // turns its outputs into NaN (tests compare against an unpoisoned run)
    if (ctx->policy & kPolPoisonWs)
      CGM_CUDA(ctx, cudaMemsetAsync(p.ws, 0xFF, static_cast<size_t>(n) * W.stride * 8, st));
    cgm::KernelParams q = p;
    q.sc_base = c0;
    q.n_sc = n;
    const long g1 = std::max<long>(1, std::min<long>(n, static_cast<long>(occ1) * ctx->sms));
    int r = timed(ctx, st, 1, [&] { k1<<<static_cast<unsigned>(g1), nt1, smem1, st>>>(q); });
    if (r) return r;
    auto moments = [&] {
      return timed(ctx, st, 3, [&] {
        km<<<static_cast<unsigned>((n + nm_spc - 1) / nm_spc), nm_t, nm_smem, st>>>(q);
      });
    };
    if (km && !p.fx && (r = moments())) return r;
    r = timed(ctx, st, 2, [&] {
      if (mode == kPairs)  // 4 warps per CTA, one (subcarrier, system group) per warp
        k2<<<static_cast<unsigned>((n * ((p.S + pair_ns - 1) / pair_ns) + 3) / 4), 128, 0, st>>>(q);
      else
        k2<<<static_cast<unsigned>(std::min(n, g2cap)), 32 * nw2, smem2, st>>>(q);
    });
    if (r) return r;
    if ((mode == kBlock || mode == kBlockT) && p.St > 0) {  // q = H_d^H v, gain, s
      cgm::PrecodeQSmem PQ;
      PQ.plan(p.B, p.St);
      r = timed(ctx, st, 4, [&] {
        pq_kernel<<<static_cast<unsigned>(n), cgm::PrecodeQSmem::NTH, PQ.total, st>>>(q, tmH);
      });
      if (r) return r;
    }
    if (km && p.fx && (r = moments())) return r;
  }
  if (dual) {
    for (int k = 0; k < 2; ++k) {
      CGM_CUDA(ctx, cudaEventRecord(ctx->join_ev[k], ctx->chunk_st[k]));
      CGM_CUDA(ctx, cudaStreamWaitEvent(call_st, ctx->join_ev[k], 0));
    }
  }
  return CGM_OK;
}

template <int UP>
int dispatch_split(cgm_ctx* ctx, cgm::KernelParams& p, bool exact, cudaStream_t st) {
  return exact ? launch_split<UP, true>(ctx, p, st) : launch_split<UP, false>(ctx, p, st);
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
  return timed(ctx, st, 2, [&] { k<<<static_cast<unsigned>(grid), cgm::alt::NT, smem, st>>>(p); });
}

// Fused small-U CG precoder (cgm_precode_small.cuh): pure precode calls with
// H_d in the reference layout, U <= 16, one warp per subcarrier.
bool precode_small_ok(cgm_ctx* ctx, const cgm::KernelParams& p) {
  if (!(p.S == 0 && p.St > 0 && p.hd_layout && p.U <= 16 && p.B <= 512 && p.B >= 4 && p.B % 2 == 0))
    return false;
  if (ctx->policy & kPolSplitSmall) return false;
  cgm::PrecodeSmallSmem L;
  L.plan(up_of(p.U), p.B, p.St);
  return L.total <= ctx->max_smem;
}

template <int UP>
int launch_precode_small(cgm_ctx* ctx, cgm::KernelParams p, cudaStream_t st) {
  cgm::PrecodeSmallSmem L;
  L.plan(UP, p.B, p.St);
  // q of an antenna pass in registers: 4 chunks of 32 antennas up to B = 128, else 16
  auto k = p.B <= 128 ? cgm::precode_small_kernel<UP, 4> : cgm::precode_small_kernel<UP, 16>;
  int occ = 0;
  CGM_PREP(ctx, k, cgm::PrecodeSmallGeo<UP>::NT, L.total, &occ);
  const long grid = std::max<long>(1, std::min<long>(p.n_sc, static_cast<long>(std::max(occ, 1)) * ctx->sms));
  p.use_tma = ((p.B % 2) == 0 && (reinterpret_cast<uintptr_t>(p.H) & 15u) == 0) ? 1 : 0;
  p.sc_base = 0;
  return timed(ctx, st, 2, [&] {
    k<<<static_cast<unsigned>(grid), cgm::PrecodeSmallGeo<UP>::NT, L.total, st>>>(p);
  });
}

// Fused small-U CG detector (cgm_uplink_small.cuh): uplink-only calls with
// U <= 16, one warp per subcarrier.
bool uplink_small_ok(cgm_ctx* ctx, const cgm::KernelParams& p, bool exact) {
  if (!(p.St == 0 && p.S >= 1 && !p.hd_layout && p.U <= 16 && p.K >= 1 && p.K <= cgm::kMaxK))
    return false;
  if (ctx->policy & kPolSplitSmall) return false;
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
  return timed(ctx, st, 2, [&] { k<<<static_cast<unsigned>(grid), 32, L.total, st>>>(p); });
}

int launch(cgm_ctx* ctx, cgm::KernelParams& p, bool exact, cudaStream_t st) {
  if (p.n_sc <= 0) return CGM_OK;
  if (p.method != cgm::alt::kCg) return launch_alt(ctx, p, st);
  const int UP = up_of(p.U);
  if (uplink_small_ok(ctx, p, exact)) {
    if (UP == 8) return exact ? launch_uplink_small<8, true>(ctx, p, st) : launch_uplink_small<8, false>(ctx, p, st);
    return exact ? launch_uplink_small<16, true>(ctx, p, st) : launch_uplink_small<16, false>(ctx, p, st);
  }
  if (precode_small_ok(ctx, p))
    return UP == 8 ? launch_precode_small<8>(ctx, p, st) : launch_precode_small<16>(ctx, p, st);
  const uintptr_t a = reinterpret_cast<uintptr_t>(p.H) | reinterpret_cast<uintptr_t>(p.Y);
  // 1: H and Y by bulk copy; 2 (odd S, channel_kernel only): H by bulk copy,
  // the padded Y rows by the threads
  p.use_tma = (!p.hd_layout && p.U == UP && (p.B % 2) == 0 && (a & 15u) == 0)
                  ? ((p.S % 2) == 0 ? 1 : 2) : 0;
  switch (UP) {
    case 8: return dispatch_split<8>(ctx, p, exact, st);
    case 16: return dispatch_split<16>(ctx, p, exact, st);
    case 32: return dispatch_split<32>(ctx, p, exact, st);
    default: return dispatch_split<64>(ctx, p, exact, st);
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
  const size_t budget = ctx->host_set_bytes;  // per buffer set (CGMIMO_HOST_SET_MB)
  long chunk = static_cast<long>(std::max<size_t>(1, budget / std::max<size_t>(per_sc, 1)));
  chunk = std::min(chunk, j.n_sc);
  // up to 8 chunks of at least ~8 MB each: small batches are bound by the
  // per-chunk API calls, not by the copy overlap (cfg1, 9.4 MB: one chunk
  // 4.1 M vec/s against 3.2 M with eight)
  const size_t total_bytes = per_sc * static_cast<size_t>(j.n_sc);
  int nch = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, total_bytes / (8ull << 20))));
  if (ctx->host_chunks > 0) nch = ctx->host_chunks;
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
  // the pipeline shares the split-path workspace with asynchronous
  // device-pointer calls on the context stream: order after them
  if (!ctx->order_ev) CGM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->order_ev, cudaEventDisableTiming));
  CGM_CUDA(ctx, cudaEventRecord(ctx->order_ev, ctx->user_stream));
  CGM_CUDA(ctx, cudaStreamWaitEvent(s_in, ctx->order_ev, 0));
  CGM_CUDA(ctx, cudaStreamWaitEvent(s_comp, ctx->order_ev, 0));
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
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&ctx->chunk_st[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->join_ev[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
  if (const char* hc = std::getenv("CGMIMO_HOST_CHUNKS")) ctx->host_chunks = std::max(0, std::atoi(hc));
  if (const char* hs = std::getenv("CGMIMO_HOST_SET_MB"))
    ctx->host_set_bytes = static_cast<size_t>(std::max(8, std::atoi(hs))) << 20;
  if (const char* cm = std::getenv("CGMIMO_CHUNK_MB")) ctx->chunk_bytes = static_cast<size_t>(std::max(1, std::atoi(cm))) << 20;
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
  for (int i = 0; i < 2; ++i) {
    if (ctx->chunk_st[i]) cudaStreamDestroy(ctx->chunk_st[i]);
    if (ctx->join_ev[i]) cudaEventDestroy(ctx->join_ev[i]);
  }
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->tscratch) cudaFree(ctx->tscratch);
  for (void* r : ctx->retired) cudaFree(r);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->order_ev) cudaEventDestroy(ctx->order_ev);
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
    (rec.first == 1 ? *channel_ms : rec.first == 3 ? *basis_ms : *solve_ms) += ms;  // 2, 4: solve
    if (rec.first == 1) ++*launches;
  }
  return CGM_OK;
}

int cgm_ctx_kernel_times_kinds(cgm_ctx* ctx, double ms[4], long* launches) {
  if (!ctx || !ms || !launches) return CGM_EINVAL;
  for (int k = 0; k < 4; ++k) ms[k] = 0.0;
  *launches = 0;
  for (auto& rec : ctx->ev_log) {
    CGM_CUDA(ctx, cudaEventSynchronize(rec.second.second));
    float t = 0.f;
    CGM_CUDA(ctx, cudaEventElapsedTime(&t, rec.second.first, rec.second.second));
    static constexpr int slot[5] = {-1, 0, 2, 1, 3};  // kind 1 channel, 2 solve, 3 moments, 4 precoder
    if (rec.first >= 1 && rec.first <= 4) ms[slot[rec.first]] += t;
    if (rec.first == 1) ++*launches;
  }
  return CGM_OK;
}

int cgm_ctx_kernel_timeline(cgm_ctx* ctx, int* kinds, double* start_ms, double* end_ms, long cap,
                            long* n) {
  if (!ctx || !n || cap < 0 || (cap > 0 && (!kinds || !start_ms || !end_ms))) return CGM_EINVAL;
  *n = static_cast<long>(ctx->ev_log.size());
  if (ctx->ev_log.empty()) return CGM_OK;
  const cudaEvent_t t0 = ctx->ev_log.front().second.first;
  long i = 0;
  for (auto& rec : ctx->ev_log) {
    if (i >= cap) break;
    CGM_CUDA(ctx, cudaEventSynchronize(rec.second.second));
    float a = 0.f, b = 0.f;
    CGM_CUDA(ctx, cudaEventElapsedTime(&a, t0, rec.second.first));
    CGM_CUDA(ctx, cudaEventElapsedTime(&b, t0, rec.second.second));
    kinds[i] = rec.first;
    start_ms[i] = a;
    end_ms[i] = b;
    ++i;
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
  if (!ctx || policy < 0 ||
      policy > (kPolFfmaChannel | kPolSplitSmall | kPolLaneSolve | kPolBlockUp | kPolRowsCta | kPolTileMoments |
                kPolSerialChunks | kPolUntiledCg | kPolPairsCg |
                kPolPoisonWs))
    return fail(ctx, CGM_EINVAL, "unknown kernel policy %d", policy);
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

int cgm_gatherv(cgm_ctx* ctx, cgm_comm* comm, const void* send, const size_t* counts,
                const size_t* displs, void* recv, int root) {
  if (!ctx || !comm || !counts || !displs) return CGM_EINVAL;
  if (root < 0 || root >= comm->nranks)
    return fail(ctx, CGM_EINVAL, "cgm_gather: root %d of %d ranks", root, comm->nranks);
  NcclApi& n = nccl_api();
  CGM_CUDA(ctx, cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->user_stream;
  if (comm->rank == root) {
    if (!recv) return fail(ctx, CGM_EINVAL, "cgm_gather: root needs a receive buffer");
    CGM_NCCL(ctx, n.GroupStart());
    for (int r = 0; r < comm->nranks; ++r) {
      char* dst = static_cast<char*>(recv) + displs[r];
      if (counts[r] == 0) continue;
      if (r == root) {
        if (dst == send) continue;  // already in place
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

int cgm_gather(cgm_ctx* ctx, cgm_comm* comm, const void* send, const size_t* counts, void* recv,
               int root) {
  if (!ctx || !comm || !counts) return CGM_EINVAL;
  std::vector<size_t> displs(static_cast<size_t>(std::max(comm->nranks, 0)));
  size_t off = 0;
  for (int r = 0; r < comm->nranks; ++r) {
    displs[r] = off;
    off += counts[r];
  }
  return cgm_gatherv(ctx, comm, send, counts, displs.data(), recv, root);
}

}  // extern "C"
