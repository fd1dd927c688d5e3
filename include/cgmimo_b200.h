/* cgmimo_b200.h -- C ABI of the B200 (sm_100a) CG detection / precoding path.
 *
 * This is the drop-in boundary: plain pointers, sizes and int status codes,
 * no CUDA or C++ types in any signature.  Each entry point replaces a
 * reference interface of /root/reference/proj (cited per function); the C++
 * drop-in headers in include/cgmimo/ (same signatures as the reference's
 * cgmimo::detect / cgmimo::precode) are implemented on top of it, and
 * INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Layouts (complex64 = interleaved float re,im; all arrays dense, row-major):
 *   H  uplink   [n_sc][B][U]   element (b,u) at b*U+u   (reference linalg.hpp:28)
 *   Hd downlink [n_sc][U][B]   element (u,b) at u*B+b   (precode.hpp:31, H_d is U x B)
 *   Y  [n_sc][B][S]            antenna-major: column s of the B x S matrix is the
 *                              s-th received vector sharing channel sc
 *   T  [n_sc][S][U]            the S transmit-symbol vectors t of channel sc
 *   xhat [n_sc][S][U] complex64, mu / rho [n_sc][S][U] float,
 *   llr  [n_sc][S][U][qam_bits] float (I-axis bits MSB first, then Q-axis bits),
 *   q / s [n_sc][S][B] complex64, gain [n_sc][S] float,
 *   status [n_sc][S] uint8: bit0 = solver breakdown (outputs zeroed; the
 *   reference throws solvers::SolverBreakdown, solvers.cpp:55-57),
 *   bit1 = zero_input (precode, precode.cpp:25-31).
 * Any output pointer may be NULL to skip that output.
 *
 * Memory spaces: without CGM_DEVICE_POINTERS every array is a HOST pointer
 * and the call is synchronous (host->device copies, kernels and device->host
 * copies are pipelined in chunks inside the call).  With CGM_DEVICE_POINTERS
 * every array is a device pointer on the context's device and the call only
 * enqueues work on the context stream (cgm_ctx_set_stream).
 *
 * Numerics: complex64 / FP32 arithmetic (the reference is FP64); see
 * DESIGN.md for the tolerance contract.  The reference's 1e-9
 * imaginary-part check on p^H A p (solvers.cpp:29-35) is not applied: A is
 * Hermitian by construction.
 */
#ifndef CGMIMO_B200_H
#define CGMIMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define CGM_OK 0
#define CGM_EINVAL 1     /* std::invalid_argument in the reference (detect.cpp:186-188) */
#define CGM_EBREAKDOWN 2 /* solvers::SolverBreakdown (solvers.cpp:55-57), per-call API only */
#define CGM_ECUDA 3
#define CGM_ENCCL 4
#define CGM_ENOMEM 5

/* SinrTracker (detect.hpp:38): same enumerator order as the reference */
#define CGM_TRACKER_EXACT 0
#define CGM_TRACKER_APPROX 1

/* flags */
#define CGM_DEVICE_POINTERS 0x1u  /* arrays are device pointers; asynchronous */
#define CGM_HD_UPLINK_LAYOUT 0x2u /* precode: matrix given as H_u [B][U], H_d = H_u^H */

typedef struct cgm_ctx cgm_ctx;

/* One context per host thread (or stream): owns the stream, device
 * workspaces and the last-error string.  device = CUDA ordinal. */
int cgm_ctx_create(int device, cgm_ctx** out);
int cgm_ctx_destroy(cgm_ctx* ctx);
/* stream = cudaStream_t (0 = legacy default stream) */
int cgm_ctx_set_stream(cgm_ctx* ctx, void* stream);
int cgm_synchronize(cgm_ctx* ctx);
/* Kernel-variant switches for A/B tests (bit mask; 0 = production
 * defaults): 1 = FFMA channel kernel instead of tcgen05 for U = 32,
 * 2 = channel + solve pair instead of the fused U <= 16 kernels,
 * 4 = lane-per-row solve kernel instead of the U = 32 row kernels,
 * 8 = shared-G block kernel for uplink-only U = 32, 16 = 8-warp row CTA
 * instead of the block kernel, 64 = 4x4-tile moments kernel instead of the
 * warp-per-subcarrier one, 128 = every workspace chunk on the call's
 * stream, 256 = lane-per-row block CG instead of the register-tiled one
 * (exact tracker with transmit vectors), 512 = warp-per-pair kernel instead
 * of the register-tiled approximate block CG (32: test only, NaN-poisoned
 * workspace).  Every variant is parity-tested against the default. */
int cgm_ctx_set_kernel_policy(cgm_ctx* ctx, int policy);
/* Per-kernel device timing: while on, every channel/solve launch pair is
 * bracketed by CUDA events on the launch stream; cgm_ctx_kernel_times
 * synchronises and returns the summed milliseconds of each kernel and the
 * number of channel-kernel launches since profiling was (re)enabled. */
int cgm_ctx_set_profiling(cgm_ctx* ctx, int on);
int cgm_ctx_kernel_times(cgm_ctx* ctx, double* channel_ms, double* solve_ms, long* launches);
/* Same, with the exact tracker's row-moment kernel (cgm_moments.cuh)
 * reported on its own as basis_ms (cgm_ctx_kernel_times adds it to channel_ms). */
int cgm_ctx_kernel_times_ex(cgm_ctx* ctx, double* channel_ms, double* basis_ms, double* solve_ms,
                            long* launches);
/* Same, by kind: ms[0] channel, ms[1] exact-tracker moments, ms[2] solve
 * (CG, extraction, LLRs), ms[3] the separate precoder kernel (q = H_d^H v,
 * gain, s; cgm_ctx_kernel_times_ex counts it in solve_ms). */
int cgm_ctx_kernel_times_kinds(cgm_ctx* ctx, double ms[4], long* launches);
/* The same launches as a timeline: for launch i (up to cap), its kind (1
 * channel, 2 solve, 3 moments, 4 precoder) and start / end in ms relative to
 * the first recorded launch's start; *n = launches recorded (may exceed cap). */
int cgm_ctx_kernel_timeline(cgm_ctx* ctx, int* kinds, double* start_ms, double* end_ms, long cap,
                            long* n);
const char* cgm_last_error(const cgm_ctx* ctx);
/* kernels this context has launched since creation (the bench's gpu_launches) */
long cgm_kernel_launches(const cgm_ctx* ctx);
/* library version string, e.g. "cgmimo_b200 0.1 sm_100a" */
const char* cgm_version(void);

/* Batched detect::detect_cg (detect.hpp:58-61, detect.cpp:182-237):
 * Gram + matched filter, K CG iterations with the exact (Eq. 10) or
 * approximate (Eq. 11) SINR tracker, max-log LLRs (detect.cpp:68-86).
 * rho_u is the regulariser argument (A = H^H H + rho_u^-1 I), n0 / es the
 * noise and symbol energies; qam_bits in {2, 4, 6}. 1 <= U <= 64, K <= 16.
 * The exact tracker's per-vector U^3 recursion and extraction are computed
 * through per-subcarrier row moments of a Chebyshev basis. */
int cgm_detect_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* H,
                  const float* Y, double rho_u, double n0, double es, int qam_bits, int K,
                  int tracker, float* xhat, float* mu, float* rho, float* llr,
                  uint8_t* status, unsigned flags);

/* Batched precode::precode_cg (precode.hpp:31-33, precode.cpp:56-71):
 * A_d = H_d H_d^H + rho_d^-1 I, K CG iterations on t, q = H_d^H v_K,
 * gain = ||q||, s = q / gain (precode.cpp:22-36). */
int cgm_precode_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* Hd,
                   const float* T, double rho_d, int K, float* q, float* s, float* gain,
                   uint8_t* status, unsigned flags);

/* Uplink detection and downlink precoding on the SAME channels (TDD
 * reciprocity, H_d = H_u^H) in one pass: the Gram matrix is formed once per
 * subcarrier and shared by the S uplink and St downlink systems.  Equivalent
 * to cgm_detect_cg(...) followed by cgm_precode_cg(..., CGM_HD_UPLINK_LAYOUT). */
int cgm_detect_precode_cg(cgm_ctx* ctx, int B, int U, long n_sc, int S, const float* H,
                          const float* Y, double rho_u, double n0, double es, int qam_bits,
                          int K, int tracker, float* xhat, float* mu, float* rho, float* llr,
                          uint8_t* status, int St, const float* T, double rho_d, int Kt,
                          float* q, float* s, float* gain, uint8_t* pstatus, unsigned flags);

/* ---- the other solvers of the reference's trade-off study (SURVEY.md
 * section 8(f) row 4), same layouts, flags and status bytes as above, plus
 * status bit2 = not positive definite / zero diagonal (the reference throws
 * solvers::NotPositiveDefinite / std::domain_error, solvers.cpp:246-247,
 * :332-333).  method follows sim::Method (sim.hpp:34). */
#define CGM_METHOD_CHOLESKY 0 /* detect_cholesky (detect.cpp:122-181) / precode_explicit (precode.cpp:45-54) */
#define CGM_METHOD_CG 1       /* detect_cg / precode_cg: same as the _cg entry points */
#define CGM_METHOD_CGLS 2     /* detect_cgls (detect.cpp:238-272) / precode_cgls (precode.cpp:73-82) */
#define CGM_METHOD_NEUMANN 3  /* detect_neumann (detect.cpp:274-326) / precode_neumann (precode.cpp:84-93) */
/* iters = CG/CGLS iterations or Neumann series terms (ignored by Cholesky);
 * tracker is used by CG only (CGLS always runs the approximate tracker,
 * detect.cpp:258-263). */
int cgm_detect(cgm_ctx* ctx, int method, int B, int U, long n_sc, int S, const float* H,
               const float* Y, double rho_u, double n0, double es, int qam_bits, int iters,
               int tracker, float* xhat, float* mu, float* rho, float* llr, uint8_t* status,
               unsigned flags);
int cgm_precode(cgm_ctx* ctx, int method, int B, int U, long n_sc, int S, const float* Hd,
                const float* T, double rho_d, int iters, float* q, float* s, float* gain,
                uint8_t* status, unsigned flags);

/* Seeded synthetic inputs on the device (always device pointers, async),
 * following the reference's stream conventions (sim.cpp:151-179,
 * channel.cpp:10-30, rng.cpp): with root = Rng(seed),
 *   H(sc)       = rayleigh_channel(B, U, root.fork(2).fork(sc))   (row-major draws)
 *   labels(i)   : root.fork(1).fork(i), qam_bits draws of next_u64() & 1 per user
 *   noise(i)    : root.fork(3).fork(i), transmit() component std sqrt(N0/2)
 *   t labels(i) : root.fork(4).fork(i)
 * with instance index i = sc*S + s, so results do not depend on sharding.
 * sc0 offsets the subcarrier index (shard start).  labels may be NULL. */
int cgm_generate_uplink(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S, uint64_t seed,
                        int qam_bits, double n0, float* H, float* Y, uint8_t* labels);
/* Downlink: Hd(sc) = U x B rayleigh draws from root.fork(2).fork(sc); T from
 * labels root.fork(4).fork(i). */
int cgm_generate_downlink(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S,
                          uint64_t seed, int qam_bits, float* Hd, float* T, uint8_t* labels);
/* Downlink symbol vectors only (T [n_sc][S][U]) from root.fork(4). */
int cgm_generate_symbols(cgm_ctx* ctx, int U, long sc0, long n_sc, int S, uint64_t seed,
                         int qam_bits, float* T, uint8_t* labels);
/* BS-side correlated channel: H_u = (H_w R^{1/2})^H per subcarrier where
 * H_w (U x B) is drawn like cgm_generate_downlink's Hd and rsqrt is the
 * B x B real symmetric square root of R (row-major float).  Then Y is drawn
 * as in cgm_generate_uplink from the correlated channel. */
int cgm_generate_uplink_correlated(cgm_ctx* ctx, int B, int U, long sc0, long n_sc, int S,
                                   uint64_t seed, int qam_bits, double n0, const float* rsqrt,
                                   float* H, float* Y, uint8_t* labels);

/* ---- coded BLER harness: the reference's
 * run_uplink_trial (sim.cpp:147-203) for a batch of trials -- frames
 * (info bits, rate-5/6 convolutional code, interleaver), channel + noise from
 * the trial's streams, ONE batched detect_cg over all (symbol, subcarrier)
 * vectors, deinterleaving and a soft Viterbi decoder on the GPU.
 * trial_keys[t] = cgm_sweep_trial_key(seed, 1, point, trial) reproduces
 * run_uplink_sweep's trials (sim.cpp:378-380); snr_db per receive antenna
 * (N0 = U / SNR, rho_u = 1 / N0).  Outputs per trial: user_errors (blocks
 * of the U users decoded wrongly) and breakdown (1: a SolverBreakdown
 * aborted the trial, no errors counted, as sim.cpp:183-188).  Host arrays. */
int cgm_uplink_trials(cgm_ctx* ctx, int B, int U, int n_sc, int qam_bits, int K, int tracker,
                      double snr_db, long n_trials, const uint64_t* trial_keys,
                      uint32_t* user_errors, uint8_t* breakdown);
/* run_downlink_trial (sim.cpp:205-275) for a batch of trials: same frames
 * and streams, H_d = H^H of the trial's Rayleigh draws, ONE batched
 * precode_cg over all (symbol, subcarrier) transmit vectors, z = H_d s plus
 * noise per user, the genie demapper (gain z_u / t_u, LLRs of y_u / gain at
 * rho = |gain|^2 / N0), deinterleaving and soft Viterbi.  snr_db per user
 * (N0 = 1 / SNR, rho_d = 1 / N0); trial_keys[t] = cgm_sweep_trial_key(seed,
 * 2, point, trial) (sim.cpp:397-399). */
int cgm_downlink_trials(cgm_ctx* ctx, int B, int U, int n_sc, int qam_bits, int K,
                        double snr_db, long n_trials, const uint64_t* trial_keys,
                        uint32_t* user_errors, uint8_t* breakdown);
/* Either direction with any sim::Method (the trade-off study, sim.cpp:
 * 120-145): direction 1 = uplink (cgm_detect with `method`, `iters`,
 * `tracker`), 2 = downlink (cgm_precode with `method`, `iters`).  A solver
 * input that is not positive definite (status bit2) fails the call with
 * CGM_EINVAL, as the reference's exception leaves run_point. */
int cgm_sweep_trials(cgm_ctx* ctx, int direction, int method, int B, int U, int n_sc,
                     int qam_bits, int iters, int tracker, double snr_db, long n_trials,
                     const uint64_t* trial_keys, uint32_t* user_errors, uint8_t* breakdown);
uint64_t cgm_sweep_trial_key(uint64_t seed, int direction, long point, long trial);
/* Soft max-log Viterbi decoding of n_cw rate-5/6 codewords (coding.cpp:90-147):
 * llrs [n_cw][coded_len] in coded-bit order (positive favours 1), coded_len a
 * multiple of 6; info_out [n_cw][coded_len/6*5 - 6].  Host arrays. */
int cgm_viterbi_decode(cgm_ctx* ctx, const double* llrs, long coded_len, long n_cw,
                       uint8_t* info_out);

/* ---- multi-GPU: one process per GPU, subcarriers
 * sharded across ranks, the one collective is the gather of each rank's
 * outputs to a root.  NCCL is loaded at run time (dlopen "libnccl.so.2"; the
 * copy torch already loaded is reused); without it these return CGM_ENCCL.
 *
 *   rank 0: cgm_comm_unique_id(id); broadcast the 128 bytes to all ranks
 *           (MPI, torch.distributed, a file, ...)
 *   every rank: cgm_comm_create(ctx, nranks, rank, id, &comm)
 *   every rank: cgm_gather(ctx, comm, send, counts, recv, root)
 *
 * cgm_gather: rank r contributes counts[r] bytes from the device buffer
 * `send`; the root receives them concatenated in rank order into the device
 * buffer `recv` (sum of counts bytes; ignored on other ranks).  counts[] is
 * identical on every rank (ragged shards allowed).  Asynchronous on the
 * context's stream (ncclSend / ncclRecv in one group); replaces the
 * reference's host-side result collection (sim.cpp:286-305 joins worker
 * threads) for the multi-GPU batch.  Reference interface: none (the
 * reference is single-process); this is the §8(b) extra "cgm_gather". */
typedef struct cgm_comm cgm_comm;
int cgm_comm_unique_id(unsigned char id[128]);
int cgm_comm_create(cgm_ctx* ctx, int nranks, int rank, const unsigned char id[128],
                    cgm_comm** out);
int cgm_comm_destroy(cgm_comm* comm);
int cgm_gather(cgm_ctx* ctx, cgm_comm* comm, const void* send, const size_t* counts, void* recv,
               int root);
/* cgm_gatherv: like cgm_gather, but rank r's counts[r] bytes land at
 * recv + displs[r] on the root (displs identical on every rank).  The
 * chunked sharded pipeline uses it to drop chunk c of every rank's shard
 * straight into its place in the whole-job output while chunk c + 1 is
 * being computed (parallel.py ShardedPipeline). */
int cgm_gatherv(cgm_ctx* ctx, cgm_comm* comm, const void* send, const size_t* counts,
                const size_t* displs, void* recv, int root);

#ifdef __cplusplus
}
#endif
#endif /* CGMIMO_B200_H */
