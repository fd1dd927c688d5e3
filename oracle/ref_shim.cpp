// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE, never part of the product path.
//
// A flat extern "C" surface over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libcgmimo_ref.so).  It loops the reference's own per-call API
// over a batch so Python tests and bench.py's reference arm can drive it:
//
//   detect::detect_cg        (detect.hpp:58-61, detect.cpp:182-237)
//   detect::detect_explicit  (detect.hpp:44-49, detect.cpp:94-126)
//   detect::detect_cholesky / detect_cgls / detect_neumann (detect.cpp:122-326)
//   precode::precode_cgls / precode_neumann (precode.cpp:73-93)
//   precode::precode_cg      (precode.hpp:31-33, precode.cpp:56-71)
//   precode::precode_explicit(precode.hpp:26-27, precode.cpp:45-54)
//   detect::compute_llrs     (detect.cpp:68-86)
//   phy::make_constellation  (constellation.cpp:37-86)
//   phy::Rng                 (rng.cpp:12-52)
//   opcount::count_detect_stages (opcount.cpp:69-138)
//   phy::conv_encode / viterbi_decode_soft / make_interleaver (coding.cpp)
//   sim::run_uplink_sweep    (sim.cpp:365-384, trials of run_uplink_trial)
//
// Batch layout (shared with the CUDA path and oracle/cg_oracle.c):
//   H  uplink   [n_sc][B][U]  element (b,u) at b*U+u   (linalg.hpp:28)
//   Hd downlink [n_sc][U][B]  element (u,b) at u*B+b
//   Y  [n_sc][S][B]; T [n_sc][S][U]
//   outputs per instance (sc,s): xhat[U] mu[U] rho[U] llr[U][bits]; q[B] s[B] gain
// Complex values are interleaved (re,im) doubles.  Status per instance:
//   bit0 = SolverBreakdown (outputs zeroed), bit1 = zero_input (precode),
//   bit2 = std::invalid_argument / other exception.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "cgmimo/channel.hpp"
#include "cgmimo/coding.hpp"
#include "cgmimo/constellation.hpp"
#include "cgmimo/sim.hpp"
#include "cgmimo/detect.hpp"
#include "cgmimo/linalg.hpp"
#include "cgmimo/opcount.hpp"
#include "cgmimo/precode.hpp"
#include "cgmimo/rng.hpp"
#include "cgmimo/solvers.hpp"

using namespace cgmimo;

namespace {

phy::Modulation modulation_of(int bits) {
  switch (bits) {
    case 2: return phy::Modulation::kQpsk;
    case 4: return phy::Modulation::kQam16;
    case 6: return phy::Modulation::kQam64;
  }
  throw std::invalid_argument("qam_bits must be 2, 4 or 6");
}

template <class F>
void parallel_for(long n, int threads, F&& body) {
  if (threads <= 1 || n <= 1) {
    for (long i = 0; i < n; ++i) body(i);
    return;
  }
  std::atomic<long> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (long i = next.fetch_add(1); i < n; i = next.fetch_add(1)) body(i);
    });
  for (auto& th : pool) th.join();
}

ComplexMatrix load_matrix(const double* p, std::size_t rows, std::size_t cols) {
  ComplexMatrix m(rows, cols);
  for (std::size_t i = 0; i < rows; ++i)
    for (std::size_t j = 0; j < cols; ++j) {
      const double* e = p + 2 * (i * cols + j);
      m(i, j) = cplx(e[0], e[1]);
    }
  return m;
}

ComplexVector load_vector(const double* p, std::size_t n) {
  ComplexVector v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = cplx(p[2 * i], p[2 * i + 1]);
  return v;
}

void store_vector(const ComplexVector& v, double* p) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}

void store_soft(const detect::SoftOutput& o, std::size_t users, int bits, double* xhat,
                double* mu, double* rho, double* llr) {
  store_vector(o.xhat, xhat);
  for (std::size_t u = 0; u < users; ++u) {
    mu[u] = o.mu[u];
    rho[u] = o.rho[u];
    for (int b = 0; b < bits; ++b) llr[u * bits + b] = o.llrs[u][b];
  }
}

// mode 0 = detect_cg, 1 = detect_explicit, 2 = detect_cholesky, 3 = detect_cgls,
// 4 = detect_neumann
int detect_batch(int mode, int B, int U, long n_sc, int S, const double* H, const double* Y,
                 double rho_u, double n0, double es, int qam_bits, int K, int tracker,
                 double* xhat, double* mu, double* rho, double* llr, uint8_t* status,
                 int threads) {
  phy::Constellation c;
  try {
    c = phy::make_constellation(modulation_of(qam_bits));
  } catch (const std::exception&) {
    return 2;
  }
  const std::size_t users = U, bs = B;
  const auto trk = tracker == 0 ? detect::SinrTracker::kExact : detect::SinrTracker::kApprox;
  parallel_for(n_sc, threads, [&](long sc) {
    const ComplexMatrix h = load_matrix(H + 2 * sc * bs * users, bs, users);
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      const ComplexVector y = load_vector(Y + 2 * inst * bs, bs);
      double* xo = xhat + 2 * inst * users;
      double* mo = mu + inst * users;
      double* ro = rho + inst * users;
      double* lo = llr + inst * users * qam_bits;
      uint8_t st = 0;
      try {
        detect::SoftOutput o;
        if (mode == 0)
          o = detect::detect_cg(h, y, rho_u, n0, es, c, static_cast<std::size_t>(K), trk);
        else if (mode == 1)
          o = detect::detect_explicit(h, y, rho_u, n0, es, c);
        else if (mode == 2)
          o = detect::detect_cholesky(h, y, rho_u, n0, es, c);
        else if (mode == 3)
          o = detect::detect_cgls(h, y, rho_u, n0, es, c, static_cast<std::size_t>(K));
        else
          o = detect::detect_neumann(h, y, rho_u, n0, es, c, static_cast<std::size_t>(K));
        store_soft(o, users, qam_bits, xo, mo, ro, lo);
      } catch (const solvers::SolverBreakdown&) {
        st = 1;
      } catch (const std::exception&) {
        st = 4;
      }
      if (st) {
        std::memset(xo, 0, sizeof(double) * 2 * users);
        std::memset(mo, 0, sizeof(double) * users);
        std::memset(ro, 0, sizeof(double) * users);
        std::memset(lo, 0, sizeof(double) * users * qam_bits);
      }
      status[inst] = st;
    }
  });
  return 0;
}

int precode_batch(int mode, int B, int U, long n_sc, int S, const double* Hd, const double* T,
                  double rho_d, int K, double* q, double* s_out, double* gain, uint8_t* status,
                  int threads) {
  const std::size_t users = U, bs = B;
  parallel_for(n_sc, threads, [&](long sc) {
    const ComplexMatrix hd = load_matrix(Hd + 2 * sc * users * bs, users, bs);
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      const ComplexVector t = load_vector(T + 2 * inst * users, users);
      double* qo = q + 2 * inst * bs;
      double* so = s_out ? s_out + 2 * inst * bs : nullptr;
      uint8_t st = 0;
      try {
        const auto k = static_cast<std::size_t>(K);
        const precode::PrecodeResult r =
            mode == 0   ? precode::precode_cg(hd, t, rho_d, k)
            : mode == 1 ? precode::precode_explicit(hd, t, rho_d)
            : mode == 2 ? precode::precode_cgls(hd, t, rho_d, k)
                        : precode::precode_neumann(hd, t, rho_d, k);
        store_vector(r.precoded, qo);
        if (so) store_vector(r.transmit, so);
        gain[inst] = r.gain;
        if (r.zero_input) st |= 2;
      } catch (const solvers::SolverBreakdown&) {
        st = 1;
      } catch (const std::exception&) {
        st = 4;
      }
      if (st & 5) {
        std::memset(qo, 0, sizeof(double) * 2 * bs);
        if (so) std::memset(so, 0, sizeof(double) * 2 * bs);
        gain[inst] = 0.0;
      }
      status[inst] = st;
    }
  });
  return 0;
}

}  // namespace

extern "C" {

int ref_detect_cg(int B, int U, long n_sc, int S, const double* H, const double* Y,
                  double rho_u, double n0, double es, int qam_bits, int K, int tracker,
                  double* xhat, double* mu, double* rho, double* llr, uint8_t* status,
                  int threads) {
  return detect_batch(0, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, K, tracker, xhat, mu,
                      rho, llr, status, threads);
}

int ref_detect_explicit(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status, int threads) {
  return detect_batch(1, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, 1, 0, xhat, mu, rho,
                      llr, status, threads);
}

int ref_detect_cholesky(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status, int threads) {
  return detect_batch(2, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, 1, 0, xhat, mu, rho,
                      llr, status, threads);
}

int ref_detect_cgls(int B, int U, long n_sc, int S, const double* H, const double* Y,
                    double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                    double* mu, double* rho, double* llr, uint8_t* status, int threads) {
  return detect_batch(3, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, K, 1, xhat, mu, rho,
                      llr, status, threads);
}

int ref_detect_neumann(int B, int U, long n_sc, int S, const double* H, const double* Y,
                       double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                       double* mu, double* rho, double* llr, uint8_t* status, int threads) {
  return detect_batch(4, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, K, 1, xhat, mu, rho,
                      llr, status, threads);
}

int ref_precode_cgls(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                     double rho_d, int K, double* q, double* s, double* gain, uint8_t* status,
                     int threads) {
  return precode_batch(2, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status, threads);
}

int ref_precode_neumann(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                        double rho_d, int K, double* q, double* s, double* gain, uint8_t* status,
                        int threads) {
  return precode_batch(3, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status, threads);
}

int ref_precode_cg(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                   double rho_d, int K, double* q, double* s, double* gain, uint8_t* status,
                   int threads) {
  return precode_batch(0, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status, threads);
}

int ref_precode_explicit(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                         double rho_d, double* q, double* s, double* gain, uint8_t* status,
                         int threads) {
  return precode_batch(1, B, U, n_sc, S, Hd, T, rho_d, 1, q, s, gain, status, threads);
}

// Max-log LLRs of one user (detect.cpp:68-86); out has qam_bits entries.
int ref_compute_llrs(double xr, double xi, double mu, double rho, int qam_bits, double* out) {
  try {
    const auto c = phy::make_constellation(modulation_of(qam_bits));
    const auto l = detect::compute_llrs(cplx(xr, xi), mu, rho, c);
    for (int b = 0; b < qam_bits; ++b) out[b] = l[b];
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// Constellation tables (constellation.cpp:37-86): points[2^bits] complex,
// axis amplitudes axis0/axis1 [axis_bits][levels/2].
int ref_constellation(int qam_bits, double* points, double* axis0, double* axis1) {
  try {
    const auto c = phy::make_constellation(modulation_of(qam_bits));
    store_vector(c.points, points);
    const int half = c.axis_bits, per = (1 << half) / 2;
    for (int p = 0; p < half; ++p)
      for (int k = 0; k < per; ++k) {
        axis0[p * per + k] = c.axis_bit0[p][k];
        axis1[p * per + k] = c.axis_bit1[p][k];
      }
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// Rng stream: Rng(key).fork(f0).fork(f1)... then n draws of next_u64.
void ref_rng_u64(uint64_t key, const uint64_t* forks, int n_forks, long n, uint64_t* out) {
  phy::Rng r(key);
  for (int i = 0; i < n_forks; ++i) r = r.fork(forks[i]);
  for (long i = 0; i < n; ++i) out[i] = r.next_u64();
}

// n complex Gaussians of the given variance from the same stream construction.
void ref_rng_cgaussian(uint64_t key, const uint64_t* forks, int n_forks, double variance,
                       long n, double* out) {
  phy::Rng r(key);
  for (int i = 0; i < n_forks; ++i) r = r.fork(forks[i]);
  for (long i = 0; i < n; ++i) {
    const auto z = r.next_cgaussian(variance);
    out[2 * i] = z.real();
    out[2 * i + 1] = z.imag();
  }
}

// rayleigh_channel (channel.cpp:10-17) from Rng(key).fork(...).
void ref_rayleigh(uint64_t key, const uint64_t* forks, int n_forks, int B, int U, double* out) {
  phy::Rng r(key);
  for (int i = 0; i < n_forks; ++i) r = r.fork(forks[i]);
  const auto h = phy::rayleigh_channel(B, U, r);
  for (int b = 0; b < B; ++b)
    for (int u = 0; u < U; ++u) {
      out[2 * (b * U + u)] = h(b, u).real();
      out[2 * (b * U + u) + 1] = h(b, u).imag();
    }
}

// The device generator's uplink inputs (repo: csrc/cgm_generate.cu) drawn on
// the host with the reference's own Rng and constellation, so the CPU
// baseline times the SAME complex64 values the GPU arm detects:
//   H  [n_sc][B][U] c64 from Rng(seed).fork(2).fork(sc)  (channel.cpp:10-17 draw order)
//      correlated (rsqrt != null, B x B float): H_w [U][B] from that stream,
//      H[b][u] = sum_k conj(H_w[u][k]) rsqrt[k][b]  (FP64 sum, then c64)
//   labels of instance i = sc*S + s: Rng(seed).fork(1).fork(i), bits next_u64() & 1
//   Y  [n_sc][B][S] c64: (H x)_b in FP64 from the c64 H, plus
//      sqrt(N0/2) (next_gaussian, next_gaussian) of Rng(seed).fork(3).fork(i) (channel.cpp:21-30)
//   T  [n_sc][S][U] c64 (optional): transmit symbols, Rng(seed).fork(4).fork(i)
int ref_gen_uplink(uint64_t seed, int B, int U, long sc0, long n_sc, int S, int qam_bits,
                   double n0, const float* rsqrt, float* H, float* Y, float* T, int threads) {
  try {
    const auto c = phy::make_constellation(modulation_of(qam_bits));
    const phy::Rng root(seed);
    const phy::Rng chan = root.fork(2), lab = root.fork(1), noise = root.fork(3), sym = root.fork(4);
    const double sd = std::sqrt(0.5 * n0);
    auto label = [&](phy::Rng& r, int u) {
      (void)u;
      unsigned l = 0;
      for (int b = 0; b < qam_bits; ++b) l = (l << 1) | static_cast<unsigned>(r.next_u64() & 1u);
      return l;
    };
    parallel_for(n_sc, threads, [&](long i) {
      const long sc = sc0 + i;
      float* h = H + 2 * i * static_cast<long>(B) * U;
      phy::Rng r = chan.fork(static_cast<uint64_t>(sc));
      if (!rsqrt) {
        for (int e = 0; e < B * U; ++e) {
          const auto z = r.next_cgaussian(1.0);
          h[2 * e] = static_cast<float>(z.real());
          h[2 * e + 1] = static_cast<float>(z.imag());
        }
      } else {
        std::vector<float> hw(2 * static_cast<size_t>(U) * B);
        for (int e = 0; e < U * B; ++e) {
          const auto z = r.next_cgaussian(1.0);
          hw[2 * e] = static_cast<float>(z.real());
          hw[2 * e + 1] = static_cast<float>(z.imag());
        }
        for (int b = 0; b < B; ++b)
          for (int u = 0; u < U; ++u) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < B; ++k) {
              const double rr = rsqrt[static_cast<size_t>(k) * B + b];
              // fused like the device code's contracted DFMA chain
              re = std::fma(static_cast<double>(hw[2 * (u * B + k)]), rr, re);
              im = std::fma(-static_cast<double>(hw[2 * (u * B + k) + 1]), rr, im);
            }
            h[2 * (b * U + u)] = static_cast<float>(re);
            h[2 * (b * U + u) + 1] = static_cast<float>(im);
          }
      }
      std::vector<cplx> x(U);
      for (int s = 0; s < S; ++s) {
        const uint64_t inst = static_cast<uint64_t>(sc * S + s);
        phy::Rng lr = lab.fork(inst);
        for (int u = 0; u < U; ++u) x[u] = c.map_label(label(lr, u));
        phy::Rng nr = noise.fork(inst);
        for (int b = 0; b < B; ++b) {
          double re = 0.0, im = 0.0;
          for (int u = 0; u < U; ++u) {
            const double hx = h[2 * (b * U + u)], hy = h[2 * (b * U + u) + 1];
            re += hx * x[u].real() - hy * x[u].imag();
            im += hx * x[u].imag() + hy * x[u].real();
          }
          const double nre = nr.next_gaussian();
          const double nim = nr.next_gaussian();
          float* y = Y + 2 * ((i * B + b) * static_cast<long>(S) + s);
          y[0] = static_cast<float>(re + sd * nre);
          y[1] = static_cast<float>(im + sd * nim);
        }
        if (T) {
          phy::Rng tr = sym.fork(inst);
          float* t = T + 2 * (i * static_cast<long>(S) + s) * U;
          for (int u = 0; u < U; ++u) {
            const cplx v = c.map_label(label(tr, u));
            t[2 * u] = static_cast<float>(v.real());
            t[2 * u + 1] = static_cast<float>(v.imag());
          }
        }
      }
    });
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

double ref_uplink_noise_variance(double snr_db, int users) {
  return phy::uplink_noise_variance(snr_db, users);
}
double ref_downlink_noise_variance(double snr_db) {
  return phy::downlink_noise_variance(snr_db);
}

// Closed-form stage counts (opcount.cpp:69-138); method 0..3 = Cholesky, CG,
// CGLS, Neumann. out has opcount::kStageCount entries.
int ref_count_detect_stages(int method, int B, int U, int K, uint64_t* out) {
  const auto m = static_cast<opcount::DetectMethod>(method);
  const auto c = opcount::count_detect_stages(m, B, U, K);
  for (int s = 0; s < opcount::kStageCount; ++s) out[s] = c.by_stage[s];
  return opcount::kStageCount;
}

// Instrumented tally of one detect_cg call (approx tracker), per stage.
int ref_tally_detect_cg(int B, int U, int K, int tracker, uint64_t seed, uint64_t* out) {
  phy::Rng rng(seed);
  ComplexMatrix h(B, U);
  for (int b = 0; b < B; ++b)
    for (int u = 0; u < U; ++u) h(b, u) = rng.next_cgaussian(1.0);
  ComplexVector y(B);
  for (auto& v : y) v = rng.next_cgaussian(1.0);
  const auto c = phy::make_constellation(phy::Modulation::kQam16);
  opcount::Tally tally;
  {
    opcount::ScopedTally scope(tally);
    (void)detect::detect_cg(h, y, 10.0, 0.1, 1.0, c, K,
                            tracker == 0 ? detect::SinrTracker::kExact
                                         : detect::SinrTracker::kApprox);
  }
  for (int s = 0; s < opcount::kStageCount; ++s)
    out[s] = tally.get(static_cast<opcount::Stage>(s));
  return opcount::kStageCount;
}

// Exact-tracker filters L_1..L_K of one (H, y) pair (detect.cpp:336-368),
// driven by cg_solve exactly as detect_cg drives it; filters [K][U][U] c128,
// iterates [K][U] c128. Used to pin the kernel's polynomial-basis tracker.
int ref_exact_filters(int B, int U, const double* H, const double* Y, double rho_u, int K,
                      double* filters, double* iterates) {
  try {
    const ComplexMatrix h = load_matrix(H, B, U);
    const ComplexVector y = load_vector(Y, B);
    const auto a = gram_regularized(h, 1.0 / rho_u, GramSide::kUplink);
    const auto a_full = a.full();
    const auto b = matvec_adjoint(h, y);
    detect::ExactSinrTracker tr(U);
    solvers::IterOptions opts;
    opts.keep_trace = true;
    int k = 0;
    opts.on_iteration = [&](std::size_t, double alpha, double beta) {
      tr.step(a_full, alpha, beta);
      const auto& f = tr.filter();
      for (int i = 0; i < U; ++i)
        for (int j = 0; j < U; ++j) {
          filters[2 * ((k * U + i) * U + j)] = f(i, j).real();
          filters[2 * ((k * U + i) * U + j) + 1] = f(i, j).imag();
        }
      ++k;
    };
    const auto res = solvers::cg_solve(a, b, K, opts);
    for (int kk = 0; kk < K; ++kk) store_vector(res.trace[kk], iterates + 2 * kk * U);
    return 0;
  } catch (const solvers::SolverBreakdown&) {
    return 1;
  } catch (const std::exception&) {
    return 2;
  }
}

// ---- coded BLER harness (sim.cpp / coding.cpp)
long ref_conv_encode(const uint8_t* info, long n, uint8_t* out) {
  try {
    const auto coded = phy::conv_encode(std::vector<uint8_t>(info, info + n));
    std::memcpy(out, coded.data(), coded.size());
    return static_cast<long>(coded.size());
  } catch (const std::exception&) {
    return -1;
  }
}

long ref_viterbi_decode(const double* llrs, long n, uint8_t* out) {
  try {
    const auto info = phy::viterbi_decode_soft(std::vector<double>(llrs, llrs + n));
    std::memcpy(out, info.data(), info.size());
    return static_cast<long>(info.size());
  } catch (const std::exception&) {
    return -1;
  }
}

void ref_make_interleaver(uint64_t key, const uint64_t* forks, int n_forks, long n, int64_t* perm) {
  phy::Rng rng(key);
  for (int i = 0; i < n_forks; ++i) rng = rng.fork(forks[i]);
  const auto p = phy::make_interleaver(static_cast<std::size_t>(n), rng);
  for (long i = 0; i < n; ++i) perm[i] = static_cast<int64_t>(p[i]);
}

// One SNR point of the reference's uplink or downlink BLER sweep (CG solver):
// out = {frames, block_errors, breakdowns, trials_run}; returns 0, or -1 on
// an exception (e.g. BreakdownBudgetExceeded is disabled by fraction 1.0).
static int sweep_point(bool downlink, int B, int U, int qam_bits, int K, int tracker,
                       double snr_db, long trials, long n_sc, uint64_t seed, int threads,
                       long* out) {
  try {
    sim::SweepConfig cfg;
    cfg.bs_antennas = static_cast<std::size_t>(B);
    cfg.users = static_cast<std::size_t>(U);
    cfg.modulation = qam_bits == 2 ? phy::Modulation::kQpsk
                                   : (qam_bits == 4 ? phy::Modulation::kQam16 : phy::Modulation::kQam64);
    cfg.method = sim::Method::kCg;
    cfg.iterations = static_cast<std::size_t>(K);
    cfg.tracker = tracker == 0 ? detect::SinrTracker::kExact : detect::SinrTracker::kApprox;
    cfg.snr_start_db = cfg.snr_stop_db = snr_db;
    cfg.snr_step_db = 1.0;
    cfg.trials = static_cast<std::size_t>(trials);
    cfg.subcarriers = static_cast<std::size_t>(n_sc);
    cfg.seed = seed;
    cfg.threads = static_cast<std::size_t>(threads);
    cfg.max_breakdown_fraction = 1.0;
    const auto r = downlink ? sim::run_downlink_sweep(cfg) : sim::run_uplink_sweep(cfg);
    const auto& pt = r.points.at(0);
    out[0] = static_cast<long>(pt.frames);
    out[1] = static_cast<long>(pt.block_errors);
    out[2] = static_cast<long>(pt.breakdowns);
    out[3] = static_cast<long>(pt.trials_run);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_uplink_sweep_point(int B, int U, int qam_bits, int K, int tracker, double snr_db,
                           long trials, long n_sc, uint64_t seed, int threads, long* out) {
  return sweep_point(false, B, U, qam_bits, K, tracker, snr_db, trials, n_sc, seed, threads, out);
}

// run_downlink_sweep (sim.cpp:386-405) at one SNR, CG precoder; same outputs
int ref_downlink_sweep_point(int B, int U, int qam_bits, int K, double snr_db, long trials,
                             long n_sc, uint64_t seed, int threads, long* out) {
  return sweep_point(true, B, U, qam_bits, K, 1, snr_db, trials, n_sc, seed, threads, out);
}

// A whole sweep (sim::run_uplink_sweep / run_downlink_sweep, sim.cpp:365-405)
// with any method and SNR grid.  out[p * 9 + ...] = {snr_db, frames,
// block_errors, bler, bler_lo, bler_hi, real_mults_mean, breakdowns,
// trials_run}; returns the number of points (<= max_points), -1 on
// ConfigError, -2 on BreakdownBudgetExceeded, -3 on any other exception.
long ref_sweep(int direction, int method, int B, int U, int qam_bits, int iters, int tracker,
               double snr_start, double snr_stop, double snr_step, long trials, long n_sc,
               uint64_t seed, long max_block_errors, double max_breakdown_fraction, int threads,
               double* out, long max_points) {
  try {
    sim::SweepConfig cfg;
    cfg.bs_antennas = static_cast<std::size_t>(B);
    cfg.users = static_cast<std::size_t>(U);
    cfg.modulation = modulation_of(qam_bits);
    cfg.method = static_cast<sim::Method>(method);
    cfg.iterations = static_cast<std::size_t>(iters);
    cfg.tracker = tracker == 0 ? detect::SinrTracker::kExact : detect::SinrTracker::kApprox;
    cfg.snr_start_db = snr_start;
    cfg.snr_stop_db = snr_stop;
    cfg.snr_step_db = snr_step;
    cfg.trials = static_cast<std::size_t>(trials);
    cfg.subcarriers = static_cast<std::size_t>(n_sc);
    cfg.seed = seed;
    cfg.threads = static_cast<std::size_t>(threads);
    cfg.max_block_errors = static_cast<std::size_t>(max_block_errors);
    cfg.max_breakdown_fraction = max_breakdown_fraction;
    const auto r = direction == 2 ? sim::run_downlink_sweep(cfg) : sim::run_uplink_sweep(cfg);
    long n = 0;
    for (const auto& p : r.points) {
      if (n >= max_points) break;
      double* o = out + 9 * n++;
      o[0] = p.snr_db; o[1] = static_cast<double>(p.frames);
      o[2] = static_cast<double>(p.block_errors); o[3] = p.bler; o[4] = p.bler_lo;
      o[5] = p.bler_hi; o[6] = p.real_mults_mean; o[7] = static_cast<double>(p.breakdowns);
      o[8] = static_cast<double>(p.trials_run);
    }
    return n;
  } catch (const sim::ConfigError&) {
    return -1;
  } catch (const sim::BreakdownBudgetExceeded&) {
    return -2;
  } catch (const std::exception&) {
    return -3;
  }
}

// sim::tradeoff_table (sim.cpp:475-497) for ONE sweep given by its points
// (snr, frames, block_errors per point; bler recomputed as the reference
// does): writes real_mults and snr_db_at_target; returns 1 when the target
// is bracketed, 0 when not (nullopt).
int ref_tradeoff_row(int method, int B, int U, int iters, const double* snr,
                     const uint64_t* frames, const uint64_t* errors, long n, double target,
                     uint64_t* real_mults, double* snr_at_target) {
  sim::SweepResult sw;
  sw.config.bs_antennas = static_cast<std::size_t>(B);
  sw.config.users = static_cast<std::size_t>(U);
  sw.config.method = static_cast<sim::Method>(method);
  sw.config.iterations = static_cast<std::size_t>(iters);
  for (long i = 0; i < n; ++i) {
    sim::SnrPointResult p;
    p.snr_db = snr[i];
    p.frames = frames[i];
    p.block_errors = errors[i];
    p.bler = p.frames > 0 ? static_cast<double>(p.block_errors) / static_cast<double>(p.frames) : 0.0;
    sw.points.push_back(p);
  }
  const auto rows = sim::tradeoff_table({sw}, target);
  *real_mults = rows.at(0).real_mults;
  if (!rows[0].snr_db_at_target) return 0;
  *snr_at_target = *rows[0].snr_db_at_target;
  return 1;
}

// sim::wilson_interval (sim.cpp:78-92)
void ref_wilson(uint64_t errors, uint64_t total, double* lo, double* hi) {
  const auto w = sim::wilson_interval(errors, total);
  *lo = w.first;
  *hi = w.second;
}

}  // extern "C"
