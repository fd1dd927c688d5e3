// cgm_dropin.cpp -- the reference's C++ entry points (include/cgmimo/*.hpp)
// implemented on the C ABI (include/cgmimo_b200.h).  A caller written
// against the reference headers relinks against libcgmimo_b200.so unchanged:
//   cgmimo::detect::detect_cg    (reference detect.hpp:58-61)
//   cgmimo::detect::detect_cholesky / detect_cgls / detect_neumann (:54-73)
//   cgmimo::precode::precode_cg  (reference precode.hpp:31-33)
//   cgmimo::precode::precode_explicit / precode_cgls / precode_neumann (:25-45)
// FP64 arguments are converted to complex64 at the boundary and results
// widened back; errors map to the reference's exception types.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cgmimo/constellation.hpp"
#include "../../include/cgmimo/detect.hpp"
#include "../../include/cgmimo/linalg.hpp"
#include "../../include/cgmimo/opcount.hpp"
#include "../../include/cgmimo/precode.hpp"
#include "../../include/cgmimo/solvers.hpp"
#include "../../include/cgmimo_b200.h"

namespace cgmimo {

namespace {

// One C-ABI context per host thread: calls stay reentrant like the
// reference's pure functions (reference linalg.hpp:4-5, sim.cpp:286-305).
struct ThreadCtx {
  cgm_ctx* ctx = nullptr;
  ~ThreadCtx() {
    if (ctx) cgm_ctx_destroy(ctx);
  }
  cgm_ctx* get() {
    if (!ctx) {
      const char* dev = std::getenv("CGMIMO_DEVICE");
      const int rc = cgm_ctx_create(dev ? std::atoi(dev) : 0, &ctx);
      if (rc != CGM_OK) {
        ctx = nullptr;
        throw std::runtime_error("cgmimo_b200: no usable sm_100 device (cgm_ctx_create rc=" +
                                 std::to_string(rc) + ")");
      }
    }
    return ctx;
  }
};
thread_local ThreadCtx t_ctx;

void check(int rc, cgm_ctx* ctx) {
  if (rc == CGM_OK) return;
  const std::string msg = cgm_last_error(ctx);
  if (rc == CGM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("cgmimo_b200: " + msg);
}

void to_c64(const cplx* src, std::size_t n, float* dst) {
  for (std::size_t i = 0; i < n; ++i) {
    dst[2 * i] = static_cast<float>(src[i].real());
    dst[2 * i + 1] = static_cast<float>(src[i].imag());
  }
}

unsigned gray_decode(unsigned g) {
  unsigned m = g;
  for (unsigned s = g >> 1; s != 0; s >>= 1) m ^= s;
  return m;
}

}  // namespace

// ---------------------------------------------------------------- opcount
namespace opcount {
namespace {
thread_local Tally* g_tally = nullptr;
}
ScopedTally::ScopedTally(Tally& t) : prev_(g_tally) { g_tally = &t; }
ScopedTally::~ScopedTally() { g_tally = prev_; }
void record(Stage stage, std::uint64_t n) {
  if (g_tally) g_tally->add(stage, n);
}
bool counting_active() { return g_tally != nullptr; }
}  // namespace opcount

// ---------------------------------------------------------- constellation
namespace phy {

Modulation parse_modulation(const std::string& name) {
  if (name == "qpsk") return Modulation::kQpsk;
  if (name == "16qam") return Modulation::kQam16;
  if (name == "64qam") return Modulation::kQam64;
  throw std::invalid_argument("unknown modulation: " + name);
}

std::string modulation_name(Modulation m) {
  return m == Modulation::kQpsk ? "qpsk" : m == Modulation::kQam16 ? "16qam" : "64qam";
}

Constellation make_constellation(Modulation kind) {
  const int bits = kind == Modulation::kQpsk ? 2 : kind == Modulation::kQam16 ? 4 : 6;
  const int half = bits / 2;
  const unsigned levels = 1u << half, count = 1u << bits;
  const double scale = 1.0 / std::sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
  Constellation c;
  c.kind = kind;
  c.bits_per_symbol = bits;
  c.axis_bits = half;
  c.points.resize(count);
  c.bit0_labels.assign(bits, {});
  c.bit1_labels.assign(bits, {});
  double energy = 0.0;
  for (unsigned label = 0; label < count; ++label) {
    const double ai = 2.0 * gray_decode(label >> half) - (levels - 1.0);
    const double aq = 2.0 * gray_decode(label & (levels - 1)) - (levels - 1.0);
    c.points[label] = cplx(ai * scale, aq * scale);
    energy += std::norm(c.points[label]);
    for (int b = 0; b < bits; ++b)
      ((label >> (bits - 1 - b)) & 1u ? c.bit1_labels : c.bit0_labels)[b].push_back(
          static_cast<int>(label));
  }
  c.symbol_energy = energy / count;
  c.axis_bit0.assign(half, {});
  c.axis_bit1.assign(half, {});
  for (unsigned g = 0; g < levels; ++g) {
    const double amp = (2.0 * gray_decode(g) - (levels - 1.0)) * scale;
    for (int p = 0; p < half; ++p)
      ((g >> (half - 1 - p)) & 1u ? c.axis_bit1 : c.axis_bit0)[p].push_back(amp);
  }
  return c;
}

std::vector<cplx> map_bits(const std::vector<std::uint8_t>& bits, const Constellation& c) {
  const std::size_t bps = c.bits_per_symbol;
  if (bits.size() % bps != 0)
    throw std::invalid_argument("map_bits: bit count not divisible by bits per symbol");
  std::vector<cplx> out(bits.size() / bps);
  for (std::size_t s = 0; s < out.size(); ++s) {
    unsigned label = 0;
    for (std::size_t b = 0; b < bps; ++b) label = (label << 1) | (bits[s * bps + b] & 1u);
    out[s] = c.points[label];
  }
  return out;
}

unsigned hard_demap(cplx received, const Constellation& c) {
  unsigned best = 0;
  double bd = std::numeric_limits<double>::infinity();
  for (unsigned l = 0; l < c.points.size(); ++l) {
    const double d = std::norm(received - c.points[l]);
    if (d < bd) {
      bd = d;
      best = l;
    }
  }
  return best;
}

}  // namespace phy

// ----------------------------------------------------------------- detect
namespace detect {

std::vector<double> compute_llrs(cplx xhat, double mu, double rho, const phy::Constellation& c) {
  std::vector<double> out(c.bits_per_symbol, 0.0);
  if (std::abs(mu) < kGainFloor) return out;
  if (rho < 0.0) rho = 0.0;
  const cplx z = xhat / mu;
  auto amin = [](double v, const std::vector<double>& a) {
    double best = std::numeric_limits<double>::infinity();
    for (double x : a) best = std::min(best, (v - x) * (v - x));
    return best;
  };
  for (int p = 0; p < c.axis_bits; ++p) {
    out[p] = std::clamp(rho * (amin(z.real(), c.axis_bit0[p]) - amin(z.real(), c.axis_bit1[p])),
                        -kLlrMax, kLlrMax);
    out[c.axis_bits + p] =
        std::clamp(rho * (amin(z.imag(), c.axis_bit0[p]) - amin(z.imag(), c.axis_bit1[p])),
                   -kLlrMax, kLlrMax);
  }
  return out;
}

namespace {

// Stage tallies the reference's instrumented path records for one call
// (linalg.cpp record() sites; opcount.cpp:94-106 for the approx closed form;
// detect.cpp:359, :379-394 for the exact tracker).  Non-frozen CG iterations
// are taken as min(K, U) unless the matched filter is zero (frozen from k=1).
void record_counts(std::size_t B, std::size_t U, std::size_t K, SinrTracker tr, bool zero_rhs) {
  using opcount::Stage;
  if (!opcount::counting_active()) return;
  const std::uint64_t b = B, u = U, k = K;
  const std::uint64_t live = zero_rhs ? 0 : std::min(k, u);
  opcount::record(Stage::kGram, 2 * b * u * u);
  opcount::record(Stage::kMatchedFilter, 4 * b * u);
  opcount::record(Stage::kCgIteration, 2 * u + live * (4 * u * u + 12 * u));
  if (tr == SinrTracker::kApprox)
    opcount::record(Stage::kTracker, k * u);
  else
    opcount::record(Stage::kTracker,
                    (k - 1) * (4 * u * u * u + 6 * u * u + 2) + 4 * u * u * u + 6 * u * u);
}

int bits_of(const phy::Constellation& c) { return c.bits_per_symbol; }

}  // namespace

std::vector<SoftOutput> detect_cg_batch(const std::vector<ComplexMatrix>& hs,
                                        const std::vector<ComplexVector>& ys, double rho_u,
                                        double n0, double es, const phy::Constellation& c,
                                        std::size_t iters, SinrTracker tracker,
                                        std::vector<std::uint8_t>* status) {
  if (hs.size() != ys.size()) throw std::invalid_argument("detect_cg: batch size mismatch");
  const long n = static_cast<long>(hs.size());
  if (n == 0) return {};
  const std::size_t B = hs[0].rows(), U = hs[0].cols();
  for (long i = 0; i < n; ++i)
    if (hs[i].rows() != B || hs[i].cols() != U || ys[i].size() != B)
      throw std::invalid_argument("detect_cg: dimension mismatch");
  const int bits = bits_of(c);
  std::vector<float> H(2 * B * U * n), Y(2 * B * n), X(2 * U * n), MU(U * n), RHO(U * n),
      L(U * bits * n);
  std::vector<std::uint8_t> st(n);
  for (long i = 0; i < n; ++i) {
    to_c64(hs[i].data(), B * U, H.data() + 2 * B * U * i);
    to_c64(ys[i].data(), B, Y.data() + 2 * B * i);
  }
  cgm_ctx* ctx = t_ctx.get();
  check(cgm_detect_cg(ctx, static_cast<int>(B), static_cast<int>(U), n, 1, H.data(), Y.data(),
                      rho_u, n0, es, bits, static_cast<int>(iters),
                      tracker == SinrTracker::kExact ? CGM_TRACKER_EXACT : CGM_TRACKER_APPROX,
                      X.data(), MU.data(), RHO.data(), L.data(), st.data(), 0),
        ctx);
  std::vector<SoftOutput> out(n);
  for (long i = 0; i < n; ++i) {
    SoftOutput& o = out[i];
    o.xhat.resize(U);
    o.mu.resize(U);
    o.rho.resize(U);
    o.llrs.assign(U, std::vector<double>(bits));
    for (std::size_t u = 0; u < U; ++u) {
      const std::size_t e = i * U + u;
      o.xhat[u] = cplx(X[2 * e], X[2 * e + 1]);
      o.mu[u] = MU[e];
      o.rho[u] = RHO[e];
      for (int b = 0; b < bits; ++b) o.llrs[u][b] = L[e * bits + b];
    }
  }
  if (status) *status = st;
  return out;
}

SoftOutput detect_cg(const ComplexMatrix& h, const ComplexVector& y, double rho_u, double n0,
                     double es, const phy::Constellation& c, std::size_t iters,
                     SinrTracker tracker) {
  // detect.cpp:186-188
  if (h.rows() != y.size()) throw std::invalid_argument("detect_cg: dimension mismatch");
  if (!(rho_u > 0.0 && n0 > 0.0 && es > 0.0))
    throw std::invalid_argument("detect_cg: bad parameters");
  if (iters < 1) throw std::invalid_argument("detect_cg: need at least one iteration");
  std::vector<std::uint8_t> st;
  auto out = detect_cg_batch({h}, {y}, rho_u, n0, es, c, iters, tracker, &st);
  if (st[0] & 1u) throw solvers::SolverBreakdown("cg_solve: non-positive curvature p^H A p");
  bool zero = true;
  for (const auto& v : y) zero = zero && v == cplx(0.0, 0.0);
  record_counts(h.rows(), h.cols(), iters, tracker, zero);
  return std::move(out[0]);
}

namespace {

// closed-form stage counts of the other detectors (opcount.cpp:69-138) as the
// reference's instrumented path records them; CGLS iterations past exact
// convergence (min(K, U)) are frozen and uncounted, like CG's
void record_alt_counts(int method, std::size_t B, std::size_t U, std::size_t K, bool zero_rhs) {
  using opcount::Stage;
  if (!opcount::counting_active()) return;
  const std::uint64_t b = B, u = U, k = K;
  if (method == CGM_METHOD_CHOLESKY) {
    opcount::record(Stage::kGram, 2 * b * u * u);
    opcount::record(Stage::kMatchedFilter, 4 * b * u);
    opcount::record(Stage::kCholesky, u * (u - 1) + 2 * u * (u - 1) * (u - 2) / 3);
    opcount::record(Stage::kSubstitution,
                    2 * (u * u * u - u) / 3 + 2 * u * u * (u - 1) + 4 * u * u + 6 * u * u + 2 * u);
  } else if (method == CGM_METHOD_CGLS) {
    const std::uint64_t live = zero_rhs ? 0 : std::min(k, u);
    opcount::record(Stage::kGram, 2 * b * u);
    opcount::record(Stage::kMatchedFilter, 4 * b * u);
    opcount::record(Stage::kCglsIteration, 2 * u + live * (8 * b * u + 4 * b + 14 * u));
    opcount::record(Stage::kTracker, k * u);
  } else {
    opcount::record(Stage::kGram, 2 * b * u * u);
    opcount::record(Stage::kMatchedFilter, 4 * b * u);
    std::uint64_t series = 0;
    if (k >= 2) series += 4 * u * (u - 1);
    if (k >= 3) series += (k - 2) * 2 * u * u * (u + 1);
    opcount::record(Stage::kNeumannTerm, series);
    opcount::record(Stage::kSubstitution, ((k == 1) ? 2 * u : 4 * u * u) +
                                              ((k == 1) ? u : 4 * u * u) + 2 * u);
  }
}

void throw_status(std::uint8_t st, int method, const char* who) {
  if (st & 1u) throw solvers::SolverBreakdown(std::string(who) + ": breakdown");
  if (st & 4u) {
    if (method == CGM_METHOD_CHOLESKY)
      throw solvers::NotPositiveDefinite("cholesky_factor: non-positive pivot");
    throw std::domain_error("neumann_inverse: zero diagonal entry");
  }
}

SoftOutput detect_alt(int method, const char* who, const ComplexMatrix& h, const ComplexVector& y,
                      double rho_u, double n0, double es, const phy::Constellation& c,
                      std::size_t iters) {
  // detect.cpp:127-129, :243-245, :279-281
  if (h.rows() != y.size()) throw std::invalid_argument(std::string(who) + ": dimension mismatch");
  if (!(rho_u > 0.0 && n0 > 0.0 && es > 0.0))
    throw std::invalid_argument(std::string(who) + ": bad parameters");
  if (iters < 1) throw std::invalid_argument(std::string(who) + ": need at least one iteration");
  const std::size_t B = h.rows(), U = h.cols();
  const int bits = bits_of(c);
  std::vector<float> H(2 * B * U), Y(2 * B), X(2 * U), MU(U), RHO(U), L(U * bits);
  std::uint8_t st = 0;
  to_c64(h.data(), B * U, H.data());
  to_c64(y.data(), B, Y.data());
  cgm_ctx* ctx = t_ctx.get();
  check(cgm_detect(ctx, method, static_cast<int>(B), static_cast<int>(U), 1, 1, H.data(), Y.data(),
                   rho_u, n0, es, bits, static_cast<int>(iters), CGM_TRACKER_APPROX, X.data(),
                   MU.data(), RHO.data(), L.data(), &st, 0),
        ctx);
  throw_status(st, method, who);
  bool zero = true;
  for (const auto& v : y) zero = zero && v == cplx(0.0, 0.0);
  record_alt_counts(method, B, U, iters, zero);
  SoftOutput o;
  o.xhat.resize(U);
  o.mu.resize(U);
  o.rho.resize(U);
  o.llrs.assign(U, std::vector<double>(bits));
  for (std::size_t u = 0; u < U; ++u) {
    o.xhat[u] = cplx(X[2 * u], X[2 * u + 1]);
    o.mu[u] = MU[u];
    o.rho[u] = RHO[u];
    for (int b = 0; b < bits; ++b) o.llrs[u][b] = L[u * bits + b];
  }
  return o;
}

}  // namespace

SoftOutput detect_cholesky(const ComplexMatrix& h, const ComplexVector& y, double rho_u,
                           double n0, double es, const phy::Constellation& c) {
  return detect_alt(CGM_METHOD_CHOLESKY, "detect_cholesky", h, y, rho_u, n0, es, c, 1);
}

SoftOutput detect_cgls(const ComplexMatrix& h, const ComplexVector& y, double rho_u, double n0,
                       double es, const phy::Constellation& c, std::size_t iters) {
  return detect_alt(CGM_METHOD_CGLS, "detect_cgls", h, y, rho_u, n0, es, c, iters);
}

SoftOutput detect_neumann(const ComplexMatrix& h, const ComplexVector& y, double rho_u,
                          double n0, double es, const phy::Constellation& c, std::size_t terms) {
  return detect_alt(CGM_METHOD_NEUMANN, "detect_neumann", h, y, rho_u, n0, es, c, terms);
}

}  // namespace detect

// ---------------------------------------------------------------- precode
namespace precode {

namespace {

ComplexVector precode_one(int method, const ComplexMatrix& h_downlink, const ComplexVector& t,
                          double rho_d, std::size_t iters, PrecodeResult* res, const char* who) {
  const std::size_t U = h_downlink.rows(), B = h_downlink.cols();
  std::vector<float> Hd(2 * U * B), T(2 * U), Q(2 * B), S(2 * B);
  to_c64(h_downlink.data(), U * B, Hd.data());
  to_c64(t.data(), U, T.data());
  cgm_ctx* ctx = t_ctx.get();
  float gain = 0.f;
  std::uint8_t st = 0;
  check(cgm_precode(ctx, method, static_cast<int>(B), static_cast<int>(U), 1, 1, Hd.data(),
                    T.data(), rho_d, static_cast<int>(iters), Q.data(), S.data(), &gain, &st, 0),
        ctx);
  detect::throw_status(st, method, who);
  ComplexVector q(B);
  for (std::size_t b = 0; b < B; ++b) q[b] = cplx(Q[2 * b], Q[2 * b + 1]);
  if (res) {
    res->zero_input = (st & 2u) != 0;
    res->gain = res->zero_input ? 0.0 : gain;
    res->transmit.resize(B);
    for (std::size_t b = 0; b < B; ++b) res->transmit[b] = cplx(S[2 * b], S[2 * b + 1]);
    res->precoded = q;
  }
  return q;
}

void precode_checks(const ComplexMatrix& h_downlink, const ComplexVector& t, double rho_d,
                    std::size_t iters, const char* who) {
  // precode.cpp:47-48, :76-77, :86-87; solvers.cpp:200-201
  if (!(rho_d > 0.0)) throw std::invalid_argument(std::string(who) + ": rho_d must be positive");
  if (h_downlink.rows() != t.size()) throw std::invalid_argument(std::string(who) + ": dimension mismatch");
  if (iters < 1) throw std::invalid_argument(std::string(who) + ": need at least one iteration");
}

}  // namespace

PrecodeResult precode_explicit(const ComplexMatrix& h_downlink, const ComplexVector& t,
                               double rho_d) {
  precode_checks(h_downlink, t, rho_d, 1, "precode_explicit");
  PrecodeResult res;
  precode_one(CGM_METHOD_CHOLESKY, h_downlink, t, rho_d, 1, &res, "precode_explicit");
  return res;
}

PrecodeResult precode_cgls(const ComplexMatrix& h_downlink, const ComplexVector& t, double rho_d,
                           std::size_t iters, std::vector<ComplexVector>* q_trace) {
  precode_checks(h_downlink, t, rho_d, iters, "precode_cgls");
  if (q_trace) {
    q_trace->clear();
    for (std::size_t k = 1; k <= iters; ++k)
      q_trace->push_back(precode_one(CGM_METHOD_CGLS, h_downlink, t, rho_d, k, nullptr, "cgls"));
  }
  PrecodeResult res;
  precode_one(CGM_METHOD_CGLS, h_downlink, t, rho_d, iters, &res, "cgls_solve_min_norm");
  return res;
}

PrecodeResult precode_neumann(const ComplexMatrix& h_downlink, const ComplexVector& t,
                              double rho_d, std::size_t terms) {
  precode_checks(h_downlink, t, rho_d, terms, "precode_neumann");
  PrecodeResult res;
  precode_one(CGM_METHOD_NEUMANN, h_downlink, t, rho_d, terms, &res, "precode_neumann");
  return res;
}

PrecodeResult precode_cg(const ComplexMatrix& h_downlink, const ComplexVector& t, double rho_d,
                         std::size_t iters, std::vector<ComplexVector>* q_trace) {
  // precode.cpp:59-60
  if (!(rho_d > 0.0)) throw std::invalid_argument("precode_cg: rho_d must be positive");
  if (h_downlink.rows() != t.size()) throw std::invalid_argument("precode_cg: dimension mismatch");
  if (iters < 1) throw std::invalid_argument("cg_solve: need at least one iteration");
  const std::size_t U = h_downlink.rows(), B = h_downlink.cols();
  std::vector<float> Hd(2 * U * B), T(2 * U), Q(2 * B), S(2 * B);
  to_c64(h_downlink.data(), U * B, Hd.data());
  to_c64(t.data(), U, T.data());
  cgm_ctx* ctx = t_ctx.get();
  auto run = [&](std::size_t k, PrecodeResult* res) {
    float gain = 0.f;
    std::uint8_t st = 0;
    check(cgm_precode_cg(ctx, static_cast<int>(B), static_cast<int>(U), 1, 1, Hd.data(), T.data(),
                         rho_d, static_cast<int>(k), Q.data(), S.data(), &gain, &st, 0),
          ctx);
    if (st & 1u) throw solvers::SolverBreakdown("cg_solve: non-positive curvature p^H A p");
    ComplexVector q(B);
    for (std::size_t b = 0; b < B; ++b) q[b] = cplx(Q[2 * b], Q[2 * b + 1]);
    if (res) {
      res->zero_input = (st & 2u) != 0;
      res->gain = res->zero_input ? 0.0 : gain;
      res->transmit.resize(B);
      for (std::size_t b = 0; b < B; ++b) res->transmit[b] = cplx(S[2 * b], S[2 * b + 1]);
      res->precoded = q;
    }
    return q;
  };
  if (q_trace) {
    // iterate k of a K-iteration run is the result of a k-iteration run
    q_trace->clear();
    for (std::size_t k = 1; k <= iters; ++k) q_trace->push_back(run(k, nullptr));
  }
  PrecodeResult res;
  run(iters, &res);
  return res;
}

}  // namespace precode

}  // namespace cgmimo
