// cgmimo/detect.hpp -- drop-in for the reference uplink detectors
// (reference proj/include/cgmimo/detect.hpp:21-73).  detect_cg keeps the
// reference signature and runs on the B200 through the C ABI
// (include/cgmimo_b200.h); detect_cg_batch is the batched form the GPU wants.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "cgmimo/constellation.hpp"
#include "cgmimo/linalg.hpp"

namespace cgmimo::detect {

inline constexpr double kLlrMax = 64.0;
inline constexpr double kGainFloor = 1e-12;

struct SoftOutput {
  ComplexVector xhat;                     // v_K, not divided by mu
  std::vector<double> mu;
  std::vector<double> rho;
  std::vector<std::vector<double>> llrs;  // [user][bit], +-kLlrMax
};

enum class SinrTracker { kExact, kApprox };

// Host max-log demapper of one user (same rule as the kernel epilogue).
std::vector<double> compute_llrs(cplx xhat, double mu, double rho, const phy::Constellation& c);

// Throws std::invalid_argument on bad arguments and solvers::SolverBreakdown
// on non-positive curvature, like the reference.
SoftOutput detect_cg(const ComplexMatrix& h, const ComplexVector& y, double rho_u, double n0,
                     double es, const phy::Constellation& c, std::size_t iters,
                     SinrTracker tracker);

// The trade-off study's other detectors (reference detect.hpp:47-73), same
// signatures and exceptions (NotPositiveDefinite from Cholesky,
// std::domain_error from a zero Neumann diagonal).
SoftOutput detect_cholesky(const ComplexMatrix& h, const ComplexVector& y, double rho_u,
                           double n0, double es, const phy::Constellation& c);
SoftOutput detect_cgls(const ComplexMatrix& h, const ComplexVector& y, double rho_u, double n0,
                       double es, const phy::Constellation& c, std::size_t iters);
SoftOutput detect_neumann(const ComplexMatrix& h, const ComplexVector& y, double rho_u,
                          double n0, double es, const phy::Constellation& c, std::size_t terms);

// Batched form: hs[i] / ys[i] pairs (every hs[i] of equal shape).  Instances
// that break down get status 1 and zeroed outputs instead of throwing.
std::vector<SoftOutput> detect_cg_batch(const std::vector<ComplexMatrix>& hs,
                                        const std::vector<ComplexVector>& ys, double rho_u,
                                        double n0, double es, const phy::Constellation& c,
                                        std::size_t iters, SinrTracker tracker,
                                        std::vector<std::uint8_t>* status = nullptr);

}  // namespace cgmimo::detect
