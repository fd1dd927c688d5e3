// cgmimo/precode.hpp -- drop-in for the reference precoders
// (reference proj/include/cgmimo/precode.hpp:17-45).
#pragma once

#include <cstddef>
#include <vector>

#include "cgmimo/linalg.hpp"

namespace cgmimo::precode {

struct PrecodeResult {
  ComplexVector precoded;   // q = H_d^H v_K, length B
  ComplexVector transmit;   // q / ||q||, zeros when zero_input
  double gain = 0.0;        // ||q||
  bool zero_input = false;
};

// (H_d H_d^H + rho_d^-1 I) v = t by K CG iterations, q = H_d^H v.  q_trace,
// when given, receives q_k for k = 1..K.
PrecodeResult precode_cg(const ComplexMatrix& h_downlink, const ComplexVector& t, double rho_d,
                         std::size_t iters, std::vector<ComplexVector>* q_trace = nullptr);

// q = H_d^H (H_d H_d^H + rho_d^-1 I)^-1 t through a Cholesky inverse.
PrecodeResult precode_explicit(const ComplexMatrix& h_downlink, const ComplexVector& t,
                               double rho_d);
// Minimum-norm CGLS; q_k per iteration into q_trace when given.
PrecodeResult precode_cgls(const ComplexMatrix& h_downlink, const ComplexVector& t, double rho_d,
                           std::size_t iters, std::vector<ComplexVector>* q_trace = nullptr);
// Truncated Neumann series of A_d^-1 with `terms` terms.
PrecodeResult precode_neumann(const ComplexMatrix& h_downlink, const ComplexVector& t,
                              double rho_d, std::size_t terms);

}  // namespace cgmimo::precode
