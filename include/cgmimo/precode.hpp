// cgmimo/precode.hpp -- drop-in for the reference CG precoder
// (reference proj/include/cgmimo/precode.hpp:17-33).
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

}  // namespace cgmimo::precode
