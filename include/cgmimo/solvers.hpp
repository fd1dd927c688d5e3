// cgmimo/solvers.hpp -- drop-in subset: the error types the hot path raises
// (reference proj/include/cgmimo/solvers.hpp:21-27).
#pragma once

#include <stdexcept>

namespace cgmimo::solvers {

// p^H A p below 1e-30 inside the CG loop (reference solvers.cpp:55-57).
struct SolverBreakdown : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct NotPositiveDefinite : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace cgmimo::solvers
