// cgmimo/linalg.hpp -- drop-in subset (B200 build).
//
// The value types the reference hot-path signatures use
// (reference proj/include/cgmimo/linalg.hpp:15-37): complex<double> scalars,
// vectors, and a dense row-major matrix with element (i, j) at i*cols + j.
// Only what detect_cg / precode_cg callers need is provided; the reference's
// BLAS-style helpers are not part of the drop-in surface.
#pragma once

#include <complex>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace cgmimo {

using cplx = std::complex<double>;
using ComplexVector = std::vector<cplx>;

class ComplexMatrix {
 public:
  ComplexMatrix() = default;
  ComplexMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), a_(rows * cols) {
    if (rows == 0 || cols == 0) throw std::invalid_argument("ComplexMatrix: empty dimensions");
  }
  static ComplexMatrix identity(std::size_t n) {
    ComplexMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  cplx& operator()(std::size_t i, std::size_t j) { return a_[i * cols_ + j]; }
  const cplx& operator()(std::size_t i, std::size_t j) const { return a_[i * cols_ + j]; }
  const cplx* row(std::size_t i) const { return a_.data() + i * cols_; }
  cplx* row(std::size_t i) { return a_.data() + i * cols_; }
  const cplx* data() const { return a_.data(); }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<cplx> a_;
};

// conj-transpose (used to express TDD reciprocity H_d = H_u^H)
inline ComplexMatrix hermitian_of(const ComplexMatrix& m) {
  ComplexMatrix t(m.cols(), m.rows());
  for (std::size_t i = 0; i < m.rows(); ++i)
    for (std::size_t j = 0; j < m.cols(); ++j) t(j, i) = std::conj(m(i, j));
  return t;
}

}  // namespace cgmimo
