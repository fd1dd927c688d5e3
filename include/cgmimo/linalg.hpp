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

// Hermitian matrix as the packed lower triangle (reference linalg.hpp:42-65,
// same member layout): entry (i, j), j <= i, at i (i + 1) / 2 + j; the upper
// triangle is the conjugate mirror on access, so M == M^H holds exactly and
// the diagonal carries no imaginary part.  The GPU path keeps the Gram matrix
// in this form's full equivalent (lower triangle + exact conjugate mirror,
// real diagonal; csrc/cgm_tc.cuh epilogue).
class HermitianMatrix {
 public:
  HermitianMatrix() = default;
  explicit HermitianMatrix(std::size_t dim) : dim_(dim), tri_(dim * (dim + 1) / 2) {
    if (dim == 0) throw std::invalid_argument("HermitianMatrix: empty dimension");
  }
  static HermitianMatrix identity(std::size_t n) {
    HermitianMatrix m(n);
    for (std::size_t i = 0; i < n; ++i) m.set(i, i, 1.0);
    return m;
  }
  std::size_t dim() const { return dim_; }
  cplx at(std::size_t i, std::size_t j) const {
    return j <= i ? tri_[index(i, j)] : std::conj(tri_[index(j, i)]);
  }
  // j <= i required; stores only the real part on the diagonal.
  void set(std::size_t i, std::size_t j, cplx value) {
    if (j > i || i >= dim_) throw std::invalid_argument("HermitianMatrix::set: need j <= i < dim");
    tri_[index(i, j)] = i == j ? cplx(value.real(), 0.0) : value;
  }
  double diag(std::size_t i) const { return tri_[index(i, i)].real(); }
  std::vector<double> real_diag() const {
    std::vector<double> d(dim_);
    for (std::size_t i = 0; i < dim_; ++i) d[i] = diag(i);
    return d;
  }
  ComplexMatrix full() const {
    ComplexMatrix m(dim_, dim_);
    for (std::size_t i = 0; i < dim_; ++i)
      for (std::size_t j = 0; j < dim_; ++j) m(i, j) = at(i, j);
    return m;
  }

 private:
  std::size_t index(std::size_t i, std::size_t j) const { return i * (i + 1) / 2 + j; }
  std::size_t dim_ = 0;
  std::vector<cplx> tri_;
};

// conj-transpose (used to express TDD reciprocity H_d = H_u^H)
inline ComplexMatrix hermitian_of(const ComplexMatrix& m) {
  ComplexMatrix t(m.cols(), m.rows());
  for (std::size_t i = 0; i < m.rows(); ++i)
    for (std::size_t j = 0; j < m.cols(); ++j) t(j, i) = std::conj(m(i, j));
  return t;
}

}  // namespace cgmimo
