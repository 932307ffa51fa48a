// Drop-in restatement of proj/core/include/h2mmp/dense.hpp:9-20 without Eigen:
// Real / Complex / Index and a column-major owning DenseMatrix<Scalar> with
// the members the MMP path's callers use (rows, cols, data, operator(),
// Zero, Identity, transpose, adjoint, conjugate, norm, products).
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace h2mmp {

using Real = double;
using Complex = std::complex<double>;
using Index = std::ptrdiff_t;

template <class Scalar>
inline constexpr bool is_complex_v = std::is_same_v<Scalar, Complex>;

template <class Scalar>
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), Scalar(0)) {}
  static DenseMatrix Zero(Index r, Index c) { return DenseMatrix(r, c); }
  static DenseMatrix Identity(Index r, Index c) {
    DenseMatrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = Scalar(1);
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Scalar* data() { return d_.data(); }
  const Scalar* data() const { return d_.data(); }
  Scalar& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
  const Scalar& operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
  void setZero() { std::fill(d_.begin(), d_.end(), Scalar(0)); }

  DenseMatrix transpose() const {
    DenseMatrix t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  DenseMatrix conjugate() const {
    DenseMatrix t = *this;
    if constexpr (is_complex_v<Scalar>)
      for (auto& x : t.d_) x = std::conj(x);
    return t;
  }
  DenseMatrix adjoint() const { return transpose().conjugate(); }
  double norm() const {
    double s = 0;
    for (const auto& x : d_) s += std::norm(x);
    return std::sqrt(s);
  }
  DenseMatrix& operator+=(const DenseMatrix& o) {
    check(o);
    for (size_t k = 0; k < d_.size(); ++k) d_[k] += o.d_[k];
    return *this;
  }
  DenseMatrix& operator-=(const DenseMatrix& o) {
    check(o);
    for (size_t k = 0; k < d_.size(); ++k) d_[k] -= o.d_[k];
    return *this;
  }
  friend DenseMatrix operator+(DenseMatrix a, const DenseMatrix& b) { return a += b; }
  friend DenseMatrix operator-(DenseMatrix a, const DenseMatrix& b) { return a -= b; }
  friend DenseMatrix operator*(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.c_ != b.r_) throw std::invalid_argument("DenseMatrix: inner dimensions differ");
    DenseMatrix c(a.r_, b.c_);
    for (Index j = 0; j < b.c_; ++j)
      for (Index k = 0; k < a.c_; ++k) {
        const Scalar bk = b(k, j);
        for (Index i = 0; i < a.r_; ++i) c(i, j) += a(i, k) * bk;
      }
    return c;
  }

 private:
  void check(const DenseMatrix& o) const {
    if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("DenseMatrix: shape mismatch");
  }
  Index r_ = 0, c_ = 0;
  std::vector<Scalar> d_;
};

template <class Scalar>
using DenseVector = DenseMatrix<Scalar>;  // n x 1

}  // namespace h2mmp
