// ORACLE — TEST INFRASTRUCTURE ONLY.  Nothing in paper_1908_05218_b200/
// links, imports or executes this directory; only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs do, as the checker.
//
// Minimal column-major dense matrix standing in for the reference's
// DenseMatrix<Scalar> = Eigen::Matrix<Scalar,Dynamic,Dynamic>
// (proj/core/include/h2mmp/dense.hpp:9-20).  Eigen is absent from this image
// (SURVEY.md §0.2); products go to OpenBLAS (the scipy wheel's bundled copy).
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace h2o {

using Real = double;
using Complex = std::complex<double>;
using Index = std::int64_t;

template <class S>
inline constexpr bool is_complex_v = std::is_same_v<S, Complex>;

template <class S>
inline S conj_s(const S& x) {
  if constexpr (is_complex_v<S>) return std::conj(x);
  else return x;
}
template <class S>
inline double abs2(const S& x) {
  if constexpr (is_complex_v<S>) return std::norm(x);
  else return x * x;
}

template <class S>
struct Mat {
  Index r = 0, c = 0;
  std::vector<S> d;

  Mat() = default;
  Mat(Index rows, Index cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols)) {}
  static Mat zero(Index rows, Index cols) { return Mat(rows, cols); }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = S(1);
    return m;
  }
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  S* data() { return d.data(); }
  const S* data() const { return d.data(); }
  S& operator()(Index i, Index j) { return d[static_cast<size_t>(i + j * r)]; }
  const S& operator()(Index i, Index j) const { return d[static_cast<size_t>(i + j * r)]; }

  Mat transpose() const {
    Mat t(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  Mat adjoint() const {
    Mat t(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) t(j, i) = conj_s((*this)(i, j));
    return t;
  }
  Mat conjugate() const {
    Mat t = *this;
    if constexpr (is_complex_v<S>)
      for (auto& x : t.d) x = std::conj(x);
    return t;
  }
  // contiguous row range [r0, r0+n)
  Mat rows_range(Index r0, Index n) const {
    Mat t(n, c);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < n; ++i) t(i, j) = (*this)(r0 + i, j);
    return t;
  }
  Mat block(Index r0, Index c0, Index nr, Index nc) const {
    Mat t(nr, nc);
    for (Index j = 0; j < nc; ++j)
      for (Index i = 0; i < nr; ++i) t(i, j) = (*this)(r0 + i, c0 + j);
    return t;
  }
  void set_block(Index r0, Index c0, const Mat& b) {
    for (Index j = 0; j < b.c; ++j)
      for (Index i = 0; i < b.r; ++i) (*this)(r0 + i, c0 + j) = b(i, j);
  }
  void add_block(Index r0, Index c0, const Mat& b) {
    for (Index j = 0; j < b.c; ++j)
      for (Index i = 0; i < b.r; ++i) (*this)(r0 + i, c0 + j) += b(i, j);
  }
  Mat& operator+=(const Mat& o) {
    if (o.r != r || o.c != c) throw std::logic_error("Mat += shape mismatch");
    for (size_t k = 0; k < d.size(); ++k) d[k] += o.d[k];
    return *this;
  }
  Mat& operator-=(const Mat& o) {
    if (o.r != r || o.c != c) throw std::logic_error("Mat -= shape mismatch");
    for (size_t k = 0; k < d.size(); ++k) d[k] -= o.d[k];
    return *this;
  }
  // Frobenius norm (Eigen's norm(): sqrt of the squared sum)
  double norm() const {
    double s = 0.0;
    for (const auto& x : d) s += abs2(x);
    return std::sqrt(s);
  }
  bool is_zero() const {
    for (const auto& x : d)
      if (x != S(0)) return false;
    return true;
  }
  void set_zero() { std::fill(d.begin(), d.end(), S(0)); }
};

template <class S>
inline Mat<S> operator-(const Mat<S>& a, const Mat<S>& b) {
  Mat<S> t = a;
  t -= b;
  return t;
}

// C = op(A) * op(B) with op in {N, T, C(adjoint)} through OpenBLAS gemm.
enum class Op { N, T, H };
template <class S>
void gemm(Op oa, Op ob, const Mat<S>& a, const Mat<S>& b, Mat<S>& c, bool accumulate);

template <class S>
inline Mat<S> mul(const Mat<S>& a, const Mat<S>& b) {
  Mat<S> c;
  gemm(Op::N, Op::N, a, b, c, false);
  return c;
}
template <class S>
inline Mat<S> mul(Op oa, const Mat<S>& a, Op ob, const Mat<S>& b) {
  Mat<S> c;
  gemm(oa, ob, a, b, c, false);
  return c;
}

}  // namespace h2o
