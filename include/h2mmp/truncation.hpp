// truncation.hpp of the reference (proj/core/include/h2mmp/truncation.hpp:7-19):
// TruncatedBasis and svd_truncate_gram with the same names and semantics, computed
// on the B200 by the product's own batched Hermitian eigensolver
// (paper_1908_05218_b200/csrc/heev.cuh) through h2c_truncate_gram.
#pragma once

#include <type_traits>
#include <vector>

#include "h2mmp/context.hpp"
#include "h2mmp/dense.hpp"

namespace h2mmp {

template <class Scalar>
struct TruncatedBasis {
  DenseMatrix<Scalar> basis;  // n x r, orthonormal columns, r >= 1
  bool degenerate = false;    // set when the Gram matrix carried no content
};

/// truncation.cpp:9-47: orthonormal eigenvectors of the Hermitian PSD Gram whose
/// eigenvalues exceed eps * lambda_max (strict), at least one; an exactly zero Gram
/// gives e_1 with the degenerate flag.  ConfigError unless square, non-empty and
/// eps in (0,1).
template <class Scalar>
TruncatedBasis<Scalar> svd_truncate_gram(const DenseMatrix<Scalar>& gram, double eps) {
  if (gram.rows() != gram.cols() || gram.rows() < 1)
    throw ConfigError("svd_truncate_gram: gram matrix must be square and non-empty");
  if (!(eps > 0.0 && eps < 1.0)) throw ConfigError("svd_truncate_gram: eps must be in (0,1)");
  const int n = static_cast<int>(gram.rows());
  const int scalar = std::is_same_v<Scalar, Complex> ? H2C_COMPLEX : H2C_REAL;
  std::vector<Scalar> basis(static_cast<size_t>(n) * n);
  int rank = 0, degen = 0;
  h2c_context* ctx = detail::default_context();
  detail::rethrow(h2c_truncate_gram(ctx, scalar, reinterpret_cast<const double*>(gram.data()), n, eps,
                                    reinterpret_cast<double*>(basis.data()), &rank, &degen),
                  ctx);
  TruncatedBasis<Scalar> out;
  out.basis = DenseMatrix<Scalar>(n, rank);
  for (int c = 0; c < rank; ++c)
    for (int r = 0; r < n; ++r) out.basis(r, c) = basis[r + static_cast<size_t>(c) * n];
  out.degenerate = degen != 0;
  return out;
}

}  // namespace h2mmp
