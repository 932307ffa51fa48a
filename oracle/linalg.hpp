// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
#pragma once

#include <vector>

#include "dense.hpp"

namespace h2o {

void set_blas_threads(int n);

// Hermitian eigendecomposition (lower triangle), eigenvalues ascending.
template <class S>
bool hermitian_eig(const Mat<S>& g, std::vector<double>& w, Mat<S>& v);

}  // namespace h2o
