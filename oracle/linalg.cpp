// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// Dense kernels behind the oracle: OpenBLAS gemm and LAPACK Hermitian
// eigensolvers from the scipy wheel's bundled OpenBLAS
// (scipy.libs/libscipy_openblas-*.so, symbols prefixed `scipy_`).  They replace
// the Eigen operator* (mmp.cpp:73) and SelfAdjointEigenSolver
// (truncation.cpp:25) of the reference, which cannot be built here
// (no Eigen).
#include <algorithm>
#include <stdexcept>

#include "dense.hpp"
#include "linalg.hpp"

extern "C" {
void scipy_cblas_dgemm(int order, int ta, int tb, int m, int n, int k, double alpha,
                       const double* a, int lda, const double* b, int ldb, double beta, double* c,
                       int ldc);
void scipy_cblas_zgemm(int order, int ta, int tb, int m, int n, int k, const void* alpha,
                       const void* a, int lda, const void* b, int ldb, const void* beta, void* c,
                       int ldc);
void scipy_dsyevd_(const char* jobz, const char* uplo, const int* n, double* a, const int* lda,
                   double* w, double* work, const int* lwork, int* iwork, const int* liwork,
                   int* info, size_t, size_t);
void scipy_zheevd_(const char* jobz, const char* uplo, const int* n, void* a, const int* lda,
                   double* w, void* work, const int* lwork, double* rwork, const int* lrwork,
                   int* iwork, const int* liwork, int* info, size_t, size_t);
void scipy_openblas_set_num_threads(int);
}

namespace h2o {

namespace {
constexpr int kColMajor = 102, kNoTrans = 111, kTrans = 112, kConjTrans = 113;
int cblas_op(Op o) { return o == Op::N ? kNoTrans : (o == Op::T ? kTrans : kConjTrans); }
}  // namespace

void set_blas_threads(int n) { scipy_openblas_set_num_threads(n); }

template <class S>
void gemm(Op oa, Op ob, const Mat<S>& a, const Mat<S>& b, Mat<S>& c, bool accumulate) {
  const Index m = oa == Op::N ? a.r : a.c;
  const Index ka = oa == Op::N ? a.c : a.r;
  const Index kb = ob == Op::N ? b.r : b.c;
  const Index n = ob == Op::N ? b.c : b.r;
  if (ka != kb) throw std::logic_error("gemm: inner dimension mismatch");
  if (!accumulate) c = Mat<S>(m, n);
  else if (c.r != m || c.c != n) throw std::logic_error("gemm: accumulate shape mismatch");
  if (m == 0 || n == 0 || ka == 0) return;
  const int lda = static_cast<int>(std::max<Index>(1, a.r));
  const int ldb = static_cast<int>(std::max<Index>(1, b.r));
  const int ldc = static_cast<int>(std::max<Index>(1, c.r));
  if constexpr (is_complex_v<S>) {
    const Complex one(1.0, 0.0), beta(accumulate ? 1.0 : 0.0, 0.0);
    scipy_cblas_zgemm(kColMajor, cblas_op(oa), cblas_op(ob), static_cast<int>(m),
                      static_cast<int>(n), static_cast<int>(ka), &one, a.data(), lda, b.data(),
                      ldb, &beta, c.data(), ldc);
  } else {
    scipy_cblas_dgemm(kColMajor, cblas_op(oa), cblas_op(ob), static_cast<int>(m),
                      static_cast<int>(n), static_cast<int>(ka), 1.0, a.data(), lda, b.data(), ldb,
                      accumulate ? 1.0 : 0.0, c.data(), ldc);
  }
}

template void gemm<Real>(Op, Op, const Mat<Real>&, const Mat<Real>&, Mat<Real>&, bool);
template void gemm<Complex>(Op, Op, const Mat<Complex>&, const Mat<Complex>&, Mat<Complex>&,
                            bool);

// Hermitian eigendecomposition, eigenvalues ascending (same convention as
// Eigen's SelfAdjointEigenSolver, which reads the lower triangle).
template <>
bool hermitian_eig<Real>(const Mat<Real>& g, std::vector<double>& w, Mat<Real>& v) {
  const int n = static_cast<int>(g.r);
  v = g;
  w.assign(n, 0.0);
  int info = 0, lwork = -1, liwork = -1, iwq = 0;
  double wq = 0;
  scipy_dsyevd_("V", "L", &n, v.data(), &n, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
  lwork = static_cast<int>(wq);
  liwork = iwq;
  std::vector<double> work(std::max(1, lwork));
  std::vector<int> iwork(std::max(1, liwork));
  scipy_dsyevd_("V", "L", &n, v.data(), &n, w.data(), work.data(), &lwork, iwork.data(), &liwork,
                &info, 1, 1);
  return info == 0;
}

template <>
bool hermitian_eig<Complex>(const Mat<Complex>& g, std::vector<double>& w, Mat<Complex>& v) {
  const int n = static_cast<int>(g.r);
  v = g;
  w.assign(n, 0.0);
  int info = 0, lwork = -1, lrwork = -1, liwork = -1, iwq = 0;
  Complex wq;
  double rwq = 0;
  scipy_zheevd_("V", "L", &n, v.data(), &n, w.data(), &wq, &lwork, &rwq, &lrwork, &iwq, &liwork,
                &info, 1, 1);
  lwork = static_cast<int>(wq.real());
  lrwork = static_cast<int>(rwq);
  liwork = iwq;
  std::vector<Complex> work(std::max(1, lwork));
  std::vector<double> rwork(std::max(1, lrwork));
  std::vector<int> iwork(std::max(1, liwork));
  scipy_zheevd_("V", "L", &n, v.data(), &n, w.data(), work.data(), &lwork, rwork.data(), &lrwork,
                iwork.data(), &liwork, &info, 1, 1);
  return info == 0;
}

}  // namespace h2o
