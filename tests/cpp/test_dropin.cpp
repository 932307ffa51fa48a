// Drop-in check of the C++ API (include/h2mmp): the reference's call sequence
// (tests/test_support.hpp:37-47 -> mmp(), test_mmp.cpp:50-59) compiled against
// the B200 headers and linked to libh2mmp_b200.so.  Prints one line per check;
// exit code 0 iff all pass.
#include <cmath>
#include <cstdio>
#include <string>
#include <memory>

#include "h2mmp/h2mmp.hpp"

using namespace h2mmp;

static int failures = 0;
#define CHECK(c)                                              \
  do {                                                        \
    const bool ok_ = (c);                                     \
    std::printf("%s: %s\n", ok_ ? "PASS" : "FAIL", #c);       \
    if (!ok_) ++failures;                                     \
  } while (0)

int main() {
  const PointSet pts = make_random_cloud(1024, 1);
  auto tree = std::make_shared<const ClusterTree>(build_cluster_tree(pts, 32));
  auto structure = build_block_tree(tree, tree, 1.0);
  CHECK(tree->depth == 5);
  CHECK(structure->c_sp() > 0);

  // operand: nested Chebyshev H^2 matrix from the library's input constructor
  h2c_h2* raw = h2c_build_chebyshev(&tree->desc, &structure->desc, tree->points.data(), 0, 0.0, 0.0, 3, 0.0, 4);
  CHECK(raw != nullptr);
  h2c_matrix d;
  h2c_h2_desc(raw, &d);
  d.tree = &tree->desc;
  d.blocks = &structure->desc;
  const H2Matrix<Real> a = detail::unflatten<Real>(d, tree, structure);
  h2c_h2_free(raw);

  const MmpResult<Real> r = mmp(a, a, 1e-6);
  CHECK(r.product.tree == a.tree && r.product.structure == a.structure);
  CHECK(r.report.pending_after_split == 0);
  CHECK(r.report.flops > 0 && r.report.levels.size() == static_cast<size_t>(tree->depth + 1));
  CHECK(r.product.coupling.size() == static_cast<size_t>(structure->admissible_count()));
  CHECK(r.product.full.size() == static_cast<size_t>(structure->inadmissible_count()));

  const DenseMatrix<Real> da = h2_to_dense(a);
  const DenseMatrix<Real> ref = da * da;
  const double err = (h2_to_dense(r.product) - ref).norm() / ref.norm();
  std::printf("dense relative error %.3e\n", err);
  CHECK(err <= 1e-4);

  const MmpResult<Real> f = formatted_mmp(a, a);
  CHECK(f.report.eps_trunc == 0.0 && !f.report.adaptive);

  bool threw = false;
  try {
    (void)mmp(a, a, 1.0);
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  auto other = std::make_shared<const ClusterTree>(build_cluster_tree(pts, 32));
  H2Matrix<Real> b = a;
  b.tree = other;
  threw = false;
  try {
    (void)mmp(a, b, 1e-6);
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  // validation order of mmp.cpp:58-63: different trees are reported even with a bad eps
  threw = false;
  try {
    (void)mmp(a, b, 2.0);
  } catch (const ConfigError& e) {
    threw = std::string(e.what()).find("share") != std::string::npos;
  }
  CHECK(threw);

  // h2_matrix.hpp:62-66 mvp (device) against the dense matrix
  DenseVector<Real> x(a.tree->size(), 1);
  for (Index i = 0; i < x.rows(); ++i) x(i, 0) = std::sin(0.37 * double(i));
  const DenseVector<Real> y = mvp(a, x);
  const DenseVector<Real> yd = da * x;
  CHECK((y - yd).norm() <= 1e-12 * yd.norm());

  // truncation.hpp:7-19 svd_truncate_gram (device eigensolver): test_truncation.cpp's KATs
  DenseMatrix<Real> g(4, 4);
  g(0, 0) = 1.0;
  g(1, 1) = 1e-1;
  g(2, 2) = 1e-3;
  const TruncatedBasis<Real> tb = svd_truncate_gram(g, 1e-2);
  CHECK(tb.basis.cols() == 2 && !tb.degenerate);
  const TruncatedBasis<Real> tz = svd_truncate_gram(DenseMatrix<Real>(5, 5), 1e-4);
  CHECK(tz.degenerate && tz.basis.cols() == 1 && tz.basis(0, 0) == 1.0);
  std::printf("%s\n", failures ? "DROPIN FAIL" : "DROPIN OK");
  return failures ? 1 : 0;
}
