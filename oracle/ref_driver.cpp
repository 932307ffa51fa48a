// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C-ABI driver around the REFERENCE's own MMP path, compiled here from the
// unmodified sources under /root/reference/proj/core (geometry.cpp,
// cluster_tree.cpp, block_tree.cpp, h2_matrix.cpp, truncation.cpp, mmp.cpp,
// metrics.cpp) with oracle/eigen_shim standing in for Eigen (absent from this
// image).  Built into oracle/_ref/libh2ref.so by `make -C oracle ref`; used
// only by tools/make_ref_golden.py (which writes tests/golden/ref_cases.npz)
// and by the CPU tests that pin the oracle restatement against it.  Nothing in
// the product path, the GPU tests or bench.py loads it.
//
// One call runs the reference's whole case pipeline (the sequence of
// proj/tests/test_mmp.cpp / acceptance.cpp):
//   generate_geometry -> build_cluster_tree -> build_block_tree ->
//   assemble_dense -> build_h2 -> mmp / formatted_mmp
// and exposes tree, block structure, A, C and the MmpReport in the flat
// layout of include/h2c_types.h.
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../include/h2c_types.h"
#include "h2mmp/block_tree.hpp"
#include "h2mmp/cluster_tree.hpp"
#include "h2mmp/errors.hpp"
#include "h2mmp/geometry.hpp"
#include "h2mmp/h2_matrix.hpp"
#include "h2mmp/metrics.hpp"
#include "h2mmp/mmp.hpp"
#include "h2mmp/truncation.hpp"

using namespace h2mmp;

namespace {

thread_local std::string g_err;

struct FlatTree {
  std::vector<int32_t> parent, child0, child1, level, begin, end, perm;
  std::vector<double> bbox;
  h2c_tree desc{};
};

struct FlatBlocks {
  std::vector<int64_t> level_ptr;
  std::vector<int32_t> row, col;
  std::vector<uint8_t> kind;
  h2c_blocks desc{};
};

struct FlatH2 {
  std::vector<int32_t> row_rank, col_rank;
  std::vector<uint8_t> row_dg, col_dg;
  std::vector<int64_t> row_off, col_off, block_off;
  std::vector<double> values;
  h2c_matrix desc{};
};

struct FlatReport {
  std::vector<int64_t> max_row_rank, max_col_rank, case_products;
  std::vector<int32_t> t1, t2, t3;
  h2c_report desc{};
};

void flatten_tree(const ClusterTree& t, FlatTree& f) {
  const int nc = static_cast<int>(t.clusters.size());
  f.parent.resize(nc);
  f.child0.resize(nc);
  f.child1.resize(nc);
  f.level.resize(nc);
  f.begin.resize(nc);
  f.end.resize(nc);
  f.bbox.resize(6 * size_t(nc));
  for (int c = 0; c < nc; ++c) {
    const Cluster& cl = t.clusters[c];
    f.parent[c] = cl.parent;
    f.child0[c] = cl.child[0];
    f.child1[c] = cl.child[1];
    f.level[c] = cl.level;
    f.begin[c] = cl.begin;
    f.end[c] = cl.end;
    for (int d = 0; d < 3; ++d) {
      f.bbox[6 * size_t(c) + d] = cl.bbox_min[d];
      f.bbox[6 * size_t(c) + 3 + d] = cl.bbox_max[d];
    }
  }
  f.perm.assign(t.perm.begin(), t.perm.end());
  f.desc = h2c_tree{t.size(), t.depth, t.leafsize, nc, f.parent.data(), f.child0.data(), f.child1.data(),
                    f.level.data(), f.begin.data(), f.end.data(), f.bbox.data(), f.perm.data()};
}

void flatten_blocks(const BlockTree& b, FlatBlocks& f) {
  f.level_ptr.assign(1, 0);
  for (int l = 0; l <= b.depth(); ++l) {
    for (const BlockEntry& e : b.level_blocks(l)) {
      f.row.push_back(e.key.row);
      f.col.push_back(e.key.col);
      f.kind.push_back(static_cast<uint8_t>(e.kind));
    }
    f.level_ptr.push_back(static_cast<int64_t>(f.row.size()));
  }
  f.desc = h2c_blocks{b.depth(), b.c_sp(), b.eta(), static_cast<int64_t>(f.row.size()), f.level_ptr.data(),
                      f.row.data(), f.col.data(), f.kind.data()};
}

template <class S>
void flatten_h2(const H2Matrix<S>& h, const FlatTree& ft, const FlatBlocks& fb, FlatH2& f) {
  constexpr int W = std::is_same_v<S, Complex> ? 2 : 1;
  const ClusterTree& t = *h.tree;
  const int nc = static_cast<int>(t.clusters.size());
  int64_t n = 0;
  auto add = [&](const DenseMatrix<S>& m) {
    const int64_t at = n;
    const double* p = reinterpret_cast<const double*>(m.data());
    f.values.insert(f.values.end(), p, p + W * m.size());
    n += m.size();
    return at;
  };
  for (int side = 0; side < 2; ++side) {
    const ClusterBasis<S>& b = side == 0 ? h.row_basis : h.col_basis;
    auto& rk = side == 0 ? f.row_rank : f.col_rank;
    auto& dg = side == 0 ? f.row_dg : f.col_dg;
    auto& off = side == 0 ? f.row_off : f.col_off;
    rk.assign(nc, 0);
    dg.assign(nc, 0);
    off.assign(nc, -1);
    for (int c = 0; c < nc; ++c) {
      rk[c] = static_cast<int32_t>(b.rank[c]);
      dg[c] = b.degenerate[c] ? 1 : 0;
      const Cluster& cl = t.clusters[c];
      if (cl.parent < 0 && !cl.is_leaf()) continue;
      off[c] = add(cl.is_leaf() ? b.leaf[c] : b.transfer[c]);
    }
  }
  f.block_off.assign(fb.row.size(), -1);
  for (size_t k = 0; k < fb.row.size(); ++k) {
    const BlockKey key{fb.row[k], fb.col[k]};
    if (fb.kind[k] == H2C_ADMISSIBLE)
      f.block_off[k] = add(h.coupling.at(key));
    else if (fb.kind[k] == H2C_INADMISSIBLE_LEAF)
      f.block_off[k] = add(h.full.at(key));
  }
  f.desc = h2c_matrix{&ft.desc, &fb.desc, W == 2 ? H2C_COMPLEX : H2C_REAL, f.row_rank.data(), f.col_rank.data(),
                      f.row_dg.data(), f.col_dg.data(), f.row_off.data(), f.col_off.data(), f.block_off.data(),
                      f.values.data(), n};
}

void flatten_report(const MmpReport& r, FlatReport& f) {
  const int nl = static_cast<int>(r.levels.size());
  for (const LevelStats& s : r.levels) {
    f.max_row_rank.push_back(s.max_row_rank);
    f.max_col_rank.push_back(s.max_col_rank);
    for (int c = 0; c < 4; ++c) f.case_products.push_back(s.case_products[c]);
    f.t1.push_back(s.max_case1_terms);
    f.t2.push_back(s.max_case2_terms);
    f.t3.push_back(s.max_case3_terms);
  }
  h2c_report& d = f.desc;
  d = h2c_report{};
  d.eps_trunc = r.eps_trunc;
  d.adaptive = r.adaptive ? 1 : 0;
  d.n_levels = nl;
  d.flops = r.flops;
  for (int c = 0; c < 4; ++c) d.case_flops[c] = r.case_flops[c];
  d.wall_seconds = r.wall_seconds;
  d.pending_after_split = r.pending_after_split;
  d.max_row_rank = f.max_row_rank.data();
  d.max_col_rank = f.max_col_rank.data();
  d.case_products = f.case_products.data();
  d.max_case1_terms = f.t1.data();
  d.max_case2_terms = f.t2.data();
  d.max_case3_terms = f.t3.data();
}

struct CaseBase {
  virtual ~CaseBase() = default;
  FlatTree tree;
  FlatBlocks blocks;
  FlatH2 a, c;
  FlatReport report;
  bool has_product = false;
  virtual void mvp(int which, const double* x, int nv, double* y) const = 0;
  virtual double relative_error(uint64_t seed, int* ref_zero) const = 0;
};

template <class S>
struct Case : CaseBase {
  std::shared_ptr<const BlockTree> structure;
  H2Matrix<S> A;
  MmpResult<S> R;
  void mvp(int which, const double* x, int nv, double* y) const override {
    const H2Matrix<S>& h = which == 0 ? A : R.product;
    const int n = h.size();
    const S* xs = reinterpret_cast<const S*>(x);
    S* ys = reinterpret_cast<S*>(y);
    for (int v = 0; v < nv; ++v) {
      DenseVector<S> xv(n);
      for (int i = 0; i < n; ++i) xv(i) = xs[size_t(v) * n + i];
      const DenseVector<S> yv = h2mmp::mvp(h, xv);
      for (int i = 0; i < n; ++i) ys[size_t(v) * n + i] = yv(i);
    }
  }
  double relative_error(uint64_t seed, int* ref_zero) const override {
    const RelativeError e = h2mmp::relative_error(A, A, R.product, seed);
    if (ref_zero) *ref_zero = e.reference_was_zero ? 1 : 0;
    return e.value;
  }
};

template <class S>
CaseBase* run_case(const PointSet& pts, int leafsize, double eta, const Kernel& kernel, double eps_h2, double eps,
                   int mode) {
  auto c = std::make_unique<Case<S>>();
  auto tree = std::make_shared<const ClusterTree>(build_cluster_tree(pts, leafsize));
  c->structure = build_block_tree(tree, tree, eta);
  const DenseMatrix<S> dense = assemble_dense<S>(pts, kernel);
  c->A = build_h2<S>(dense, c->structure, eps_h2);
  flatten_tree(*tree, c->tree);
  flatten_blocks(*c->structure, c->blocks);
  flatten_h2(c->A, c->tree, c->blocks, c->a);
  if (mode != 2) {
    c->R = mode == 0 ? mmp(c->A, c->A, eps) : formatted_mmp(c->A, c->A);
    flatten_h2(c->R.product, c->tree, c->blocks, c->c);
    flatten_report(c->R.report, c->report);
    c->has_product = true;
  }
  return c.release();
}

}  // namespace

extern "C" {

const char* h2r_last_error(void) { return g_err.c_str(); }

/* family: 0 random_cloud, 1 bus, 2 slab, 3 cube_array; helmholtz 0/1;
 * mode: 0 mmp(A, A, eps), 1 formatted_mmp(A, A), 2 build A only.
 * Returns nullptr on error (h2r_last_error; *code = 2 ConfigError,
 * 3 InvariantError, 1 other). */
void* h2r_run(int family, uint64_t seed, int n, int bus_count, int samples_per_meter, int slab_width,
              int slab_thickness, int array_edge, int cube_points, int leafsize, double eta, int helmholtz,
              double wavenumber, int has_diag, double diag, double eps_h2, double eps, int mode, int* code) {
  *code = 0;
  try {
    GeometrySpec spec;
    spec.family = static_cast<Family>(family);
    spec.seed = seed;
    spec.n = n;
    spec.bus_count = bus_count;
    spec.samples_per_meter = samples_per_meter;
    spec.slab_width = slab_width;
    spec.slab_thickness = slab_thickness;
    spec.array_edge = array_edge;
    spec.cube_points = cube_points;
    const PointSet pts = generate_geometry(spec);
    Kernel kernel;
    kernel.kind = helmholtz ? KernelKind::helmholtz : KernelKind::laplace;
    kernel.wavenumber = wavenumber;
    if (has_diag) kernel.diagonal_value = diag;
    if (helmholtz) return run_case<Complex>(pts, leafsize, eta, kernel, eps_h2, eps, mode);
    return run_case<Real>(pts, leafsize, eta, kernel, eps_h2, eps, mode);
  } catch (const ConfigError& e) {
    g_err = e.what();
    *code = 2;
  } catch (const InvariantError& e) {
    g_err = e.what();
    *code = 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    *code = 1;
  }
  return nullptr;
}

void h2r_tree(const void* h, h2c_tree* out) { *out = static_cast<const CaseBase*>(h)->tree.desc; }
void h2r_blocks(const void* h, h2c_blocks* out) { *out = static_cast<const CaseBase*>(h)->blocks.desc; }
/* which: 0 = A, 1 = C (0 if the case ran mode 2) */
int h2r_matrix(const void* h, int which, h2c_matrix* out) {
  const CaseBase* c = static_cast<const CaseBase*>(h);
  if (which == 1 && !c->has_product) return 2;
  *out = which == 0 ? c->a.desc : c->c.desc;
  return 0;
}
int h2r_report(const void* h, h2c_report* out) {
  const CaseBase* c = static_cast<const CaseBase*>(h);
  if (!c->has_product) return 2;
  *out = c->report.desc;
  return 0;
}
/* y[:, v] = M x[:, v] with the reference's mvp (h2_matrix.cpp:213-278), M = A or C */
int h2r_mvp(const void* h, int which, const double* x, int nv, double* y) {
  const CaseBase* c = static_cast<const CaseBase*>(h);
  if (which == 1 && !c->has_product) return 2;
  try {
    c->mvp(which, x, nv, y);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
  return 0;
}
/* metrics.cpp:37-55 with a = b = A, c = C */
double h2r_relative_error(const void* h, uint64_t seed, int* ref_zero) {
  return static_cast<const CaseBase*>(h)->relative_error(seed, ref_zero);
}
/* truncation.cpp:9-47 on one Gram (n x n, complex interleaved); basis_out n*n scalars */
int h2r_truncate_gram(int complex_, const double* gram, int n, double eps, double* basis_out, int* rank,
                      int* degenerate) {
  try {
    auto run = [&](auto tag) {
      using S = decltype(tag);
      constexpr int W = std::is_same_v<S, Complex> ? 2 : 1;
      DenseMatrix<S> g(n, n);
      std::memcpy(static_cast<void*>(g.data()), gram, sizeof(double) * W * n * n);
      const TruncatedBasis<S> t = svd_truncate_gram<S>(g, eps);
      *rank = static_cast<int>(t.basis.cols());
      *degenerate = t.degenerate ? 1 : 0;
      std::memcpy(basis_out, static_cast<const void*>(t.basis.data()), sizeof(double) * W * t.basis.size());
    };
    if (complex_)
      run(Complex{});
    else
      run(Real{});
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const InvariantError& e) {
    g_err = e.what();
    return 3;
  }
  return 0;
}
void h2r_free(void* h) { delete static_cast<CaseBase*>(h); }

}  // extern "C"

extern "C" {
/* products whose inner dimensions disagreed (Eigen's compiled-out assert; must stay 0 for real cases) */
long long h2r_shape_mismatches(void) { return Eigen::internal::shape_mismatches(); }
}
