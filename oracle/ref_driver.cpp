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

// ---------------------------------------------------------------------------
// Sliced reference arm of bench.py (`--impl reference`): the reference's own mmp()
// (single-threaded, as documented at mmp.hpp:58-66) run back to back on the bench
// workload, with its operands converted from the flat descriptors into the
// reference's types.  Progress is read from the Eigen shim's MAC counter (products +
// 9 n^3 per eigensolve, the reference's counting rule), so any time window of a
// running product yields a rate; completed products report their exact flops.
#include <chrono>
#include <thread>

extern "C" void scipy_openblas_set_num_threads(int);

namespace {

std::shared_ptr<const ClusterTree> tree_from_desc(const h2c_tree& d) {
  auto t = std::make_shared<ClusterTree>();
  t->clusters.resize(d.n_clusters);
  t->depth = d.depth;
  t->leafsize = d.leafsize;
  t->levels.assign(d.depth + 1, {});
  for (int c = 0; c < d.n_clusters; ++c) {
    Cluster& cl = t->clusters[c];
    cl.id = c;
    cl.parent = d.parent[c];
    cl.level = d.level[c];
    cl.begin = d.begin[c];
    cl.end = d.end[c];
    cl.child = {d.child0[c], d.child1[c]};
    if (d.bbox)
      for (int k = 0; k < 3; ++k) {
        cl.bbox_min[k] = d.bbox[6 * size_t(c) + k];
        cl.bbox_max[k] = d.bbox[6 * size_t(c) + 3 + k];
      }
    t->levels[cl.level].push_back(c);
  }
  for (auto& lv : t->levels)
    std::sort(lv.begin(), lv.end(), [&](int a, int b) { return t->clusters[a].begin < t->clusters[b].begin; });
  t->perm.assign(d.perm, d.perm + d.n_points);
  t->inv_perm.assign(d.n_points, 0);
  for (int p = 0; p < d.n_points; ++p) t->inv_perm[d.perm[p]] = p;
  return t;
}

template <class S>
DenseMatrix<S> read_mat(const h2c_matrix& d, int64_t off, Index r, Index c) {
  DenseMatrix<S> m(r, c);
  if (r * c) std::memcpy(static_cast<void*>(m.data()), reinterpret_cast<const S*>(d.values) + off, sizeof(S) * r * c);
  return m;
}

template <class S>
H2Matrix<S> h2_from_desc(const h2c_matrix& d, std::shared_ptr<const ClusterTree> tree,
                         std::shared_ptr<const BlockTree> st) {
  H2Matrix<S> h;
  h.tree = tree;
  h.structure = st;
  const int nc = static_cast<int>(tree->clusters.size());
  for (int side = 0; side < 2; ++side) {
    ClusterBasis<S>& b = side == 0 ? h.row_basis : h.col_basis;
    const int32_t* rk = side == 0 ? d.row_rank : d.col_rank;
    const uint8_t* dg = side == 0 ? d.row_degenerate : d.col_degenerate;
    const int64_t* off = side == 0 ? d.row_offset : d.col_offset;
    b.resize(nc);
    for (int c = 0; c < nc; ++c) {
      b.rank[c] = rk[c];
      b.degenerate[c] = dg[c];
      const Cluster& cl = tree->clusters[c];
      if (off[c] < 0) continue;
      if (cl.is_leaf())
        b.leaf[c] = read_mat<S>(d, off[c], cl.size(), rk[c]);
      else
        b.transfer[c] = read_mat<S>(d, off[c], rk[cl.child[0]] + rk[cl.child[1]], rk[c]);
    }
  }
  const h2c_blocks& bd = *d.blocks;
  for (int64_t k = 0; k < bd.n_blocks; ++k) {
    const BlockKey key{bd.row[k], bd.col[k]};
    if (bd.kind[k] == H2C_ADMISSIBLE)
      h.coupling[key] = read_mat<S>(d, d.block_offset[k], d.row_rank[key.row], d.col_rank[key.col]);
    else if (bd.kind[k] == H2C_INADMISSIBLE_LEAF)
      h.full[key] =
          read_mat<S>(d, d.block_offset[k], tree->clusters[key.row].size(), tree->clusters[key.col].size());
  }
  return h;
}

struct SlicedBase {
  virtual ~SlicedBase() = default;
  std::thread th;
  std::atomic<long long> products{0};
  std::atomic<long long> product_flops{0};
  std::string error;
};

template <class S>
struct Sliced : SlicedBase {
  H2Matrix<S> A, B;
  bool same = false;
  double eps = 0.0;
  bool adaptive = true;
  void loop() {
    try {
      for (;;) {
        const MmpResult<S> r = adaptive ? mmp(A, same ? A : B, eps) : formatted_mmp(A, same ? A : B);
        product_flops += r.report.flops;
        ++products;
      }
    } catch (const Eigen::internal::Aborted&) {
    } catch (const std::exception& e) {
      error = e.what();
    }
  }
};

}  // namespace

extern "C" {

/* Convert the operands (flat descriptors, same tree/blocks) into the reference's types and start
 * the reference's products back to back on a worker thread (BLAS single-threaded, like Eigen
 * without OpenMP).  Returns nullptr on error; *code as h2r_run. */
void* h2r_sliced_start(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive, int* code) {
  *code = 0;
  try {
    if (a->tree != b->tree || a->blocks != b->blocks)
      throw ConfigError("mmp: operands must share cluster trees and block structure");
    scipy_openblas_set_num_threads(1);
    auto tree = tree_from_desc(*a->tree);
    auto st = build_block_tree(tree, tree, a->blocks->eta);
    // the reference's partition must be the one the descriptors carry
    FlatBlocks fb;
    flatten_blocks(*st, fb);
    const h2c_blocks& d = *a->blocks;
    if (fb.row.size() != size_t(d.n_blocks) || !std::equal(fb.row.begin(), fb.row.end(), d.row) ||
        !std::equal(fb.col.begin(), fb.col.end(), d.col) || !std::equal(fb.kind.begin(), fb.kind.end(), d.kind))
      throw InvariantError("reference block tree differs from the descriptor's");
    auto start = [&](auto tag) -> SlicedBase* {
      using S = decltype(tag);
      auto s = std::make_unique<Sliced<S>>();
      s->A = h2_from_desc<S>(*a, tree, st);
      s->same = a == b || (a->values == b->values && a->row_offset == b->row_offset);
      if (!s->same) s->B = h2_from_desc<S>(*b, tree, st);
      s->eps = eps;
      s->adaptive = adaptive != 0;
      Eigen::internal::abort_flag() = false;
      Sliced<S>* raw = s.get();
      s->th = std::thread([raw] { raw->loop(); });
      return s.release();
    };
    if (a->scalar == H2C_COMPLEX) return start(Complex{});
    return start(Real{});
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

/* Let the product run for `seconds`; returns the elapsed wall time, the MACs counted in the window
 * and the number of products completed so far (and their exact reference flops). */
int h2r_sliced_step(void* h, double seconds, double* elapsed, int64_t* macs, int64_t* products,
                    int64_t* product_flops) {
  auto* s = static_cast<SlicedBase*>(h);
  const long long m0 = Eigen::internal::mac_counter().load();
  const auto t0 = std::chrono::steady_clock::now();
  std::this_thread::sleep_for(std::chrono::duration<double>(seconds));
  const long long m1 = Eigen::internal::mac_counter().load();
  *elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *macs = m1 - m0;
  *products = s->products.load();
  *product_flops = s->product_flops.load();
  if (!s->error.empty()) {
    g_err = s->error;
    return 1;
  }
  return 0;
}

void h2r_sliced_stop(void* h) {
  auto* s = static_cast<SlicedBase*>(h);
  Eigen::internal::abort_flag() = true;
  if (s->th.joinable()) s->th.join();
  Eigen::internal::abort_flag() = false;
  delete s;
}

/* MACs counted by the shim since load (for checking the counter against MmpReport.flops) */
long long h2r_mac_counter(void) { return Eigen::internal::mac_counter().load(); }

}  // extern "C"
