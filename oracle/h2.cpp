// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// Restatement of truncation.cpp (Gram-eigenvalue truncation), h2_matrix.cpp
// (dense -> H^2 construction for small N, materialisation, exact MVP,
// footprint) and metrics.cpp (random vectors, MVP-based relative error).
#include <algorithm>
#include <cmath>
#include <random>

#include "linalg.hpp"
#include "model.hpp"

namespace h2o {

// truncation.cpp:9-47 — keep eigenvectors with lambda_i > eps * lambda_max
// (strict), at least one; exactly-zero Gram -> flagged e_1; descending order.
template <class S>
TruncatedBasis<S> svd_truncate_gram(const Mat<S>& gram, double eps) {
  if (gram.r != gram.c || gram.r < 1)
    throw ConfigError("svd_truncate_gram: gram matrix must be square and non-empty");
  if (!(eps > 0.0 && eps < 1.0)) throw ConfigError("svd_truncate_gram: eps must be in (0,1)");
  const Index n = gram.r;
  auto unit = [n] {
    TruncatedBasis<S> u;
    u.basis = Mat<S>(n, 1);
    u.basis(0, 0) = S(1);
    u.degenerate = true;
    return u;
  };
  if (gram.is_zero()) return unit();
  std::vector<double> w;
  Mat<S> v;
  if (!hermitian_eig(gram, w, v)) throw InvariantError("svd_truncate_gram: eigendecomposition failed");
  for (auto& x : w) x = std::max(x, 0.0);
  const double top = w[n - 1];
  if (top <= 0.0) return unit();
  Index rank = 0;
  while (rank < n && w[n - 1 - rank] > eps * top) ++rank;
  rank = std::max<Index>(rank, 1);
  TruncatedBasis<S> out;
  out.basis = Mat<S>(n, rank);
  for (Index c = 0; c < rank; ++c)
    for (Index r = 0; r < n; ++r) out.basis(r, c) = v(r, n - 1 - c);
  out.degenerate = false;
  out.eigenvalues = std::move(w);
  return out;
}
template TruncatedBasis<Real> svd_truncate_gram<Real>(const Mat<Real>&, double);
template TruncatedBasis<Complex> svd_truncate_gram<Complex>(const Mat<Complex>&, double);

namespace {

template <class S>
Mat<S> tree_order(const Mat<S>& dense, const ClusterTree& t) {
  const int n = t.size();
  Mat<S> out(n, n);
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a) out(a, b) = dense(t.perm[a], t.perm[b]);
  return out;
}

// h2_matrix.cpp:21-47 — admissible partners of a cluster and of all its
// ancestors (its far field)
std::vector<std::vector<int>> far_field(const BlockTree& bt, bool row_side) {
  const ClusterTree& t = row_side ? bt.rows() : bt.cols();
  std::vector<std::vector<int>> p(t.clusters.size());
  for (int l = 0; l <= bt.depth(); ++l)
    for (const BlockEntry& e : bt.level_blocks(l)) {
      if (e.kind != BlockKind::admissible) continue;
      if (row_side) p[e.key.row].push_back(e.key.col);
      else p[e.key.col].push_back(e.key.row);
    }
  for (int l = 0; l < bt.depth(); ++l)
    for (int id : t.levels[l]) {
      const Cluster& c = t.clusters[id];
      if (c.is_leaf()) continue;
      for (int ch : c.child) p[ch].insert(p[ch].end(), p[id].begin(), p[id].end());
    }
  return p;
}

// h2_matrix.cpp:49-122 — one side's nested orthonormal basis from far-field
// Gram sums, leaves first, then transfers bottom-up.
template <class S>
struct Side {
  const ClusterTree& t;
  const ClusterTree& other;
  const Mat<S>& dt;
  const std::vector<std::vector<int>>& partners;
  bool transposed;
  double eps;
  ClusterBasis<S> basis;
  std::vector<Mat<S>> mat;

  Mat<S> far_block(const Cluster& c, int partner) const {
    const Cluster& s = other.clusters[partner];
    if (transposed) return dt.block(s.begin, c.begin, s.size(), c.size()).transpose();
    return dt.block(c.begin, s.begin, c.size(), s.size());
  }
  void build() {
    basis.resize(t.clusters.size());
    mat.resize(t.clusters.size());
    for (int id : t.levels[t.depth]) leaf(t.clusters[id]);
    for (int l = t.depth - 1; l >= 1; --l)
      for (int id : t.levels[l]) transfer(t.clusters[id]);
  }
  void leaf(const Cluster& c) {
    Mat<S> g(c.size(), c.size());
    for (int p : partners[c.id]) {
      const Mat<S> blk = far_block(c, p);
      gemm(Op::N, Op::H, blk, blk, g, true);
    }
    auto tr = svd_truncate_gram<S>(g, eps);
    basis.leaf[c.id] = tr.basis;
    basis.rank[c.id] = tr.basis.c;
    basis.degenerate[c.id] = tr.degenerate || partners[c.id].empty();
    mat[c.id] = basis.leaf[c.id];
  }
  void transfer(const Cluster& c) {
    const Mat<S>& m1 = mat[c.child[0]];
    const Mat<S>& m2 = mat[c.child[1]];
    const Index k1 = m1.c, k2 = m2.c;
    const Cluster& c1 = t.clusters[c.child[0]];
    Mat<S> g(k1 + k2, k1 + k2);
    for (int p : partners[c.id]) {
      const Mat<S> blk = far_block(c, p);
      Mat<S> z(k1 + k2, blk.c);
      z.set_block(0, 0, mul(Op::H, m1, Op::N, blk.rows_range(0, c1.size())));
      z.set_block(k1, 0, mul(Op::H, m2, Op::N, blk.rows_range(c1.size(), c.size() - c1.size())));
      gemm(Op::N, Op::H, z, z, g, true);
    }
    auto tr = svd_truncate_gram<S>(g, eps);
    basis.transfer[c.id] = tr.basis;
    basis.rank[c.id] = tr.basis.c;
    basis.degenerate[c.id] = tr.degenerate || partners[c.id].empty();
    Mat<S> m(c.size(), tr.basis.c);
    m.set_block(0, 0, mul(m1, tr.basis.rows_range(0, k1)));
    m.set_block(c1.size(), 0, mul(m2, tr.basis.rows_range(k1, k2)));
    mat[c.id] = std::move(m);
  }
};

// h2_matrix.cpp:124-137
template <class S>
Mat<S> materialize(const ClusterBasis<S>& b, const ClusterTree& t, int id) {
  const Cluster& c = t.clusters[id];
  if (c.is_leaf()) return b.leaf[id];
  const Mat<S>& tr = b.transfer[id];
  if (tr.size() == 0) return Mat<S>(c.size(), 0);
  const Mat<S> m1 = materialize(b, t, c.child[0]);
  const Mat<S> m2 = materialize(b, t, c.child[1]);
  Mat<S> out(c.size(), tr.c);
  out.set_block(0, 0, mul(m1, tr.rows_range(0, m1.c)));
  out.set_block(m1.r, 0, mul(m2, tr.rows_range(m1.c, m2.c)));
  return out;
}

}  // namespace

template <class S>
H2Matrix<S> build_h2(const Mat<S>& dense, std::shared_ptr<const BlockTree> st, double eps_h2) {
  if (!st) throw ConfigError("build_h2: null structure");
  const ClusterTree& t = st->rows();
  if (dense.r != t.size() || dense.c != t.size())
    throw ConfigError("build_h2: dense size does not match the block structure");
  if (!(eps_h2 > 0.0 && eps_h2 < 1.0)) throw ConfigError("build_h2: eps_h2 must be in (0,1)");
  const Mat<S> dt = tree_order(dense, t);
  const auto rf = far_field(*st, true);
  const auto cf = far_field(*st, false);
  Side<S> rows{st->rows(), st->cols(), dt, rf, false, eps_h2, {}, {}};
  rows.build();
  Side<S> cols{st->cols(), st->rows(), dt, cf, true, eps_h2, {}, {}};
  cols.build();
  H2Matrix<S> h;
  h.tree = std::shared_ptr<const ClusterTree>(st, &st->rows());
  h.structure = st;
  h.row_basis = std::move(rows.basis);
  h.col_basis = std::move(cols.basis);
  for (int l = 0; l <= st->depth(); ++l)
    for (const BlockEntry& e : st->level_blocks(l)) {
      const Cluster& a = t.clusters[e.key.row];
      const Cluster& b = t.clusters[e.key.col];
      if (e.kind == BlockKind::admissible) {
        const Mat<S> blk = dt.block(a.begin, b.begin, a.size(), b.size());
        h.coupling[e.key] =
            mul(mul(Op::H, rows.mat[a.id], Op::N, blk), cols.mat[b.id].conjugate());
      } else if (e.kind == BlockKind::inadmissible_leaf) {
        h.full[e.key] = dt.block(a.begin, b.begin, a.size(), b.size());
      }
    }
  return h;
}

template <class S>
Mat<S> materialized_row_basis(const H2Matrix<S>& h, int id) {
  return materialize(h.row_basis, *h.tree, id);
}
template <class S>
Mat<S> materialized_col_basis(const H2Matrix<S>& h, int id) {
  return materialize(h.col_basis, *h.tree, id);
}

// h2_matrix.cpp:183-211
template <class S>
Mat<S> h2_to_dense(const H2Matrix<S>& h) {
  const ClusterTree& t = *h.tree;
  const int n = t.size();
  Mat<S> dt(n, n);
  std::vector<Mat<S>> rm(t.clusters.size()), cm(t.clusters.size());
  for (const auto& [key, s] : h.coupling) {
    if (rm[key.row].size() == 0) rm[key.row] = materialized_row_basis(h, key.row);
    if (cm[key.col].size() == 0) cm[key.col] = materialized_col_basis(h, key.col);
    const Cluster& a = t.clusters[key.row];
    const Cluster& b = t.clusters[key.col];
    dt.add_block(a.begin, b.begin, mul(Op::N, mul(rm[key.row], s), Op::T, cm[key.col]));
  }
  for (const auto& [key, f] : h.full) {
    const Cluster& a = t.clusters[key.row];
    const Cluster& b = t.clusters[key.col];
    dt.add_block(a.begin, b.begin, f);
  }
  Mat<S> out(n, n);
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a) out(t.perm[a], t.perm[b]) = dt(a, b);
  return out;
}

// h2_matrix.cpp:213-278 — forward transform, couplings, backward transform,
// near field.
template <class S>
std::vector<S> mvp(const H2Matrix<S>& h, const std::vector<S>& x) {
  const ClusterTree& t = *h.tree;
  const int n = t.size();
  if (static_cast<int>(x.size()) != n) throw ConfigError("mvp: vector length does not match the matrix");
  auto col = [](const std::vector<S>& v, Index off, Index len) {
    Mat<S> m(len, 1);
    for (Index i = 0; i < len; ++i) m(i, 0) = v[off + i];
    return m;
  };
  std::vector<S> xt(n), yt(n, S(0));
  for (int a = 0; a < n; ++a) xt[a] = x[t.perm[a]];
  std::vector<Mat<S>> xh(t.clusters.size());
  for (int l = t.depth; l >= 1; --l)
    for (int id : t.levels[l]) {
      const Cluster& c = t.clusters[id];
      if (c.is_leaf()) {
        xh[id] = mul(Op::T, h.col_basis.leaf[id], Op::N, col(xt, c.begin, c.size()));
      } else {
        const Mat<S>& tr = h.col_basis.transfer[id];
        const Index k1 = xh[c.child[0]].r;
        xh[id] = mul(Op::T, tr.rows_range(0, k1), Op::N, xh[c.child[0]]);
        gemm(Op::T, Op::N, tr.rows_range(k1, tr.r - k1), xh[c.child[1]], xh[id], true);
      }
    }
  std::vector<Mat<S>> yh(t.clusters.size());
  for (const auto& [key, s] : h.coupling) {
    if (yh[key.row].size() == 0) yh[key.row] = Mat<S>(h.row_basis.rank[key.row], 1);
    gemm(Op::N, Op::N, s, xh[key.col], yh[key.row], true);
  }
  for (int l = 1; l < t.depth; ++l)
    for (int id : t.levels[l]) {
      const Cluster& c = t.clusters[id];
      if (c.is_leaf() || yh[id].size() == 0) continue;
      const Mat<S>& tr = h.row_basis.transfer[id];
      const Index k1 = h.row_basis.rank[c.child[0]];
      if (yh[c.child[0]].size() == 0) yh[c.child[0]] = Mat<S>(k1, 1);
      if (yh[c.child[1]].size() == 0) yh[c.child[1]] = Mat<S>(tr.r - k1, 1);
      gemm(Op::N, Op::N, tr.rows_range(0, k1), yh[id], yh[c.child[0]], true);
      gemm(Op::N, Op::N, tr.rows_range(k1, tr.r - k1), yh[id], yh[c.child[1]], true);
    }
  for (int id : t.levels[t.depth]) {
    if (yh[id].size() == 0) continue;
    const Cluster& c = t.clusters[id];
    const Mat<S> y = mul(h.row_basis.leaf[id], yh[id]);
    for (Index i = 0; i < y.r; ++i) yt[c.begin + i] += y(i, 0);
  }
  for (const auto& [key, f] : h.full) {
    const Cluster& a = t.clusters[key.row];
    const Cluster& b = t.clusters[key.col];
    const Mat<S> y = mul(f, col(xt, b.begin, b.size()));
    for (Index i = 0; i < y.r; ++i) yt[a.begin + i] += y(i, 0);
  }
  std::vector<S> y(n);
  for (int a = 0; a < n; ++a) y[t.perm[a]] = yt[a];
  return y;
}

// h2_matrix.cpp:280-292
template <class S>
std::int64_t memory_footprint(const H2Matrix<S>& h) {
  std::int64_t n = 0;
  for (const auto* b : {&h.row_basis, &h.col_basis}) {
    for (const auto& m : b->leaf) n += m.size();
    for (const auto& m : b->transfer) n += m.size();
  }
  for (const auto& [k, m] : h.coupling) n += m.size();
  for (const auto& [k, m] : h.full) n += m.size();
  return n;
}

// metrics.cpp:11-35
template <>
std::vector<Real> random_vector<Real>(int n, std::uint64_t seed) {
  std::mt19937_64 eng(seed);
  std::vector<Real> x(n);
  for (auto& v : x) v = 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0;
  return x;
}
template <>
std::vector<Complex> random_vector<Complex>(int n, std::uint64_t seed) {
  std::mt19937_64 eng(seed);
  std::vector<Complex> x(n);
  for (auto& v : x) {
    const double re = 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0;
    const double im = 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0;
    v = Complex(re, im);
  }
  return x;
}

// metrics.cpp:37-55
template <class S>
double relative_error(const H2Matrix<S>& a, const H2Matrix<S>& b, const H2Matrix<S>& c,
                      std::uint64_t seed, bool* ref_zero) {
  if (a.size() != b.size() || a.size() != c.size())
    throw ConfigError("relative_error: operand sizes disagree");
  const auto x = random_vector<S>(a.size(), seed);
  const auto ref = mvp(a, mvp(b, x));
  const auto cx = mvp(c, x);
  double rn = 0, dn = 0, cn = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    rn += abs2(ref[i]);
    dn += abs2(cx[i] - ref[i]);
    cn += abs2(cx[i]);
  }
  if (ref_zero) *ref_zero = rn == 0.0;
  return rn == 0.0 ? std::sqrt(cn) : std::sqrt(dn) / std::sqrt(rn);
}

#define H2O_INST(S)                                                                           \
  template H2Matrix<S> build_h2<S>(const Mat<S>&, std::shared_ptr<const BlockTree>, double); \
  template Mat<S> h2_to_dense<S>(const H2Matrix<S>&);                                        \
  template std::vector<S> mvp<S>(const H2Matrix<S>&, const std::vector<S>&);                 \
  template std::int64_t memory_footprint<S>(const H2Matrix<S>&);                             \
  template Mat<S> materialized_row_basis<S>(const H2Matrix<S>&, int);                        \
  template Mat<S> materialized_col_basis<S>(const H2Matrix<S>&, int);                        \
  template double relative_error<S>(const H2Matrix<S>&, const H2Matrix<S>&,                  \
                                    const H2Matrix<S>&, std::uint64_t, bool*);
H2O_INST(Real)
H2O_INST(Complex)

}  // namespace h2o
