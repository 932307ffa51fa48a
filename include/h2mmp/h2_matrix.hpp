// H2Matrix / ClusterBasis of proj/core/include/h2mmp/h2_matrix.hpp:19-79 with
// the same fields, plus the verification helpers of that header
// (h2_to_dense, mvp, memory_footprint, materialized_*_basis; host code, not on
// the product path).  flatten()/unflatten() translate to the C-ABI layout.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <thread>
#include <utility>
#include <vector>

#include "h2mmp/block_tree.hpp"
#include "h2mmp/context.hpp"
#include "h2mmp/truncation.hpp"
#include "h2mmp/dense.hpp"

namespace h2mmp {

template <class Scalar>
struct ClusterBasis {
  std::vector<DenseMatrix<Scalar>> leaf;
  std::vector<DenseMatrix<Scalar>> transfer;
  std::vector<Index> rank;
  std::vector<char> degenerate;
  void resize(std::size_t n) {
    leaf.assign(n, {});
    transfer.assign(n, {});
    rank.assign(n, 0);
    degenerate.assign(n, 0);
  }
};

template <class Scalar>
struct H2Matrix {
  std::shared_ptr<const ClusterTree> tree;
  std::shared_ptr<const BlockTree> structure;
  ClusterBasis<Scalar> row_basis;
  ClusterBasis<Scalar> col_basis;
  std::map<BlockKey, DenseMatrix<Scalar>> coupling;
  std::map<BlockKey, DenseMatrix<Scalar>> full;
  int size() const { return tree ? tree->size() : 0; }
};

namespace detail {

// Flat copy of an H2Matrix in the layout of h2c_types.h (owning buffers).  The values live in one
// uninitialised allocation (no zero fill of several GB) filled by parallel copies.
template <class Scalar>
struct Flat {
  std::vector<int32_t> row_rank, col_rank;
  std::vector<uint8_t> row_dg, col_dg;
  std::vector<int64_t> row_off, col_off, block_off;
  struct FreeDeleter {
    void operator()(void* p) const { std::free(p); }
  };
  std::unique_ptr<Scalar, FreeDeleter> values;
  h2c_matrix desc{};
};

// f(k) for k in [0, n) on the host's hardware threads (contiguous ranges)
template <class F>
void parallel_ranges(int64_t n, F&& f) {
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 64));
  if (nt <= 1) {
    for (int64_t k = 0; k < n; ++k) f(k);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      for (int64_t k = n * w / nt; k < n * (w + 1) / nt; ++k) f(k);
    });
  for (auto& x : th) x.join();
}

template <class Scalar>
Flat<Scalar> flatten(const H2Matrix<Scalar>& h) {
  const ClusterTree& t = *h.tree;
  const BlockTree& bt = *h.structure;
  const int nc = static_cast<int>(t.clusters.size());
  Flat<Scalar> f;
  // pass 1: offsets and sources; pass 2: parallel copies into one allocation
  std::vector<std::pair<const DenseMatrix<Scalar>*, int64_t>> jobs;
  int64_t n = 0;
  auto add = [&](const DenseMatrix<Scalar>& m) {
    const int64_t at = n;
    jobs.emplace_back(&m, at);
    n += m.size();
    return at;
  };
  for (int side = 0; side < 2; ++side) {
    const ClusterBasis<Scalar>& b = side == 0 ? h.row_basis : h.col_basis;
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
  const h2c_blocks& d = bt.desc;
  f.block_off.assign(d.n_blocks, -1);
  for (int64_t k = 0; k < d.n_blocks; ++k) {
    const BlockKey key{d.row[k], d.col[k]};
    if (d.kind[k] == H2C_ADMISSIBLE) f.block_off[k] = add(h.coupling.at(key));
    else if (d.kind[k] == H2C_INADMISSIBLE_LEAF) f.block_off[k] = add(h.full.at(key));
  }
  f.values.reset(static_cast<Scalar*>(std::malloc(std::max<size_t>(1, sizeof(Scalar) * static_cast<size_t>(n)))));
  if (!f.values) throw std::bad_alloc();
  Scalar* dst = f.values.get();
  parallel_ranges(static_cast<int64_t>(jobs.size()), [&](int64_t k) {
    const DenseMatrix<Scalar>& m = *jobs[k].first;
    if (m.size()) std::memcpy(static_cast<void*>(dst + jobs[k].second), m.data(), sizeof(Scalar) * m.size());
  });
  f.desc = h2c_matrix{&t.desc, &bt.desc, is_complex_v<Scalar> ? H2C_COMPLEX : H2C_REAL, f.row_rank.data(),
                      f.col_rank.data(), f.row_dg.data(), f.col_dg.data(), f.row_off.data(), f.col_off.data(),
                      f.block_off.data(), reinterpret_cast<const double*>(dst), n};
  return f;
}

template <class Scalar>
DenseMatrix<Scalar> read(const h2c_matrix& d, int64_t off, Index r, Index c) {
  DenseMatrix<Scalar> m(r, c);
  if (r * c) std::memcpy(static_cast<void*>(m.data()), reinterpret_cast<const Scalar*>(d.values) + off, sizeof(Scalar) * r * c);
  return m;
}

template <class Scalar>
H2Matrix<Scalar> unflatten(const h2c_matrix& d, std::shared_ptr<const ClusterTree> tree,
                           std::shared_ptr<const BlockTree> structure) {
  H2Matrix<Scalar> h;
  h.tree = std::move(tree);
  h.structure = std::move(structure);
  const ClusterTree& t = *h.tree;
  const int nc = static_cast<int>(t.clusters.size());
  // pass 1 (serial): the containers and the (destination, offset, shape) of every matrix;
  // pass 2 (parallel): allocate and copy
  struct Job {
    DenseMatrix<Scalar>* dst;
    int64_t off;
    Index r, c;
  };
  std::vector<Job> jobs;
  for (int side = 0; side < 2; ++side) {
    ClusterBasis<Scalar>& b = side == 0 ? h.row_basis : h.col_basis;
    const int32_t* rk = side == 0 ? d.row_rank : d.col_rank;
    const uint8_t* dg = side == 0 ? d.row_degenerate : d.col_degenerate;
    const int64_t* off = side == 0 ? d.row_offset : d.col_offset;
    b.resize(nc);
    for (int c = 0; c < nc; ++c) {
      b.rank[c] = rk[c];
      b.degenerate[c] = dg[c];
      const Cluster& cl = t.clusters[c];
      if (off[c] < 0) continue;
      if (cl.is_leaf()) jobs.push_back({&b.leaf[c], off[c], cl.size(), rk[c]});
      else jobs.push_back({&b.transfer[c], off[c], rk[cl.child[0]] + rk[cl.child[1]], rk[c]});
    }
  }
  const h2c_blocks& bd = h.structure->desc;
  for (int64_t k = 0; k < bd.n_blocks; ++k) {
    const BlockKey key{bd.row[k], bd.col[k]};
    if (bd.kind[k] == H2C_ADMISSIBLE)
      jobs.push_back({&h.coupling[key], d.block_offset[k], d.row_rank[key.row], d.col_rank[key.col]});
    else if (bd.kind[k] == H2C_INADMISSIBLE_LEAF)
      jobs.push_back({&h.full[key], d.block_offset[k], t.clusters[key.row].size(), t.clusters[key.col].size()});
  }
  parallel_ranges(static_cast<int64_t>(jobs.size()), [&](int64_t k) {
    const Job& j = jobs[k];
    *j.dst = read<Scalar>(d, j.off, j.r, j.c);
  });
  return h;
}

template <class Scalar>
DenseMatrix<Scalar> materialize(const ClusterBasis<Scalar>& b, const ClusterTree& t, int c) {
  const Cluster& cl = t.clusters[c];
  if (cl.is_leaf()) return b.leaf[c];
  const DenseMatrix<Scalar>& tr = b.transfer[c];
  if (tr.size() == 0) return DenseMatrix<Scalar>(cl.size(), 0);
  const DenseMatrix<Scalar> m1 = materialize(b, t, cl.child[0]);
  const DenseMatrix<Scalar> m2 = materialize(b, t, cl.child[1]);
  DenseMatrix<Scalar> out(cl.size(), tr.cols());
  for (Index j = 0; j < tr.cols(); ++j) {
    for (Index i = 0; i < m1.rows(); ++i)
      for (Index k = 0; k < m1.cols(); ++k) out(i, j) += m1(i, k) * tr(k, j);
    for (Index i = 0; i < m2.rows(); ++i)
      for (Index k = 0; k < m2.cols(); ++k) out(m1.rows() + i, j) += m2(i, k) * tr(m1.cols() + k, j);
  }
  return out;
}

}  // namespace detail

/// h2_matrix.cpp:294-302
template <class Scalar>
DenseMatrix<Scalar> materialized_row_basis(const H2Matrix<Scalar>& h, int c) {
  return detail::materialize(h.row_basis, *h.tree, c);
}
template <class Scalar>
DenseMatrix<Scalar> materialized_col_basis(const H2Matrix<Scalar>& h, int c) {
  return detail::materialize(h.col_basis, *h.tree, c);
}

/// h2_matrix.cpp:280-292
template <class Scalar>
std::int64_t memory_footprint(const H2Matrix<Scalar>& h) {
  std::int64_t n = 0;
  for (const auto* b : {&h.row_basis, &h.col_basis}) {
    for (const auto& m : b->leaf) n += m.size();
    for (const auto& m : b->transfer) n += m.size();
  }
  for (const auto& [k, m] : h.coupling) n += m.size();
  for (const auto& [k, m] : h.full) n += m.size();
  return n;
}

/// h2_matrix.cpp:183-211 (original ordering; small N only)
template <class Scalar>
DenseMatrix<Scalar> h2_to_dense(const H2Matrix<Scalar>& h) {
  const ClusterTree& t = *h.tree;
  const int n = t.size();
  DenseMatrix<Scalar> dt(n, n);
  for (const auto& [key, s] : h.coupling) {
    const DenseMatrix<Scalar> blk = materialized_row_basis(h, key.row) * s * materialized_col_basis(h, key.col).transpose();
    const Cluster& a = t.clusters[key.row];
    const Cluster& b = t.clusters[key.col];
    for (Index j = 0; j < blk.cols(); ++j)
      for (Index i = 0; i < blk.rows(); ++i) dt(a.begin + i, b.begin + j) += blk(i, j);
  }
  for (const auto& [key, f] : h.full) {
    const Cluster& a = t.clusters[key.row];
    const Cluster& b = t.clusters[key.col];
    for (Index j = 0; j < f.cols(); ++j)
      for (Index i = 0; i < f.rows(); ++i) dt(a.begin + i, b.begin + j) += f(i, j);
  }
  DenseMatrix<Scalar> out(n, n);
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a) out(t.perm[a], t.perm[b]) = dt(a, b);
  return out;
}

/// h2_matrix.cpp:213-278: exact H^2 matrix-vector product (forward transform, coupling
/// products, backward transform, near field), on the B200 (h2c_mvp), original ordering.
template <class Scalar>
DenseVector<Scalar> mvp(const H2Matrix<Scalar>& h, const DenseVector<Scalar>& x) {
  const int n = h.tree->size();
  if (x.rows() != n || x.cols() != 1) throw ConfigError("mvp: vector length must match the matrix");
  const detail::Flat<Scalar> f = detail::flatten(h);
  DenseVector<Scalar> y(n, 1);
  h2c_context* ctx = detail::default_context();
  detail::rethrow(h2c_mvp(ctx, &f.desc, reinterpret_cast<const double*>(x.data()), 1, reinterpret_cast<double*>(y.data())),
                  ctx);
  return y;
}

}  // namespace h2mmp
