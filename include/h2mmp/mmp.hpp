// The MMP entry points of proj/core/include/h2mmp/mmp.hpp:16-74 with the same
// names, types and semantics, executed by the B200 library through the
// C-ABI (include/h2c.h):  mmp(a, b, eps) -> h2c_mmp, formatted_mmp(a, b) ->
// h2c_formatted_mmp.  Errors are re-thrown as the reference's exception types.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "h2mmp/context.hpp"
#include "h2mmp/h2_matrix.hpp"

namespace h2mmp {

struct LevelStats {
  int level = 0;
  Index max_row_rank = 0;
  Index max_col_rank = 0;
  std::array<std::int64_t, 4> case_products{0, 0, 0, 0};
  int max_case1_terms = 0;
  int max_case2_terms = 0;
  int max_case3_terms = 0;
};

struct MmpReport {
  double eps_trunc = 0.0;
  bool adaptive = true;
  std::vector<LevelStats> levels;
  std::int64_t flops = 0;
  std::array<std::int64_t, 4> case_flops{0, 0, 0, 0};
  double wall_seconds = 0.0;
  int pending_after_split = 0;
  // B200 extensions
  std::int64_t flops_exec = 0;
  double device_seconds = 0.0;
  Index max_rank() const {
    Index r = 0;
    for (const auto& s : levels) r = std::max({r, s.max_row_rank, s.max_col_rank});
    return r;
  }
};

template <class Scalar>
struct MmpResult {
  H2Matrix<Scalar> product;
  MmpReport report;
};

namespace detail {

template <class Scalar>
MmpResult<Scalar> run(const H2Matrix<Scalar>& a, const H2Matrix<Scalar>& b, double eps, bool adaptive) {
  // mmp.cpp:58-63 — shared tree and structure objects first, then eps (adaptive only)
  if (a.tree != b.tree || a.structure != b.structure)
    throw ConfigError("mmp: operands must share cluster trees and block structure");
  if (adaptive && !(eps > 0.0 && eps < 1.0)) throw ConfigError("mmp: eps_trunc must be in (0,1)");
  h2c_context* ctx = default_context();
  const Flat<Scalar> fa = flatten(a);
  const Flat<Scalar> fb = (&a == &b) ? Flat<Scalar>{} : flatten(b);
  const h2c_matrix* db = (&a == &b) ? &fa.desc : &fb.desc;
  h2c_result* res = nullptr;
  const int rc = adaptive ? h2c_mmp(ctx, &fa.desc, db, eps, &res) : h2c_formatted_mmp(ctx, &fa.desc, db, &res);
  rethrow(rc, ctx);
  struct Free {
    h2c_result* r;
    ~Free() { h2c_result_free(r); }
  } guard{res};
  h2c_matrix dc;
  h2c_result_matrix(res, &dc);
  h2c_report rp;
  h2c_result_report(res, &rp);
  MmpResult<Scalar> out{unflatten<Scalar>(dc, a.tree, a.structure), {}};  // C shares A's tree (mmp.cpp:25-26)
  MmpReport& r = out.report;
  r.eps_trunc = rp.eps_trunc;
  r.adaptive = rp.adaptive != 0;
  r.flops = rp.flops;
  for (int c = 0; c < 4; ++c) r.case_flops[c] = rp.case_flops[c];
  r.wall_seconds = rp.wall_seconds;
  r.pending_after_split = rp.pending_after_split;
  r.flops_exec = rp.flops_exec;
  r.device_seconds = rp.device_seconds;
  r.levels.resize(rp.n_levels);
  for (int l = 0; l < rp.n_levels; ++l) {
    LevelStats& s = r.levels[l];
    s.level = l;
    s.max_row_rank = rp.max_row_rank[l];
    s.max_col_rank = rp.max_col_rank[l];
    for (int c = 0; c < 4; ++c) s.case_products[c] = rp.case_products[4 * l + c];
    s.max_case1_terms = rp.max_case1_terms[l];
    s.max_case2_terms = rp.max_case2_terms[l];
    s.max_case3_terms = rp.max_case3_terms[l];
  }
  return out;
}

}  // namespace detail

/// mmp.cpp:688-691
template <class Scalar>
MmpResult<Scalar> mmp(const H2Matrix<Scalar>& a, const H2Matrix<Scalar>& b, double eps_trunc) {
  return detail::run(a, b, eps_trunc, true);
}

/// mmp.cpp:716-719
template <class Scalar>
MmpResult<Scalar> formatted_mmp(const H2Matrix<Scalar>& a, const H2Matrix<Scalar>& b) {
  return detail::run(a, b, 0.0, false);
}

/// mmp.cpp:693-714 (host; O(N k^2), not on the device path)
template <class Scalar>
std::vector<DenseMatrix<Scalar>> basis_products(const H2Matrix<Scalar>& a, const H2Matrix<Scalar>& b) {
  if (a.tree != b.tree) throw ConfigError("basis_products: operands must share cluster trees");
  const ClusterTree& t = *a.tree;
  std::vector<DenseMatrix<Scalar>> out(t.clusters.size());
  for (int id : t.levels[t.depth]) out[id] = a.col_basis.leaf[id].transpose() * b.row_basis.leaf[id];
  for (int l = t.depth - 1; l >= 1; --l)
    for (int id : t.levels[l]) {
      const Cluster& c = t.clusters[id];
      const DenseMatrix<Scalar>& ta = a.col_basis.transfer[id];
      const DenseMatrix<Scalar>& tb = b.row_basis.transfer[id];
      const Index ka1 = a.col_basis.rank[c.child[0]], kb1 = b.row_basis.rank[c.child[0]];
      auto rows = [](const DenseMatrix<Scalar>& m, Index r0, Index n) {
        DenseMatrix<Scalar> o(n, m.cols());
        for (Index j = 0; j < m.cols(); ++j)
          for (Index i = 0; i < n; ++i) o(i, j) = m(r0 + i, j);
        return o;
      };
      out[id] = rows(ta, 0, ka1).transpose() * out[c.child[0]] * rows(tb, 0, kb1) +
                rows(ta, ka1, ta.rows() - ka1).transpose() * out[c.child[1]] * rows(tb, kb1, tb.rows() - kb1);
    }
  return out;
}

}  // namespace h2mmp
