// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// Flat C-ABI over the oracle (oracle/h2o.h): converts the shared descriptors of
// include/h2c_types.h to the reference-shaped C++ model and back.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "h2o.h"
#include "linalg.hpp"
#include "model.hpp"

using namespace h2o;

namespace {
thread_local std::string g_err;
int g_mmp_threads = 1;  // h2o_set_mmp_threads

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return H2C_OK;
  } catch (const ConfigError& e) {
    return fail(e, H2C_ERR_CONFIG);
  } catch (const InvariantError& e) {
    return fail(e, H2C_ERR_INVARIANT);
  } catch (const std::exception& e) {
    return fail(e, H2C_ERR_INVARIANT);
  }
}

GeometrySpec spec_of(int family, uint64_t seed, int n, int bus_count, int spm, int sw, int st,
                     int ae, int cp) {
  GeometrySpec g;
  g.family = static_cast<Family>(family);
  g.seed = seed;
  g.n = n;
  g.bus_count = bus_count;
  g.samples_per_meter = spm;
  g.slab_width = sw;
  g.slab_thickness = st;
  g.array_edge = ae;
  g.cube_points = cp;
  return g;
}

// ---- flat <-> model ---------------------------------------------------------
std::shared_ptr<ClusterTree> tree_from(const h2c_tree& d) {
  auto t = std::make_shared<ClusterTree>();
  t->depth = d.depth;
  t->leafsize = d.leafsize;
  t->clusters.resize(d.n_clusters);
  for (int i = 0; i < d.n_clusters; ++i) {
    Cluster& c = t->clusters[i];
    c.id = i;
    c.parent = d.parent[i];
    c.level = d.level[i];
    c.begin = d.begin[i];
    c.end = d.end[i];
    c.child = {d.child0[i], d.child1[i]};
    if (d.bbox) {
      c.bbox_min = {d.bbox[6 * i], d.bbox[6 * i + 1], d.bbox[6 * i + 2]};
      c.bbox_max = {d.bbox[6 * i + 3], d.bbox[6 * i + 4], d.bbox[6 * i + 5]};
    }
  }
  t->perm.assign(d.perm, d.perm + d.n_points);
  t->inv_perm.resize(d.n_points);
  for (int i = 0; i < d.n_points; ++i) t->inv_perm[t->perm[i]] = i;
  t->levels.assign(d.depth + 1, {});
  for (const Cluster& c : t->clusters) t->levels[c.level].push_back(c.id);
  for (auto& lv : t->levels)
    std::sort(lv.begin(), lv.end(),
              [&](int a, int b) { return t->clusters[a].begin < t->clusters[b].begin; });
  return t;
}

std::shared_ptr<BlockTree> blocks_from(std::shared_ptr<const ClusterTree> t, const h2c_blocks& d) {
  std::vector<std::vector<BlockEntry>> lv(d.depth + 1);
  for (int l = 0; l <= d.depth; ++l)
    for (int64_t b = d.level_ptr[l]; b < d.level_ptr[l + 1]; ++b)
      lv[l].push_back({BlockKey{d.row[b], d.col[b]}, static_cast<BlockKind>(d.kind[b])});
  return std::make_shared<BlockTree>(t, d.eta, std::move(lv));
}

struct Converted {
  std::shared_ptr<ClusterTree> tree;
  std::shared_ptr<BlockTree> blocks;
};
Converted convert_structure(const h2c_tree* t, const h2c_blocks* b) {
  Converted c;
  c.tree = tree_from(*t);
  c.blocks = blocks_from(c.tree, *b);
  return c;
}

template <class S>
Mat<S> read_mat(const h2c_matrix& d, int64_t off, Index r, Index c) {
  Mat<S> m(r, c);
  if (r * c == 0) return m;
  if (off < 0 || off + r * c > d.n_values) throw ConfigError("matrix descriptor offset out of range");
  std::memcpy(static_cast<void*>(m.data()), d.values + (is_complex_v<S> ? 2 : 1) * off, sizeof(S) * r * c);
  return m;
}

template <class S>
H2Matrix<S> matrix_from(const h2c_matrix& d, const Converted& cs) {
  const ClusterTree& t = *cs.tree;
  H2Matrix<S> h;
  h.tree = cs.tree;
  h.structure = cs.blocks;
  const int nc = static_cast<int>(t.clusters.size());
  for (int side = 0; side < 2; ++side) {
    ClusterBasis<S>& cb = side == 0 ? h.row_basis : h.col_basis;
    const int32_t* rank = side == 0 ? d.row_rank : d.col_rank;
    const uint8_t* dg = side == 0 ? d.row_degenerate : d.col_degenerate;
    const int64_t* off = side == 0 ? d.row_offset : d.col_offset;
    cb.resize(nc);
    for (int i = 0; i < nc; ++i) {
      const Cluster& c = t.clusters[i];
      cb.rank[i] = rank[i];
      cb.degenerate[i] = dg ? dg[i] : 0;
      if (c.parent < 0 && !c.is_leaf()) continue;  // a non-leaf root carries no basis
      if (c.is_leaf()) cb.leaf[i] = read_mat<S>(d, off[i], c.size(), rank[i]);
      else cb.transfer[i] = read_mat<S>(d, off[i], rank[c.child[0]] + rank[c.child[1]], rank[i]);
    }
  }
  const h2c_blocks& b = *d.blocks;
  for (int64_t k = 0; k < b.n_blocks; ++k) {
    const BlockKey key{b.row[k], b.col[k]};
    if (b.kind[k] == H2C_ADMISSIBLE)
      h.coupling[key] = read_mat<S>(d, d.block_offset[k], d.row_rank[key.row], d.col_rank[key.col]);
    else if (b.kind[k] == H2C_INADMISSIBLE_LEAF)
      h.full[key] = read_mat<S>(d, d.block_offset[k], t.clusters[key.row].size(),
                                t.clusters[key.col].size());
  }
  return h;
}

}  // namespace

// ---- owned flat objects -------------------------------------------------------
struct h2o_tree {
  std::vector<int32_t> parent, child0, child1, level, begin, end, perm;
  std::vector<double> bbox;
  int32_t n_points = 0, depth = 0, leafsize = 0;
};
struct h2o_blocks {
  std::vector<int64_t> level_ptr;
  std::vector<int32_t> row, col;
  std::vector<uint8_t> kind;
  int32_t depth = 0, c_sp = 0;
  double eta = 0;
};
struct h2o_matrix {
  const h2c_tree* tree = nullptr;
  const h2c_blocks* blocks = nullptr;
  int32_t scalar = 0;
  std::vector<int32_t> row_rank, col_rank;
  std::vector<uint8_t> row_dg, col_dg;
  std::vector<int64_t> row_off, col_off, block_off;
  std::vector<double> values;
};
struct h2o_result {
  h2o_matrix m;
  MmpReport rep;
  std::vector<int64_t> max_row, max_col, case_products;
  std::vector<int32_t> t1, t2, t3;
};

namespace {
template <class S>
void matrix_to(const H2Matrix<S>& h, const h2c_tree* td, const h2c_blocks* bd, h2o_matrix& out) {
  const ClusterTree& t = *h.tree;
  const int nc = static_cast<int>(t.clusters.size());
  out.tree = td;
  out.blocks = bd;
  out.scalar = is_complex_v<S> ? H2C_COMPLEX : H2C_REAL;
  const int w = is_complex_v<S> ? 2 : 1;
  int64_t n = 0;
  auto push = [&](const Mat<S>& m) {
    const int64_t at = n;
    out.values.resize(static_cast<size_t>(w * (n + m.size())));
    if (m.size()) std::memcpy(out.values.data() + w * n, m.data(), sizeof(S) * m.size());
    n += m.size();
    return at;
  };
  for (int side = 0; side < 2; ++side) {
    const ClusterBasis<S>& cb = side == 0 ? h.row_basis : h.col_basis;
    auto& rank = side == 0 ? out.row_rank : out.col_rank;
    auto& dg = side == 0 ? out.row_dg : out.col_dg;
    auto& off = side == 0 ? out.row_off : out.col_off;
    rank.resize(nc);
    dg.resize(nc);
    off.assign(nc, -1);
    for (int i = 0; i < nc; ++i) {
      rank[i] = static_cast<int32_t>(cb.rank[i]);
      dg[i] = cb.degenerate[i] ? 1 : 0;
      if (t.clusters[i].parent < 0 && !t.clusters[i].is_leaf()) continue;
      off[i] = push(t.clusters[i].is_leaf() ? cb.leaf[i] : cb.transfer[i]);
    }
  }
  out.block_off.assign(bd->n_blocks, -1);
  for (int64_t k = 0; k < bd->n_blocks; ++k) {
    const BlockKey key{bd->row[k], bd->col[k]};
    if (bd->kind[k] == H2C_ADMISSIBLE) out.block_off[k] = push(h.coupling.at(key));
    else if (bd->kind[k] == H2C_INADMISSIBLE_LEAF) out.block_off[k] = push(h.full.at(key));
  }
}

void fill_desc(const h2o_matrix& m, h2c_matrix* d) {
  d->tree = m.tree;
  d->blocks = m.blocks;
  d->scalar = m.scalar;
  d->row_rank = m.row_rank.data();
  d->col_rank = m.col_rank.data();
  d->row_degenerate = m.row_dg.data();
  d->col_degenerate = m.col_dg.data();
  d->row_offset = m.row_off.data();
  d->col_offset = m.col_off.data();
  d->block_offset = m.block_off.data();
  d->values = m.values.data();
  d->n_values = static_cast<int64_t>(m.values.size()) / (m.scalar == H2C_COMPLEX ? 2 : 1);
}
}  // namespace

// (C linkage comes from the declarations in h2o.h)

const char* h2o_last_error(void) { return g_err.c_str(); }
void h2o_set_threads(int n) { set_blas_threads(n); }
void h2o_set_mmp_threads(int n) { g_mmp_threads = n < 1 ? 1 : n; }

int64_t h2o_geometry_count(int family, uint64_t seed, int n, int bc, int spm, int sw, int st, int ae,
                           int cp) {
  try {
    return generate_geometry(spec_of(family, seed, n, bc, spm, sw, st, ae, cp)).size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int h2o_geometry_fill(int family, uint64_t seed, int n, int bc, int spm, int sw, int st, int ae,
                      int cp, double* xyz) {
  return guarded([&] {
    const PointSet p = generate_geometry(spec_of(family, seed, n, bc, spm, sw, st, ae, cp));
    for (int i = 0; i < p.size(); ++i) {
      xyz[3 * i] = p.points[i].x;
      xyz[3 * i + 1] = p.points[i].y;
      xyz[3 * i + 2] = p.points[i].z;
    }
  });
}

int h2o_assemble_dense(const double* xyz, int n, int kind, double k, int has_diag, double diag,
                       double* out) {
  return guarded([&] {
    PointSet p;
    for (int i = 0; i < n; ++i) p.points.push_back({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
    Kernel ker;
    ker.kind = static_cast<KernelKind>(kind);
    ker.wavenumber = k;
    if (has_diag) ker.diagonal_value = diag;
    if (kind == 0) {
      const Mat<Real> m = assemble_dense<Real>(p, ker);
      std::memcpy(out, m.data(), sizeof(double) * m.size());
    } else {
      const Mat<Complex> m = assemble_dense<Complex>(p, ker);
      std::memcpy(out, m.data(), sizeof(Complex) * m.size());
    }
  });
}

h2o_tree* h2o_build_tree(const double* xyz, int n, int leafsize) {
  try {
    PointSet p;
    for (int i = 0; i < n; ++i) p.points.push_back({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
    const ClusterTree t = build_cluster_tree(p, leafsize);
    auto* o = new h2o_tree;
    o->n_points = n;
    o->depth = t.depth;
    o->leafsize = leafsize;
    for (const Cluster& c : t.clusters) {
      o->parent.push_back(c.parent);
      o->child0.push_back(c.child[0]);
      o->child1.push_back(c.child[1]);
      o->level.push_back(c.level);
      o->begin.push_back(c.begin);
      o->end.push_back(c.end);
      for (int a = 0; a < 3; ++a) o->bbox.push_back(c.bbox_min[a]);
      for (int a = 0; a < 3; ++a) o->bbox.push_back(c.bbox_max[a]);
    }
    o->perm.assign(t.perm.begin(), t.perm.end());
    return o;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void h2o_tree_desc(const h2o_tree* t, h2c_tree* d) {
  d->n_points = t->n_points;
  d->depth = t->depth;
  d->leafsize = t->leafsize;
  d->n_clusters = static_cast<int32_t>(t->parent.size());
  d->parent = t->parent.data();
  d->child0 = t->child0.data();
  d->child1 = t->child1.data();
  d->level = t->level.data();
  d->begin = t->begin.data();
  d->end = t->end.data();
  d->bbox = t->bbox.data();
  d->perm = t->perm.data();
}
void h2o_tree_free(h2o_tree* t) { delete t; }

h2o_blocks* h2o_build_blocks(const h2c_tree* td, double eta) {
  try {
    std::shared_ptr<const ClusterTree> t = tree_from(*td);
    const BlockTree bt(t, t, eta);
    auto* o = new h2o_blocks;
    o->depth = bt.depth();
    o->c_sp = bt.c_sp();
    o->eta = eta;
    o->level_ptr.push_back(0);
    for (int l = 0; l <= bt.depth(); ++l) {
      for (const BlockEntry& e : bt.level_blocks(l)) {
        o->row.push_back(e.key.row);
        o->col.push_back(e.key.col);
        o->kind.push_back(static_cast<uint8_t>(e.kind));
      }
      o->level_ptr.push_back(static_cast<int64_t>(o->row.size()));
    }
    return o;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void h2o_blocks_desc(const h2o_blocks* b, h2c_blocks* d) {
  d->depth = b->depth;
  d->c_sp = b->c_sp;
  d->eta = b->eta;
  d->n_blocks = static_cast<int64_t>(b->row.size());
  d->level_ptr = b->level_ptr.data();
  d->row = b->row.data();
  d->col = b->col.data();
  d->kind = b->kind.data();
}
void h2o_blocks_free(h2o_blocks* b) { delete b; }

int h2o_target_status(const h2c_tree* td, const h2c_blocks* bd, int t, int s) {
  try {
    const Converted c = convert_structure(td, bd);
    return static_cast<int>(c.blocks->target_status(t, s));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

h2o_matrix* h2o_build_h2(const h2c_tree* td, const h2c_blocks* bd, int scalar, const double* dense,
                         double eps) {
  try {
    const Converted cs = convert_structure(td, bd);
    const int n = td->n_points;
    auto* o = new h2o_matrix;
    if (scalar == H2C_REAL) {
      Mat<Real> d(n, n);
      std::memcpy(static_cast<void*>(d.data()), dense, sizeof(double) * n * n);
      H2Matrix<Real> h = build_h2<Real>(d, cs.blocks, eps);
      h.tree = cs.tree;
      matrix_to(h, td, bd, *o);
    } else {
      Mat<Complex> d(n, n);
      std::memcpy(static_cast<void*>(d.data()), dense, sizeof(Complex) * n * n);
      H2Matrix<Complex> h = build_h2<Complex>(d, cs.blocks, eps);
      h.tree = cs.tree;
      matrix_to(h, td, bd, *o);
    }
    return o;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void h2o_matrix_desc(const h2o_matrix* m, h2c_matrix* d) { fill_desc(*m, d); }
void h2o_matrix_free(h2o_matrix* m) { delete m; }

int h2o_truncate_gram(int scalar, const double* gram, int n, double eps, double* basis, int* rank,
                      int* degenerate) {
  return guarded([&] {
    if (n < 1) throw ConfigError("svd_truncate_gram: gram matrix must be square and non-empty");
    if (scalar == H2C_REAL) {
      Mat<Real> g(n, n);
      std::memcpy(static_cast<void*>(g.data()), gram, sizeof(double) * n * n);
      const auto t = svd_truncate_gram<Real>(g, eps);
      std::memcpy(basis, t.basis.data(), sizeof(double) * t.basis.size());
      *rank = static_cast<int>(t.basis.c);
      *degenerate = t.degenerate;
    } else {
      Mat<Complex> g(n, n);
      std::memcpy(static_cast<void*>(g.data()), gram, sizeof(Complex) * n * n);
      const auto t = svd_truncate_gram<Complex>(g, eps);
      std::memcpy(basis, t.basis.data(), sizeof(Complex) * t.basis.size());
      *rank = static_cast<int>(t.basis.c);
      *degenerate = t.degenerate;
    }
  });
}

namespace {
template <class S>
void run_mmp(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive, int64_t cache,
             h2o_result* r) {
  const Converted cs = convert_structure(a->tree, a->blocks);
  const H2Matrix<S> ha = matrix_from<S>(*a, cs);
  const H2Matrix<S> hb = matrix_from<S>(*b, cs);
  MmpOptions opt;
  opt.ff_cache_bytes = cache;
  opt.threads = g_mmp_threads;
  MmpResult<S> res = adaptive ? mmp<S>(ha, hb, eps, opt) : formatted_mmp<S>(ha, hb, opt);
  matrix_to(res.product, a->tree, a->blocks, r->m);
  r->rep = res.report;
}
}  // namespace

int h2o_mmp(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive, int64_t cache,
            h2o_result** out) {
  *out = nullptr;
  auto* r = new h2o_result;
  const int rc = guarded([&] {
    // mmp.cpp:58-63: pointer identity of the shared tree and structure
    if (a->tree != b->tree || a->blocks != b->blocks)
      throw ConfigError("mmp: operands must share cluster trees and block structure");
    if (a->scalar != b->scalar) throw ConfigError("mmp: operands must share the scalar type");
    if (adaptive && !(eps > 0.0 && eps < 1.0)) throw ConfigError("mmp: eps_trunc must be in (0,1)");
    if (a->scalar == H2C_REAL) run_mmp<Real>(a, b, eps, adaptive, cache, r);
    else run_mmp<Complex>(a, b, eps, adaptive, cache, r);
    for (const LevelStats& s : r->rep.levels) {
      r->max_row.push_back(s.max_row_rank);
      r->max_col.push_back(s.max_col_rank);
      for (int c = 0; c < 4; ++c) r->case_products.push_back(s.case_products[c]);
      r->t1.push_back(s.max_case1_terms);
      r->t2.push_back(s.max_case2_terms);
      r->t3.push_back(s.max_case3_terms);
    }
  });
  if (rc != H2C_OK) {
    delete r;
    return rc;
  }
  *out = r;
  return rc;
}

void h2o_result_matrix(const h2o_result* r, h2c_matrix* d) { fill_desc(r->m, d); }
void h2o_result_report(const h2o_result* r, h2c_report* d) {
  std::memset(d, 0, sizeof(*d));
  d->eps_trunc = r->rep.eps_trunc;
  d->adaptive = r->rep.adaptive;
  d->n_levels = static_cast<int32_t>(r->rep.levels.size());
  d->flops = r->rep.flops;
  for (int c = 0; c < 4; ++c) d->case_flops[c] = r->rep.case_flops[c];
  d->wall_seconds = r->rep.wall_seconds;
  d->pending_after_split = r->rep.pending_after_split;
  d->max_row_rank = r->max_row.data();
  d->max_col_rank = r->max_col.data();
  d->case_products = r->case_products.data();
  d->max_case1_terms = r->t1.data();
  d->max_case2_terms = r->t2.data();
  d->max_case3_terms = r->t3.data();
}
double h2o_result_min_margin(const h2o_result* r) { return r->rep.min_threshold_margin; }
void h2o_result_free(h2o_result* r) { delete r; }

namespace {
template <class S>
int64_t bp_impl(const h2c_matrix* a, const h2c_matrix* b, int64_t* offs, int32_t* rows,
                int32_t* cols, double* vals, int64_t cap) {
  const Converted cs = convert_structure(a->tree, a->blocks);
  const H2Matrix<S> ha = matrix_from<S>(*a, cs);
  const H2Matrix<S> hb = matrix_from<S>(*b, cs);
  const auto bp = basis_products<S>(ha, hb);
  int64_t n = 0;
  for (const auto& m : bp) n += m.size();
  if (cap < n) return n;
  int64_t at = 0;
  const int w = is_complex_v<S> ? 2 : 1;
  for (size_t i = 0; i < bp.size(); ++i) {
    offs[i] = at;
    rows[i] = static_cast<int32_t>(bp[i].r);
    cols[i] = static_cast<int32_t>(bp[i].c);
    if (bp[i].size()) std::memcpy(vals + w * at, bp[i].data(), sizeof(S) * bp[i].size());
    at += bp[i].size();
  }
  return n;
}
template <class S>
std::vector<S> vec_in(const double* x, int n) {
  std::vector<S> v(n);
  std::memcpy(static_cast<void*>(v.data()), x, sizeof(S) * n);
  return v;
}
}  // namespace

int64_t h2o_basis_products(const h2c_matrix* a, const h2c_matrix* b, int64_t* offs, int32_t* rows,
                           int32_t* cols, double* vals, int64_t cap) {
  try {
    if (a->tree != b->tree) throw ConfigError("basis_products: operands must share cluster trees");
    return a->scalar == H2C_REAL ? bp_impl<Real>(a, b, offs, rows, cols, vals, cap)
                                 : bp_impl<Complex>(a, b, offs, rows, cols, vals, cap);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int h2o_h2_to_dense(const h2c_matrix* m, double* out) {
  return guarded([&] {
    const Converted cs = convert_structure(m->tree, m->blocks);
    if (m->scalar == H2C_REAL) {
      const Mat<Real> d = h2_to_dense(matrix_from<Real>(*m, cs));
      std::memcpy(out, d.data(), sizeof(double) * d.size());
    } else {
      const Mat<Complex> d = h2_to_dense(matrix_from<Complex>(*m, cs));
      std::memcpy(out, d.data(), sizeof(Complex) * d.size());
    }
  });
}

int h2o_mvp(const h2c_matrix* m, const double* x, double* y) {
  return guarded([&] {
    const Converted cs = convert_structure(m->tree, m->blocks);
    const int n = m->tree->n_points;
    if (m->scalar == H2C_REAL) {
      const auto r = mvp(matrix_from<Real>(*m, cs), vec_in<Real>(x, n));
      std::memcpy(y, r.data(), sizeof(double) * n);
    } else {
      const auto r = mvp(matrix_from<Complex>(*m, cs), vec_in<Complex>(x, n));
      std::memcpy(y, r.data(), sizeof(Complex) * n);
    }
  });
}

int64_t h2o_memory_footprint(const h2c_matrix* m) {
  try {
    const Converted cs = convert_structure(m->tree, m->blocks);
    return m->scalar == H2C_REAL ? memory_footprint(matrix_from<Real>(*m, cs))
                                 : memory_footprint(matrix_from<Complex>(*m, cs));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int h2o_random_vector(int n, uint64_t seed, int scalar, double* out) {
  return guarded([&] {
    if (scalar == H2C_REAL) {
      const auto v = random_vector<Real>(n, seed);
      std::memcpy(out, v.data(), sizeof(double) * n);
    } else {
      const auto v = random_vector<Complex>(n, seed);
      std::memcpy(out, v.data(), sizeof(Complex) * n);
    }
  });
}

int h2o_relative_error(const h2c_matrix* a, const h2c_matrix* b, const h2c_matrix* c, uint64_t seed,
                       double* value, int* ref_zero) {
  return guarded([&] {
    bool z = false;
    if (a->tree != b->tree || a->tree != c->tree)
      throw ConfigError("relative_error: operands must share the cluster tree");
    const Converted cs = convert_structure(a->tree, a->blocks);
    if (a->scalar == H2C_REAL)
      *value = relative_error(matrix_from<Real>(*a, cs), matrix_from<Real>(*b, cs),
                              matrix_from<Real>(*c, cs), seed, &z);
    else
      *value = relative_error(matrix_from<Complex>(*a, cs), matrix_from<Complex>(*b, cs),
                              matrix_from<Complex>(*c, cs), seed, &z);
    if (ref_zero) *ref_zero = z;
  });
}


// ---- multi-vector exact MVP (one conversion for nv vectors) -------------------
int h2o_mvp_multi(const h2c_matrix* m, const double* x, int nv, double* y) {
  // one conversion, the nv independent MVPs on the mmp thread count (h2o_set_mmp_threads)
  return guarded([&] {
    const Converted cs = convert_structure(m->tree, m->blocks);
    const int n = m->tree->n_points;
    auto run = [&](auto tag) {
      using S = decltype(tag);
      const int w = is_complex_v<S> ? 2 : 1;
      const H2Matrix<S> h = matrix_from<S>(*m, cs);
      std::atomic<int> next{0};
      std::vector<std::thread> th;
      for (int t = 0; t < std::max(1, std::min(g_mmp_threads, nv)); ++t)
        th.emplace_back([&] {
          for (int v; (v = next.fetch_add(1)) < nv;) {
            const auto r = mvp(h, vec_in<S>(x + w * size_t(v) * n, n));
            std::memcpy(y + w * size_t(v) * n, r.data(), sizeof(S) * n);
          }
        });
      for (auto& t : th) t.join();
    };
    if (m->scalar == H2C_REAL) run(Real{});
    else run(Complex{});
  });
}

// ---- sliced all-cores product (bench.py CPU baseline) ----------------------
// One engine thread runs complete products back to back (mmp with
// MmpOptions::threads); its slice points block once the granted slice time has
// elapsed, so the caller measures consecutive slices of the very same product.
namespace {
struct Stopped {};
struct SlicedBase {
  virtual ~SlicedBase() = default;
  std::mutex mu;
  std::condition_variable cv;
  bool paused = true, stop = false, failed = false;
  double slice_s = 0;
  std::chrono::steady_clock::time_point slice_t0;
  int64_t macs_now = 0, products = 0;
  std::string err;
  std::thread th;
  void gate(int64_t macs) {
    std::unique_lock<std::mutex> lk(mu);
    macs_now = macs;
    if (stop) throw Stopped{};
    if (paused || std::chrono::duration<double>(std::chrono::steady_clock::now() - slice_t0).count() >= slice_s) {
      paused = true;
      cv.notify_all();
      cv.wait(lk, [&] { return !paused || stop; });
      if (stop) throw Stopped{};
    }
  }
};
template <class S>
struct Sliced : SlicedBase {
  Converted cs;
  H2Matrix<S> a, b;
  bool same = false;
  double eps = 0;
  int adaptive = 1, threads = 1;
  void loop() {
    try {
      gate(0);  // wait for the first slice
      int64_t base = 0;
      for (;;) {
        MmpOptions opt;
        opt.threads = threads;
        opt.gate = [this, &base](int64_t c) { gate(base + c); };
        const H2Matrix<S>& bb = same ? a : b;
        const int64_t f = adaptive ? mmp<S>(a, bb, eps, opt).report.flops : formatted_mmp<S>(a, bb, opt).report.flops;
        base += f;
        std::lock_guard<std::mutex> g(mu);
        ++products;
      }
    } catch (const Stopped&) {
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> g(mu);
      err = e.what();
      failed = true;
      paused = true;
      cv.notify_all();
    }
  }
};
}  // namespace

struct h2o_sliced {
  std::unique_ptr<SlicedBase> s;
};

h2o_sliced* h2o_sliced_start(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive, int threads) {
  try {
    if (a->tree != b->tree || a->blocks != b->blocks)
      throw ConfigError("mmp: operands must share cluster trees and block structure");
    auto* h = new h2o_sliced;
    auto start = [&](auto* x) {
      using T = std::remove_pointer_t<decltype(x)>;
      using S = std::remove_reference_t<decltype(x->a.row_basis.leaf[0](0, 0))>;
      x->cs = convert_structure(a->tree, a->blocks);
      x->a = matrix_from<S>(*a, x->cs);
      x->same = a == b || (a->values == b->values && a->n_values == b->n_values && a->row_rank == b->row_rank &&
                           a->col_rank == b->col_rank && a->row_offset == b->row_offset &&
                           a->col_offset == b->col_offset && a->block_offset == b->block_offset);
      if (!x->same) x->b = matrix_from<S>(*b, x->cs);
      x->eps = eps;
      x->adaptive = adaptive;
      x->threads = threads < 1 ? 1 : threads;
      (void)sizeof(T);
      h->s.reset(x);
      x->th = std::thread([x] { x->loop(); });
    };
    if (a->scalar == H2C_REAL) start(new Sliced<Real>);
    else start(new Sliced<Complex>);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int h2o_sliced_step(h2o_sliced* h, double seconds, double* elapsed, int64_t* macs, int64_t* products) {
  SlicedBase& s = *h->s;
  std::unique_lock<std::mutex> lk(s.mu);
  if (s.failed) {
    g_err = s.err;
    return H2C_ERR_INVARIANT;
  }
  const int64_t m0 = s.macs_now;
  const auto t0 = std::chrono::steady_clock::now();
  s.slice_s = seconds;
  s.slice_t0 = t0;
  s.paused = false;
  s.cv.notify_all();
  s.cv.wait(lk, [&] { return s.paused; });
  *elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *macs = s.macs_now - m0;
  *products = s.products;
  if (s.failed) {
    g_err = s.err;
    return H2C_ERR_INVARIANT;
  }
  return H2C_OK;
}

void h2o_sliced_stop(h2o_sliced* h) {
  if (!h) return;
  {
    std::lock_guard<std::mutex> g(h->s->mu);
    h->s->stop = true;
    h->s->paused = false;
    h->s->cv.notify_all();
  }
  if (h->s->th.joinable()) h->s->th.join();
  delete h;
}
