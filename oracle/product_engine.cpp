// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// Single-threaded CPU restatement of the reference's accuracy-controlled H^2
// matrix-matrix product (ProductEngine, proj/core/src/mmp.cpp:13-684).  The
// control flow, accumulation order and MAC counters follow the reference
// exactly; line citations name the reference statement each step restates.
//
// One deliberate difference, value-neutral: the leaf F^A*F^B cache
// (mmp.cpp:127-133) is bounded by MmpOptions::ff_cache_bytes; past the bound
// products are recomputed, but still counted once per (i,j,k) exactly where
// the reference's cache would first have computed them.
#include <algorithm>
#include <chrono>
#include <cmath>

#include "linalg.hpp"
#include "model.hpp"

namespace h2o {

namespace {

template <class S>
class Engine {
  using M = Mat<S>;

 public:
  Engine(const H2Matrix<S>& a, const H2Matrix<S>& b, double eps, bool adaptive,
         const MmpOptions& opt)
      : A(a), B(b), T(*a.tree), BT(*a.structure), eps_(eps), adaptive_(adaptive), opt_(opt) {}

  MmpResult<S> run() {
    const auto t0 = std::chrono::steady_clock::now();
    // mmp.cpp:58-63
    if (A.tree != B.tree || A.structure != B.structure)
      throw ConfigError("mmp: operands must share cluster trees and block structure");
    if (adaptive_ && !(eps_ > 0.0 && eps_ < 1.0)) throw ConfigError("mmp: eps_trunc must be in (0,1)");

    const size_t nc = T.clusters.size();
    C.tree = A.tree;  // mmp.cpp:25-35
    C.structure = A.structure;
    C.row_basis.resize(nc);
    C.col_basis.resize(nc);
    pa_.assign(nc, {});
    pb_.assign(nc, {});
    rep_.eps_trunc = adaptive_ ? eps_ : 0.0;
    rep_.adaptive = adaptive_;
    rep_.levels.resize(T.depth + 1);
    for (int l = 0; l <= T.depth; ++l) rep_.levels[l].level = l;

    adjacency();
    basis_products_pass();
    leaf_phase();
    ff_.clear();
    for (int l = T.depth - 1; l >= 1; --l) upper_level(l);
    if (!pending_.empty()) throw InvariantError("mmp: pending couplings left after the bottom-up pass");
    split_down();
    if (!nl_.empty()) throw InvariantError("mmp: couplings left on non-leaf blocks after the split");
    rep_.pending_after_split = 0;
    rep_.flops = flops_;
    rep_.case_flops = case_flops_;
    rep_.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(C), std::move(rep_)};
  }

  std::vector<M> take_basis_products() { return std::move(bp_); }
  void only_basis_products() { adjacency(); basis_products_pass(); }

 private:
  // ---- counted algebra (mmp.cpp:67-85) -----------------------------------
  void count(std::int64_t w) {
    flops_ += w;
    if (case_ >= 0) case_flops_[case_] += w;
  }
  M mm(Op oa, const M& x, Op ob, const M& y) {
    const Index m = oa == Op::N ? x.r : x.c;
    const Index k = oa == Op::N ? x.c : x.r;
    const Index n = ob == Op::N ? y.c : y.r;
    count(m * k * n);
    return mul(oa, x, ob, y);
  }
  M mm(const M& x, const M& y) { return mm(Op::N, x, Op::N, y); }
  // acc += x x^H with the reference's hand count rows*rows*cols (mmp.cpp:240-243)
  void outer(M& acc, const M& x) {
    gemm(Op::N, Op::H, x, x, acc, true);
    flops_ += x.r * x.r * x.c;
  }
  TruncatedBasis<S> trunc(const M& g) {
    flops_ += 9 * g.r * g.r * g.r;  // mmp.cpp:78
    auto t = svd_truncate_gram<S>(g, eps_);
    // oracle diagnostic: distance of the eigenvalues to the strict threshold
    if (!t.eigenvalues.empty()) {
      const double top = t.eigenvalues.back();
      for (double w : t.eigenvalues)
        if (w > 0) rep_.min_threshold_margin =
            std::min(rep_.min_threshold_margin, std::abs(w - eps_ * top) / (eps_ * top));
    }
    return t;
  }
  static void add_normed(M& acc, const M& g) {  // mmp.cpp:82-85
    const double n = g.norm();
    if (n > 0.0)
      for (size_t i = 0; i < acc.d.size(); ++i) acc.d[i] += g.d[i] / n;
  }
  Index kcr(int id) const { return C.row_basis.rank[id]; }
  Index kcc(int id) const { return C.col_basis.rank[id]; }
  int sz(int id) const { return T.clusters[id].size(); }

  // ---- adjacency (mmp.cpp:92-103) ----------------------------------------
  void adjacency() {
    rows_.assign(T.clusters.size(), {});
    cols_.assign(T.clusters.size(), {});
    for (int l = 0; l <= BT.depth(); ++l)
      for (const BlockEntry& e : BT.level_blocks(l)) {
        rows_[e.key.row].push_back({e.key.col, e.kind});
        cols_[e.key.col].push_back({e.key.row, e.kind});
      }
    for (auto& v : rows_) std::sort(v.begin(), v.end());
    for (auto& v : cols_) std::sort(v.begin(), v.end());
  }

  // ---- B_j = (V^A_col,j)^T V^B_row,j (mmp.cpp:106-124) -------------------
  void basis_products_pass() {
    bp_.assign(T.clusters.size(), {});
    for (int id : T.levels[T.depth]) bp_[id] = mm(Op::T, A.col_basis.leaf[id], Op::N, B.row_basis.leaf[id]);
    for (int l = T.depth - 1; l >= 1; --l)
      for (int id : T.levels[l]) {
        const Cluster& c = T.clusters[id];
        const M& ta = A.col_basis.transfer[id];
        const M& tb = B.row_basis.transfer[id];
        const Index ka = A.col_basis.rank[c.child[0]], kb = B.row_basis.rank[c.child[0]];
        bp_[id] = mm(mm(Op::T, ta.rows_range(0, ka), Op::N, bp_[c.child[0]]), tb.rows_range(0, kb));
        bp_[id] += mm(mm(Op::T, ta.rows_range(ka, ta.r - ka), Op::N, bp_[c.child[1]]),
                      tb.rows_range(kb, tb.r - kb));
      }
  }

  // ---- leaf F^A_ij F^B_jk (mmp.cpp:127-133) ------------------------------
  // `first_touch` marks the statement at which the reference's cache would
  // compute (and count) the product.
  M ff(int i, int j, int k, bool first_touch) {
    const auto key = std::make_tuple(i, j, k);
    if (auto it = ff_.find(key); it != ff_.end()) return it->second;
    if (first_touch) count(Index(sz(i)) * sz(j) * sz(k));
    M p = mul(A.full.at({i, j}), B.full.at({j, k}));
    const std::int64_t bytes = std::int64_t(p.size()) * sizeof(S);
    if (ff_bytes_ + bytes <= opt_.ff_cache_bytes) {
      ff_bytes_ += bytes;
      ff_.emplace(key, p);
    }
    return p;
  }
  bool qualifying(int i, int k) const {  // mmp.cpp:135-138
    const TargetStatus s = BT.target_status(i, k);
    return s == TargetStatus::admissible || s == TargetStatus::inside_admissible;
  }
  void deposit(int i, int k, TargetStatus st, const M& x) {  // mmp.cpp:140-160
    switch (st) {
      case TargetStatus::admissible: C.coupling.at({i, k}) += x; return;
      case TargetStatus::inside_admissible: {
        M& s = pending_[{i, k}];
        if (s.size() == 0) s = M(kcr(i), kcc(k));
        s += x;
        return;
      }
      case TargetStatus::subdivided: {
        M& s = nl_[{i, k}];
        if (s.size() == 0) s = M(kcr(i), kcc(k));
        s += x;
        return;
      }
      case TargetStatus::full_block: throw InvariantError("mmp: coupling contribution aimed at a full block");
    }
  }

  // ---- leaf bases (mmp.cpp:164-238) --------------------------------------
  M leaf_row(int i, LevelStats& st, bool& degen) {
    const Index n = sz(i);
    M g1(n, n), g2(n, n);
    int t1 = 0, t2 = 0;
    for (const auto& [j, ka] : rows_[i]) {
      if (ka != BlockKind::inadmissible_leaf) continue;
      for (const auto& [k, kb] : rows_[j]) {
        if (kb != BlockKind::inadmissible_leaf || !qualifying(i, k)) continue;
        const M x = ff(i, j, k, /*first_touch=*/adaptive_);
        gemm(Op::N, Op::H, x, x, g1, true);
        flops_ += x.r * x.r * x.c;
        ++t1;
      }
      outer(g2, mm(A.full.at({i, j}), B.row_basis.leaf[j]));  // mmp.cpp:179-185
      ++t2;
    }
    const M& va = A.row_basis.leaf[i];
    const M g3 = mm(Op::N, va, Op::H, va);
    st.max_case1_terms = std::max(st.max_case1_terms, t1);
    st.max_case2_terms = std::max(st.max_case2_terms, t2);
    M g(n, n);
    add_normed(g, g1);
    add_normed(g, g2);
    add_normed(g, g3);
    auto tb = trunc(g);
    degen = tb.degenerate || (g1.norm() == 0.0 && g2.norm() == 0.0 && A.row_basis.degenerate[i]);
    return tb.basis;
  }
  M leaf_col(int k, LevelStats& st, bool& degen) {
    const Index n = sz(k);
    M g1(n, n), g2(n, n);
    int t1 = 0, t3 = 0;
    for (const auto& [j, kb] : cols_[k]) {
      if (kb != BlockKind::inadmissible_leaf) continue;
      for (const auto& [i, ka] : cols_[j]) {
        if (ka != BlockKind::inadmissible_leaf || !qualifying(i, k)) continue;
        const M x = ff(i, j, k, false);
        gemm(Op::T, Op::N, x, x.conjugate(), g1, true);  // x^T conj(x)
        flops_ += x.c * x.c * x.r;
        ++t1;
      }
      const M x = mm(Op::T, A.col_basis.leaf[j], Op::N, B.full.at({j, k}));
      outer(g2, x.transpose());
      ++t3;
    }
    const M& vb = B.col_basis.leaf[k];
    const M g3 = mm(Op::N, vb, Op::H, vb);
    st.max_case1_terms = std::max(st.max_case1_terms, t1);
    st.max_case3_terms = std::max(st.max_case3_terms, t3);
    M g(n, n);
    add_normed(g, g1);
    add_normed(g, g2);
    add_normed(g, g3);
    auto tb = trunc(g);
    degen = tb.degenerate || (g1.norm() == 0.0 && g2.norm() == 0.0 && B.col_basis.degenerate[k]);
    return tb.basis;
  }

  // ---- leaf level (mmp.cpp:245-340) --------------------------------------
  void leaf_phase() {
    const int L = T.depth;
    LevelStats& st = rep_.levels[L];
    for (int id : T.levels[L]) {
      bool dg = false;
      if (adaptive_) C.row_basis.leaf[id] = leaf_row(id, st, dg);
      else { C.row_basis.leaf[id] = A.row_basis.leaf[id]; dg = A.row_basis.degenerate[id]; }
      C.row_basis.rank[id] = C.row_basis.leaf[id].c;
      C.row_basis.degenerate[id] = dg;
      st.max_row_rank = std::max(st.max_row_rank, C.row_basis.rank[id]);
    }
    for (int id : T.levels[L]) {
      bool dg = false;
      if (adaptive_) C.col_basis.leaf[id] = leaf_col(id, st, dg);
      else { C.col_basis.leaf[id] = B.col_basis.leaf[id]; dg = B.col_basis.degenerate[id]; }
      C.col_basis.rank[id] = C.col_basis.leaf[id].c;
      C.col_basis.degenerate[id] = dg;
      st.max_col_rank = std::max(st.max_col_rank, C.col_basis.rank[id]);
    }
    for (int id : T.levels[L]) {  // mmp.cpp:275-284
      if (adaptive_) {
        pa_[id] = mm(Op::H, C.row_basis.leaf[id], Op::N, A.row_basis.leaf[id]);
        pb_[id] = mm(Op::T, B.col_basis.leaf[id], Op::N, C.col_basis.leaf[id].conjugate());
      } else {
        pa_[id] = M::identity(A.row_basis.rank[id]);
        pb_[id] = M::identity(B.col_basis.rank[id]);
      }
    }
    for (const BlockEntry& e : BT.level_blocks(L)) {  // mmp.cpp:287-298
      const int i = e.key.row, j = e.key.col;
      if (e.kind == BlockKind::inadmissible_leaf) {
        ca_[e.key] = mm(mm(Op::H, C.row_basis.leaf[i], Op::N, A.full.at(e.key)), B.row_basis.leaf[j]);
        cb_[e.key] = mm(mm(Op::T, A.col_basis.leaf[i], Op::N, B.full.at(e.key)),
                        C.col_basis.leaf[j].conjugate());
        C.full[e.key] = M(sz(i), sz(j));
      } else if (e.kind == BlockKind::admissible) {
        C.coupling[e.key] = M(kcr(i), kcc(j));
      }
    }
    // mmp.cpp:301-339 — products over the shared middle cluster j
    for (int j : T.levels[L])
      for (const auto& [i, kind_a] : cols_[j])
        for (const auto& [k, kind_b] : rows_[j]) {
          const bool fa = kind_a == BlockKind::inadmissible_leaf;
          const bool fb = kind_b == BlockKind::inadmissible_leaf;
          const int ci = fa ? (fb ? 0 : 1) : (fb ? 2 : 3);
          ++st.case_products[ci];
          const TargetStatus ts = BT.target_status(i, k);
          if (ts == TargetStatus::full_block) {
            const M da = fa ? A.full.at({i, j})
                            : mm(Op::N, mm(A.row_basis.leaf[i], A.coupling.at({i, j})), Op::T,
                                 A.col_basis.leaf[j]);
            const M db = fb ? B.full.at({j, k})
                            : mm(Op::N, mm(B.row_basis.leaf[j], B.coupling.at({j, k})), Op::T,
                                 B.col_basis.leaf[k]);
            C.full.at({i, k}) += mm(da, db);
          } else {
            case_ = ci;
            M x;
            if (fa && fb) {
              x = mm(mm(Op::H, C.row_basis.leaf[i], Op::N, ff(i, j, k, !adaptive_)),
                     C.col_basis.leaf[k].conjugate());
            } else if (fa) {
              x = mm(mm(ca_.at({i, j}), B.coupling.at({j, k})), pb_[k]);
            } else if (fb) {
              x = mm(mm(pa_[i], A.coupling.at({i, j})), cb_.at({j, k}));
            } else {
              x = mm(mm(mm(mm(pa_[i], A.coupling.at({i, j})), bp_[j]), B.coupling.at({j, k})), pb_[k]);
            }
            deposit(i, k, ts, x);
          }
          case_ = -1;
        }
  }

  // ---- non-leaf levels (mmp.cpp:344-613) ---------------------------------
  void merge_children(int level) {  // mmp.cpp:344-365
    std::map<BlockKey, M> child = std::move(pending_);
    pending_.clear();
    merged_.clear();
    for (auto& [key, s] : child) {
      const Cluster& ci = T.clusters[key.row];
      const Cluster& ck = T.clusters[key.col];
      if (ci.level != level + 1) throw InvariantError("mmp: pending coupling at an unexpected level");
      const Cluster& pi = T.clusters[ci.parent];
      const Cluster& pk = T.clusters[ck.parent];
      M& m = merged_[{pi.id, pk.id}];
      if (m.size() == 0)
        m = M(kcr(pi.child[0]) + kcr(pi.child[1]), kcc(pk.child[0]) + kcc(pk.child[1]));
      m.add_block(key.row == pi.child[0] ? 0 : kcr(pi.child[0]),
                  key.col == pk.child[0] ? 0 : kcc(pk.child[0]), s);
    }
  }

  void assemble(int level) {  // mmp.cpp:370-404
    asm_a_.clear();
    asm_b_.clear();
    for (const BlockEntry& e : BT.level_blocks(level)) {
      if (e.kind != BlockKind::subdivided) continue;
      const Cluster& ct = T.clusters[e.key.row];
      const Cluster& cs = T.clusters[e.key.col];
      M am(kcr(ct.child[0]) + kcr(ct.child[1]),
           B.row_basis.rank[cs.child[0]] + B.row_basis.rank[cs.child[1]]);
      M bm(A.col_basis.rank[ct.child[0]] + A.col_basis.rank[ct.child[1]],
           kcc(cs.child[0]) + kcc(cs.child[1]));
      for (int ti = 0; ti < 2; ++ti)
        for (int si = 0; si < 2; ++si) {
          const int tc = ct.child[ti], sc = cs.child[si];
          M qa, qb;
          if (BT.kind(tc, sc).value() == BlockKind::admissible) {
            qa = mm(mm(pa_[tc], A.coupling.at({tc, sc})), bp_[sc]);
            qb = mm(mm(bp_[tc], B.coupling.at({tc, sc})), pb_[sc]);
          } else {
            qa = ca_.at({tc, sc});
            qb = cb_.at({tc, sc});
          }
          am.set_block(ti == 0 ? 0 : kcr(ct.child[0]), si == 0 ? 0 : B.row_basis.rank[cs.child[0]], qa);
          bm.set_block(ti == 0 ? 0 : A.col_basis.rank[ct.child[0]], si == 0 ? 0 : kcc(cs.child[0]), qb);
        }
      asm_a_[e.key] = std::move(am);
      asm_b_[e.key] = std::move(bm);
    }
  }

  void transfers(int level, LevelStats& st, const std::map<int, std::vector<BlockKey>>& mrow,
                 const std::map<int, std::vector<BlockKey>>& mcol) {  // mmp.cpp:406-513
    for (int id : T.levels[level]) {
      const Cluster& c = T.clusters[id];
      bool dg = false;
      if (adaptive_) {
        const Index nch = kcr(c.child[0]) + kcr(c.child[1]);
        M g1(nch, nch), g2(nch, nch), g3(nch, nch);
        int t1 = 0, t2 = 0;
        if (auto it = mrow.find(id); it != mrow.end())
          for (const BlockKey& key : it->second) { outer(g1, merged_.at(key)); ++t1; }
        for (const auto& [j, ka] : rows_[id]) {
          if (ka != BlockKind::subdivided) continue;
          outer(g2, mm(asm_a_.at({id, j}), B.row_basis.transfer[j]));
          ++t2;
        }
        M pch(nch, A.row_basis.rank[c.child[0]] + A.row_basis.rank[c.child[1]]);
        pch.set_block(0, 0, pa_[c.child[0]]);
        pch.set_block(pa_[c.child[0]].r, pa_[c.child[0]].c, pa_[c.child[1]]);
        outer(g3, mm(pch, A.row_basis.transfer[id]));
        st.max_case1_terms = std::max(st.max_case1_terms, t1);
        st.max_case2_terms = std::max(st.max_case2_terms, t2);
        M g(nch, nch);
        add_normed(g, g1);
        add_normed(g, g2);
        add_normed(g, g3);
        auto tb = trunc(g);
        dg = tb.degenerate || (g1.norm() == 0.0 && g2.norm() == 0.0 && A.row_basis.degenerate[id]);
        C.row_basis.transfer[id] = tb.basis;
      } else {
        C.row_basis.transfer[id] = A.row_basis.transfer[id];
        dg = A.row_basis.degenerate[id];
      }
      C.row_basis.rank[id] = C.row_basis.transfer[id].c;
      C.row_basis.degenerate[id] = dg;
      st.max_row_rank = std::max(st.max_row_rank, C.row_basis.rank[id]);
    }
    for (int id : T.levels[level]) {
      const Cluster& c = T.clusters[id];
      bool dg = false;
      if (adaptive_) {
        const Index nch = kcc(c.child[0]) + kcc(c.child[1]);
        M g1(nch, nch), g2(nch, nch), g3(nch, nch);
        int t1 = 0, t3 = 0;
        if (auto it = mcol.find(id); it != mcol.end())
          for (const BlockKey& key : it->second) { outer(g1, merged_.at(key).transpose()); ++t1; }
        for (const auto& [j, kb] : cols_[id]) {
          if (kb != BlockKind::subdivided) continue;
          outer(g2, mm(Op::T, A.col_basis.transfer[j], Op::N, asm_b_.at({j, id})).transpose());
          ++t3;
        }
        M pch(B.col_basis.rank[c.child[0]] + B.col_basis.rank[c.child[1]], nch);
        pch.set_block(0, 0, pb_[c.child[0]]);
        pch.set_block(pb_[c.child[0]].r, pb_[c.child[0]].c, pb_[c.child[1]]);
        outer(g3, mm(Op::T, pch, Op::N, B.col_basis.transfer[id].conjugate()));
        st.max_case1_terms = std::max(st.max_case1_terms, t1);
        st.max_case3_terms = std::max(st.max_case3_terms, t3);
        M g(nch, nch);
        add_normed(g, g1);
        add_normed(g, g2);
        add_normed(g, g3);
        auto tb = trunc(g);
        dg = tb.degenerate || (g1.norm() == 0.0 && g2.norm() == 0.0 && B.col_basis.degenerate[id]);
        C.col_basis.transfer[id] = tb.basis;
      } else {
        C.col_basis.transfer[id] = B.col_basis.transfer[id];
        dg = B.col_basis.degenerate[id];
      }
      C.col_basis.rank[id] = C.col_basis.transfer[id].c;
      C.col_basis.degenerate[id] = dg;
      st.max_col_rank = std::max(st.max_col_rank, C.col_basis.rank[id]);
    }
  }

  void projections_and_collects(int level) {  // mmp.cpp:515-553
    for (int id : T.levels[level]) {
      const Cluster& c = T.clusters[id];
      if (adaptive_) {
        const M& tc = C.row_basis.transfer[id];
        const M& ta = A.row_basis.transfer[id];
        const Index kc1 = kcr(c.child[0]), ka1 = A.row_basis.rank[c.child[0]];
        pa_[id] = mm(mm(Op::H, tc.rows_range(0, kc1), Op::N, pa_[c.child[0]]), ta.rows_range(0, ka1));
        pa_[id] += mm(mm(Op::H, tc.rows_range(kc1, tc.r - kc1), Op::N, pa_[c.child[1]]),
                      ta.rows_range(ka1, ta.r - ka1));
        const M& tcc = C.col_basis.transfer[id];
        const M& tb = B.col_basis.transfer[id];
        const Index kq1 = kcc(c.child[0]), kb1 = B.col_basis.rank[c.child[0]];
        pb_[id] = mm(mm(Op::T, tb.rows_range(0, kb1), Op::N, pb_[c.child[0]]),
                     tcc.rows_range(0, kq1).conjugate());
        pb_[id] += mm(mm(Op::T, tb.rows_range(kb1, tb.r - kb1), Op::N, pb_[c.child[1]]),
                      tcc.rows_range(kq1, tcc.r - kq1).conjugate());
      } else {
        pa_[id] = M::identity(A.row_basis.rank[id]);
        pb_[id] = M::identity(B.col_basis.rank[id]);
      }
    }
    for (const BlockEntry& e : BT.level_blocks(level)) {
      if (e.kind != BlockKind::subdivided) continue;
      const int t = e.key.row, s = e.key.col;
      ca_[e.key] = mm(mm(Op::H, C.row_basis.transfer[t], Op::N, asm_a_.at(e.key)), B.row_basis.transfer[s]);
      cb_[e.key] = mm(mm(Op::T, A.col_basis.transfer[t], Op::N, asm_b_.at(e.key)),
                      C.col_basis.transfer[s].conjugate());
    }
  }

  void upper_level(int level) {  // mmp.cpp:555-613
    LevelStats& st = rep_.levels[level];
    merge_children(level);
    assemble(level);
    std::map<int, std::vector<BlockKey>> mrow, mcol;
    for (const auto& [key, m] : merged_) {
      mrow[key.row].push_back(key);
      mcol[key.col].push_back(key);
    }
    transfers(level, st, mrow, mcol);
    projections_and_collects(level);
    for (const BlockEntry& e : BT.level_blocks(level))
      if (e.kind == BlockKind::admissible) C.coupling[e.key] = M(kcr(e.key.row), kcc(e.key.col));
    for (const auto& [key, m] : merged_) {  // case 1 (mmp.cpp:573-585)
      ++st.case_products[0];
      case_ = 0;
      const M x = mm(mm(Op::H, C.row_basis.transfer[key.row], Op::N, m),
                     C.col_basis.transfer[key.col].conjugate());
      case_ = -1;
      const TargetStatus ts = BT.target_status(key.row, key.col);
      if (ts != TargetStatus::admissible && ts != TargetStatus::inside_admissible)
        throw InvariantError("mmp: merged coupling with an impossible target");
      deposit(key.row, key.col, ts, x);
    }
    for (int j : T.levels[level])  // cases 2-4 (mmp.cpp:587-612)
      for (const auto& [i, kind_a] : cols_[j])
        for (const auto& [k, kind_b] : rows_[j]) {
          const bool na = kind_a == BlockKind::subdivided, nb = kind_b == BlockKind::subdivided;
          if (na && nb) continue;
          const int ci = na ? 1 : (nb ? 2 : 3);
          ++st.case_products[ci];
          case_ = ci;
          M x;
          if (na) x = mm(mm(ca_.at({i, j}), B.coupling.at({j, k})), pb_[k]);
          else if (nb) x = mm(mm(pa_[i], A.coupling.at({i, j})), cb_.at({j, k}));
          else x = mm(mm(mm(mm(pa_[i], A.coupling.at({i, j})), bp_[j]), B.coupling.at({j, k})), pb_[k]);
          case_ = -1;
          deposit(i, k, BT.target_status(i, k), x);
        }
  }

  // ---- top-down split (mmp.cpp:617-659) ----------------------------------
  void split_down() {
    for (int level = 1; level < T.depth; ++level) {
      std::vector<BlockKey> keys;
      for (const auto& [key, m] : nl_)
        if (T.clusters[key.row].level == level) keys.push_back(key);
      for (const BlockKey& key : keys) {
        const M s = std::move(nl_.at(key));
        nl_.erase(key);
        const Cluster& ci = T.clusters[key.row];
        const Cluster& ck = T.clusters[key.col];
        const M& tr = C.row_basis.transfer[key.row];
        const M& tc = C.col_basis.transfer[key.col];
        Index ro = 0;
        for (int ic : ci.child) {
          const Index kr = kcr(ic);
          Index co = 0;
          for (int kc : ck.child) {
            const Index kk = kcc(kc);
            const M x = mm(Op::N, mm(tr.rows_range(ro, kr), s), Op::T, tc.rows_range(co, kk));
            switch (BT.kind(ic, kc).value()) {
              case BlockKind::admissible: C.coupling.at({ic, kc}) += x; break;
              case BlockKind::subdivided: {
                M& slot = nl_[{ic, kc}];
                if (slot.size() == 0) slot = M(kr, kk);
                slot += x;
                break;
              }
              case BlockKind::inadmissible_leaf:
                C.full.at({ic, kc}) += mm(Op::N, mm(C.row_basis.leaf[ic], x), Op::T, C.col_basis.leaf[kc]);
                break;
            }
            co += kk;
          }
          ro += kr;
        }
      }
    }
  }

  const H2Matrix<S>& A;
  const H2Matrix<S>& B;
  const ClusterTree& T;
  const BlockTree& BT;
  double eps_;
  bool adaptive_;
  MmpOptions opt_;
  H2Matrix<S> C;
  MmpReport rep_;
  std::vector<std::vector<std::pair<int, BlockKind>>> rows_, cols_;
  std::vector<M> bp_, pa_, pb_;
  std::map<BlockKey, M> ca_, cb_, pending_, nl_, merged_, asm_a_, asm_b_;
  std::map<std::tuple<int, int, int>, M> ff_;
  std::int64_t ff_bytes_ = 0;
  std::int64_t flops_ = 0;
  std::array<std::int64_t, 4> case_flops_{0, 0, 0, 0};
  int case_ = -1;
};

}  // namespace

template <class S>
MmpResult<S> mmp(const H2Matrix<S>& a, const H2Matrix<S>& b, double eps, const MmpOptions& opt) {
  return Engine<S>(a, b, eps, true, opt).run();
}
template <class S>
MmpResult<S> formatted_mmp(const H2Matrix<S>& a, const H2Matrix<S>& b, const MmpOptions& opt) {
  return Engine<S>(a, b, 0.0, false, opt).run();
}
// mmp.cpp:693-714 (uncounted public variant)
template <class S>
std::vector<Mat<S>> basis_products(const H2Matrix<S>& a, const H2Matrix<S>& b) {
  if (a.tree != b.tree) throw ConfigError("basis_products: operands must share cluster trees");
  Engine<S> e(a, b, 0.5, true, MmpOptions{});
  e.only_basis_products();
  return e.take_basis_products();
}

template MmpResult<Real> mmp<Real>(const H2Matrix<Real>&, const H2Matrix<Real>&, double, const MmpOptions&);
template MmpResult<Complex> mmp<Complex>(const H2Matrix<Complex>&, const H2Matrix<Complex>&, double,
                                         const MmpOptions&);
template MmpResult<Real> formatted_mmp<Real>(const H2Matrix<Real>&, const H2Matrix<Real>&, const MmpOptions&);
template MmpResult<Complex> formatted_mmp<Complex>(const H2Matrix<Complex>&, const H2Matrix<Complex>&,
                                                   const MmpOptions&);
template std::vector<Mat<Real>> basis_products<Real>(const H2Matrix<Real>&, const H2Matrix<Real>&);
template std::vector<Mat<Complex>> basis_products<Complex>(const H2Matrix<Complex>&,
                                                           const H2Matrix<Complex>&);

}  // namespace h2o
