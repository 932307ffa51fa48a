// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// CPU restatement of the reference's accuracy-controlled H^2 matrix-matrix
// product (ProductEngine, proj/core/src/mmp.cpp:13-684).  The control flow,
// accumulation order and MAC counters follow the reference exactly; line
// citations name the reference statement each step restates.
//
// Threads (MmpOptions::threads, a small std::thread pool): the reference is single-threaded
// (mmp.hpp:56-59).  With more than one thread the oracle runs every per-cluster
// and per-block loop of a phase in parallel WITHOUT changing any value: each
// output (basis, collect, target block) is owned by exactly one task, and the
// contributions to a coupling target (i,k) are still added in the reference's
// order — case 1 first, then the triples in ascending position of the middle
// cluster j (mmp.cpp:301-339, 573-612) — because one task walks row i's blocks
// in exactly that order.  Counters are integers summed per thread.  Result:
// bit-identical C and MmpReport for any thread count (tests/test_oracle_pins.py).
//
// Value-neutral difference: the leaf F^A*F^B cache (mmp.cpp:127-133) is
// bounded by MmpOptions::ff_cache_bytes (0 with threads > 1); past the bound
// products are recomputed, but still counted once per (i,j,k) exactly where
// the reference's cache would first have computed them.
//
// Slicing (MmpOptions::gate): between chunks of a parallel loop the engine
// calls gate(macs counted so far); the sliced CPU baseline of bench.py uses it
// to pause the product at slice boundaries (oracle/capi.cpp, h2o_sliced_*).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>

#include "linalg.hpp"
#include "model.hpp"

namespace h2o {

namespace {

// worker index of the calling thread inside Pool::run (0 = the caller)
thread_local int t_tid = 0;

// Fixed pool of n-1 workers plus the calling thread; run() hands out the
// indices of [a, b) dynamically and returns when all are done.
class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int w = 1; w < n; ++w) th_.emplace_back([this, w] { worker(w); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(std::int64_t a, std::int64_t b, const std::function<void(std::int64_t)>& fn) {
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      next_.store(a);
      end_ = b;
      busy_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    drain(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return busy_ == 0; });
    fn_ = nullptr;
  }

 private:
  void drain(int w) {
    t_tid = w;
    for (;;) {
      const std::int64_t x = next_.fetch_add(1);
      if (x >= end_) break;
      (*fn_)(x);
    }
    t_tid = 0;
  }
  void worker(int w) {
    std::uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
      }
      drain(w);
      std::lock_guard<std::mutex> g(mu_);
      if (--busy_ == 0) done_.notify_all();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(std::int64_t)>* fn_ = nullptr;
  std::atomic<std::int64_t> next_{0};
  std::int64_t end_ = 0;
  int busy_ = 0;
  std::uint64_t gen_ = 0;
  bool quit_ = false;
};

struct alignas(64) Tally {
  std::int64_t flops = 0;
  std::array<std::int64_t, 4> cf{0, 0, 0, 0};
  int case_ = -1;
  double margin = 1e300;
};

void merge_stats(LevelStats& st, const std::vector<LevelStats>& part) {
  for (const LevelStats& p : part) {
    st.max_row_rank = std::max(st.max_row_rank, p.max_row_rank);
    st.max_col_rank = std::max(st.max_col_rank, p.max_col_rank);
    for (int c = 0; c < 4; ++c) st.case_products[c] += p.case_products[c];
    st.max_case1_terms = std::max(st.max_case1_terms, p.max_case1_terms);
    st.max_case2_terms = std::max(st.max_case2_terms, p.max_case2_terms);
    st.max_case3_terms = std::max(st.max_case3_terms, p.max_case3_terms);
  }
}

template <class S>
class Engine {
  using M = Mat<S>;

 public:
  Engine(const H2Matrix<S>& a, const H2Matrix<S>& b, double eps, bool adaptive,
         const MmpOptions& opt)
      : A(a), B(b), T(*a.tree), BT(*a.structure), eps_(eps), adaptive_(adaptive), opt_(opt) {
    threads_ = std::max(1, opt_.threads);
    if (threads_ > 1) opt_.ff_cache_bytes = 0;  // the cache is shared mutable state
    tl_.resize(threads_);
    if (threads_ > 1) pool_ = std::make_unique<Pool>(threads_);
  }

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
    rep_.flops = 0;
    rep_.case_flops = {0, 0, 0, 0};
    for (const Tally& t : tl_) {
      rep_.flops += t.flops;
      for (int c = 0; c < 4; ++c) rep_.case_flops[c] += t.cf[c];
      rep_.min_threshold_margin = std::min(rep_.min_threshold_margin, t.margin);
    }
    rep_.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(C), std::move(rep_)};
  }

  std::vector<M> take_basis_products() { return std::move(bp_); }
  void only_basis_products() { adjacency(); basis_products_pass(); }

 private:
  // ---- threads --------------------------------------------------------------
  Tally& me() { return tl_[t_tid]; }
  int tid() const { return t_tid; }
  std::int64_t counted() const {
    std::int64_t s = 0;
    for (const Tally& t : tl_) s += t.flops;
    return s;
  }
  // slice point (serial): report progress; the gate may block or throw
  void tick() {
    if (opt_.gate) opt_.gate(counted());
  }
  // parallel for over [0, n); exceptions are rethrown after the loop.  With a
  // gate, the loop runs in up to 64 consecutive chunks (of >= 16 tasks per thread)
  // with a slice point after each.
  template <class F>
  void pfor(std::int64_t n, F&& fn) {
    if (n <= 0) return;
    const std::int64_t nch =
        opt_.gate ? std::max<std::int64_t>(1, std::min<std::int64_t>(64, n / (16 * std::int64_t(threads_)))) : 1;
    for (std::int64_t c = 0; c < nch; ++c) {
      const std::int64_t a = n * c / nch, b = n * (c + 1) / nch;
      std::exception_ptr err;
      if (threads_ == 1) {
        for (std::int64_t x = a; x < b; ++x) fn(x);
      } else {
        std::mutex em;
        const std::function<void(std::int64_t)> body = [&](std::int64_t x) {
          try {
            fn(x);
          } catch (...) {
            std::lock_guard<std::mutex> g(em);
            if (!err) err = std::current_exception();
          }
        };
        pool_->run(a, b, body);
      }
      if (err) std::rethrow_exception(err);
      tick();
    }
  }
  std::vector<LevelStats> stats_parts() const { return std::vector<LevelStats>(threads_); }

  // ---- counted algebra (mmp.cpp:67-80) -----------------------------------
  void count(std::int64_t w) {
    Tally& t = me();
    t.flops += w;
    if (t.case_ >= 0) t.cf[t.case_] += w;
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
    me().flops += x.r * x.r * x.c;
  }
  TruncatedBasis<S> trunc(const M& g) {
    me().flops += 9 * g.r * g.r * g.r;  // mmp.cpp:78
    auto t = svd_truncate_gram<S>(g, eps_);
    // oracle diagnostic: distance of the eigenvalues to the strict threshold
    if (!t.eigenvalues.empty()) {
      const double top = t.eigenvalues.back();
      double& mg = me().margin;
      for (double w : t.eigenvalues)
        if (w > 0) mg = std::min(mg, std::abs(w - eps_ * top) / (eps_ * top));
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
    // position of each cluster in its level list (the middle-cluster order of
    // the four-case loops, mmp.cpp:301,587: `for j in levels[l]`)
    pos_.assign(T.clusters.size(), 0);
    for (const auto& lv : T.levels)
      for (size_t p = 0; p < lv.size(); ++p) pos_[lv[p]] = static_cast<int>(p);
  }

  // ---- B_j = (V^A_col,j)^T V^B_row,j (mmp.cpp:106-124) -------------------
  void basis_products_pass() {
    bp_.assign(T.clusters.size(), {});
    const auto& leaves = T.levels[T.depth];
    pfor(leaves.size(), [&](std::int64_t x) {
      const int id = leaves[x];
      bp_[id] = mm(Op::T, A.col_basis.leaf[id], Op::N, B.row_basis.leaf[id]);
    });
    for (int l = T.depth - 1; l >= 1; --l) {
      const auto& ids = T.levels[l];
      pfor(ids.size(), [&](std::int64_t x) {
        const int id = ids[x];
        const Cluster& c = T.clusters[id];
        const M& ta = A.col_basis.transfer[id];
        const M& tb = B.row_basis.transfer[id];
        const Index ka = A.col_basis.rank[c.child[0]], kb = B.row_basis.rank[c.child[0]];
        M v = mm(mm(Op::T, ta.rows_range(0, ka), Op::N, bp_[c.child[0]]), tb.rows_range(0, kb));
        v += mm(mm(Op::T, ta.rows_range(ka, ta.r - ka), Op::N, bp_[c.child[1]]), tb.rows_range(kb, tb.r - kb));
        bp_[id] = std::move(v);
      });
    }
  }

  // ---- leaf F^A_ij F^B_jk (mmp.cpp:127-133) ------------------------------
  // `first_touch` marks the statement at which the reference's cache would
  // compute (and count) the product.
  M ff(int i, int j, int k, bool first_touch) {
    const auto key = std::make_tuple(i, j, k);
    if (opt_.ff_cache_bytes > 0)
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

  // ---- coupling targets (mmp.cpp:140-160) --------------------------------
  // Every target (i,k) of a level is resolved once, by the serial pass that
  // creates the reference's lazily-created pending_ / nl_ entries for exactly
  // the targets that receive a contribution; the parallel tasks then add into
  // the resolved blocks in the reference's order.
  struct Target {
    int k;
    TargetStatus st;
    M* dst;
  };
  using RowTargets = std::vector<Target>;  // sorted by k
  static Target* find_target(RowTargets& v, int k) {
    auto it = std::lower_bound(v.begin(), v.end(), k, [](const Target& t, int kk) { return t.k < kk; });
    return (it != v.end() && it->k == k) ? &*it : nullptr;
  }
  void resolve_targets(std::vector<RowTargets>& rt) {
    for (size_t i = 0; i < rt.size(); ++i)
      for (Target& t : rt[i]) {
        const int ii = static_cast<int>(i);
        switch (t.st) {
          case TargetStatus::admissible: t.dst = &C.coupling.at({ii, t.k}); break;
          case TargetStatus::inside_admissible: {
            M& s = pending_[{ii, t.k}];
            if (s.size() == 0) s = M(kcr(ii), kcc(t.k));
            t.dst = &s;
            break;
          }
          case TargetStatus::subdivided: {
            M& s = nl_[{ii, t.k}];
            if (s.size() == 0) s = M(kcr(ii), kcc(t.k));
            t.dst = &s;
            break;
          }
          case TargetStatus::full_block: t.dst = nullptr; break;
        }
      }
  }
  static void deposit(const Target& t, const M& x) {  // mmp.cpp:140-160
    if (!t.dst) throw InvariantError("mmp: coupling contribution aimed at a full block");
    *t.dst += x;
  }
  // blocks of row i in the order the middle cluster j is visited (its level position)
  std::vector<std::pair<int, BlockKind>> row_in_order(int i, int level) const {
    std::vector<std::pair<int, BlockKind>> r;
    for (const auto& e : rows_[i])
      if (T.clusters[e.first].level == level) r.push_back(e);
    std::stable_sort(r.begin(), r.end(), [&](const auto& a, const auto& b) { return pos_[a.first] < pos_[b.first]; });
    return r;
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
        me().flops += x.r * x.r * x.c;
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
        me().flops += x.c * x.c * x.r;
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
    const auto& ids = T.levels[L];
    {
      auto part = stats_parts();
      pfor(ids.size(), [&](std::int64_t x) {
        const int id = ids[x];
        LevelStats& s = part[tid()];
        bool dg = false;
        if (adaptive_) C.row_basis.leaf[id] = leaf_row(id, s, dg);
        else { C.row_basis.leaf[id] = A.row_basis.leaf[id]; dg = A.row_basis.degenerate[id]; }
        C.row_basis.rank[id] = C.row_basis.leaf[id].c;
        C.row_basis.degenerate[id] = dg;
        s.max_row_rank = std::max(s.max_row_rank, C.row_basis.rank[id]);
      });
      merge_stats(st, part);
    }
    {
      auto part = stats_parts();
      pfor(ids.size(), [&](std::int64_t x) {
        const int id = ids[x];
        LevelStats& s = part[tid()];
        bool dg = false;
        if (adaptive_) C.col_basis.leaf[id] = leaf_col(id, s, dg);
        else { C.col_basis.leaf[id] = B.col_basis.leaf[id]; dg = B.col_basis.degenerate[id]; }
        C.col_basis.rank[id] = C.col_basis.leaf[id].c;
        C.col_basis.degenerate[id] = dg;
        s.max_col_rank = std::max(s.max_col_rank, C.col_basis.rank[id]);
      });
      merge_stats(st, part);
    }
    pfor(ids.size(), [&](std::int64_t x) {  // mmp.cpp:275-284
      const int id = ids[x];
      if (adaptive_) {
        pa_[id] = mm(Op::H, C.row_basis.leaf[id], Op::N, A.row_basis.leaf[id]);
        pb_[id] = mm(Op::T, B.col_basis.leaf[id], Op::N, C.col_basis.leaf[id].conjugate());
      } else {
        pa_[id] = M::identity(A.row_basis.rank[id]);
        pb_[id] = M::identity(B.col_basis.rank[id]);
      }
    });
    // mmp.cpp:287-298 (map slots created serially, filled in parallel)
    const auto& blocks = BT.level_blocks(L);
    std::vector<std::pair<M*, M*>> coll(blocks.size(), {nullptr, nullptr});
    for (size_t b = 0; b < blocks.size(); ++b) {
      const BlockEntry& e = blocks[b];
      const int i = e.key.row, j = e.key.col;
      if (e.kind == BlockKind::inadmissible_leaf) {
        coll[b] = {&ca_[e.key], &cb_[e.key]};
        C.full[e.key] = M(sz(i), sz(j));
      } else if (e.kind == BlockKind::admissible) {
        C.coupling[e.key] = M(kcr(i), kcc(j));
      }
    }
    pfor(blocks.size(), [&](std::int64_t b) {
      const BlockEntry& e = blocks[b];
      if (e.kind != BlockKind::inadmissible_leaf) return;
      const int i = e.key.row, j = e.key.col;
      *coll[b].first = mm(mm(Op::H, C.row_basis.leaf[i], Op::N, A.full.at(e.key)), B.row_basis.leaf[j]);
      *coll[b].second = mm(mm(Op::T, A.col_basis.leaf[i], Op::N, B.full.at(e.key)), C.col_basis.leaf[j].conjugate());
    });

    // mmp.cpp:301-339 — products over the shared middle cluster j, one task per
    // target row i (contributions to (i,k) in ascending position of j)
    const int nc = static_cast<int>(T.clusters.size());
    std::vector<RowTargets> rt(nc);
    pfor(ids.size(), [&](std::int64_t x) {
      const int i = ids[x];
      RowTargets& v = rt[i];
      for (const auto& [j, ka] : rows_[i]) {
        if (T.clusters[j].level != L) continue;
        for (const auto& [k, kb] : rows_[j]) {
          (void)kb;
          if (find_target(v, k)) continue;
          auto it = std::lower_bound(v.begin(), v.end(), k, [](const Target& t, int kk) { return t.k < kk; });
          v.insert(it, Target{k, BT.target_status(i, k), nullptr});
        }
      }
    });
    resolve_targets(rt);
    auto part = stats_parts();
    pfor(ids.size(), [&](std::int64_t x) {
      const int i = ids[x];
      LevelStats& s = part[tid()];
      RowTargets& v = rt[i];
      for (const auto& [j, kind_a] : row_in_order(i, L))
        for (const auto& [k, kind_b] : rows_[j]) {
          const bool fa = kind_a == BlockKind::inadmissible_leaf;
          const bool fb = kind_b == BlockKind::inadmissible_leaf;
          const int ci = fa ? (fb ? 0 : 1) : (fb ? 2 : 3);
          ++s.case_products[ci];
          const Target& tg = *find_target(v, k);
          if (tg.st == TargetStatus::full_block) {
            const M da = fa ? A.full.at({i, j})
                            : mm(Op::N, mm(A.row_basis.leaf[i], A.coupling.at({i, j})), Op::T,
                                 A.col_basis.leaf[j]);
            const M db = fb ? B.full.at({j, k})
                            : mm(Op::N, mm(B.row_basis.leaf[j], B.coupling.at({j, k})), Op::T,
                                 B.col_basis.leaf[k]);
            C.full.at({i, k}) += mm(da, db);
          } else {
            me().case_ = ci;
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
            me().case_ = -1;
            deposit(tg, x);
          }
        }
    });
    merge_stats(st, part);
  }

  // ---- non-leaf levels (mmp.cpp:344-613) ---------------------------------
  void merge_children(int level) {  // mmp.cpp:344-365
    std::map<BlockKey, M> child = std::move(pending_);
    pending_.clear();
    merged_.clear();
    struct Put {
      M* dst;
      Index r0, c0;
      const M* src;
    };
    std::vector<Put> puts;
    puts.reserve(child.size());
    for (auto& [key, s] : child) {
      const Cluster& ci = T.clusters[key.row];
      const Cluster& ck = T.clusters[key.col];
      if (ci.level != level + 1) throw InvariantError("mmp: pending coupling at an unexpected level");
      const Cluster& pi = T.clusters[ci.parent];
      const Cluster& pk = T.clusters[ck.parent];
      M& m = merged_[{pi.id, pk.id}];
      if (m.size() == 0)
        m = M(kcr(pi.child[0]) + kcr(pi.child[1]), kcc(pk.child[0]) + kcc(pk.child[1]));
      puts.push_back({&m, key.row == pi.child[0] ? 0 : kcr(pi.child[0]), key.col == pk.child[0] ? 0 : kcc(pk.child[0]),
                      &s});
    }
    pfor(puts.size(), [&](std::int64_t x) { puts[x].dst->add_block(puts[x].r0, puts[x].c0, *puts[x].src); });
  }

  void assemble(int level) {  // mmp.cpp:370-404
    asm_a_.clear();
    asm_b_.clear();
    const auto& blocks = BT.level_blocks(level);
    std::vector<std::pair<M*, M*>> dst(blocks.size(), {nullptr, nullptr});
    for (size_t b = 0; b < blocks.size(); ++b)
      if (blocks[b].kind == BlockKind::subdivided) dst[b] = {&asm_a_[blocks[b].key], &asm_b_[blocks[b].key]};
    pfor(blocks.size(), [&](std::int64_t b) {
      const BlockEntry& e = blocks[b];
      if (e.kind != BlockKind::subdivided) return;
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
      *dst[b].first = std::move(am);
      *dst[b].second = std::move(bm);
    });
  }

  void transfers(int level, LevelStats& st, const std::map<int, std::vector<BlockKey>>& mrow,
                 const std::map<int, std::vector<BlockKey>>& mcol) {  // mmp.cpp:406-513
    const auto& ids = T.levels[level];
    {
      auto part = stats_parts();
      pfor(ids.size(), [&](std::int64_t x) {
        const int id = ids[x];
        LevelStats& s = part[tid()];
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
          s.max_case1_terms = std::max(s.max_case1_terms, t1);
          s.max_case2_terms = std::max(s.max_case2_terms, t2);
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
        s.max_row_rank = std::max(s.max_row_rank, C.row_basis.rank[id]);
      });
      merge_stats(st, part);
    }
    {
      auto part = stats_parts();
      pfor(ids.size(), [&](std::int64_t x) {
        const int id = ids[x];
        LevelStats& s = part[tid()];
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
          s.max_case1_terms = std::max(s.max_case1_terms, t1);
          s.max_case3_terms = std::max(s.max_case3_terms, t3);
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
        s.max_col_rank = std::max(s.max_col_rank, C.col_basis.rank[id]);
      });
      merge_stats(st, part);
    }
  }

  void projections_and_collects(int level) {  // mmp.cpp:515-553
    const auto& ids = T.levels[level];
    pfor(ids.size(), [&](std::int64_t x) {
      const int id = ids[x];
      const Cluster& c = T.clusters[id];
      if (adaptive_) {
        const M& tc = C.row_basis.transfer[id];
        const M& ta = A.row_basis.transfer[id];
        const Index kc1 = kcr(c.child[0]), ka1 = A.row_basis.rank[c.child[0]];
        M pa = mm(mm(Op::H, tc.rows_range(0, kc1), Op::N, pa_[c.child[0]]), ta.rows_range(0, ka1));
        pa += mm(mm(Op::H, tc.rows_range(kc1, tc.r - kc1), Op::N, pa_[c.child[1]]), ta.rows_range(ka1, ta.r - ka1));
        const M& tcc = C.col_basis.transfer[id];
        const M& tb = B.col_basis.transfer[id];
        const Index kq1 = kcc(c.child[0]), kb1 = B.col_basis.rank[c.child[0]];
        M pb = mm(mm(Op::T, tb.rows_range(0, kb1), Op::N, pb_[c.child[0]]), tcc.rows_range(0, kq1).conjugate());
        pb += mm(mm(Op::T, tb.rows_range(kb1, tb.r - kb1), Op::N, pb_[c.child[1]]),
                 tcc.rows_range(kq1, tcc.r - kq1).conjugate());
        pa_[id] = std::move(pa);
        pb_[id] = std::move(pb);
      } else {
        pa_[id] = M::identity(A.row_basis.rank[id]);
        pb_[id] = M::identity(B.col_basis.rank[id]);
      }
    });
    const auto& blocks = BT.level_blocks(level);
    std::vector<std::pair<M*, M*>> dst(blocks.size(), {nullptr, nullptr});
    for (size_t b = 0; b < blocks.size(); ++b)
      if (blocks[b].kind == BlockKind::subdivided) dst[b] = {&ca_[blocks[b].key], &cb_[blocks[b].key]};
    pfor(blocks.size(), [&](std::int64_t b) {
      const BlockEntry& e = blocks[b];
      if (e.kind != BlockKind::subdivided) return;
      const int t = e.key.row, s = e.key.col;
      *dst[b].first = mm(mm(Op::H, C.row_basis.transfer[t], Op::N, asm_a_.at(e.key)), B.row_basis.transfer[s]);
      *dst[b].second =
          mm(mm(Op::T, A.col_basis.transfer[t], Op::N, asm_b_.at(e.key)), C.col_basis.transfer[s].conjugate());
    });
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
    // case 1 (mmp.cpp:573-585) and cases 2-4 (:587-612), one task per target
    // row i: merged (i,k) first, then the triples in ascending position of j
    const auto& ids = T.levels[level];
    const int nc = static_cast<int>(T.clusters.size());
    std::vector<RowTargets> rt(nc);
    pfor(ids.size(), [&](std::int64_t x) {
      const int i = ids[x];
      RowTargets& v = rt[i];
      auto add = [&](int k) {
        if (find_target(v, k)) return;
        auto it = std::lower_bound(v.begin(), v.end(), k, [](const Target& t, int kk) { return t.k < kk; });
        v.insert(it, Target{k, BT.target_status(i, k), nullptr});
      };
      if (auto it = mrow.find(i); it != mrow.end())
        for (const BlockKey& key : it->second) add(key.col);
      for (const auto& [j, ka] : rows_[i]) {
        if (T.clusters[j].level != level) continue;
        for (const auto& [k, kb] : rows_[j]) {
          if (ka == BlockKind::subdivided && kb == BlockKind::subdivided) continue;
          add(k);
        }
      }
    });
    resolve_targets(rt);
    auto part = stats_parts();
    pfor(ids.size(), [&](std::int64_t x) {
      const int i = ids[x];
      LevelStats& s = part[tid()];
      RowTargets& v = rt[i];
      if (auto it = mrow.find(i); it != mrow.end())
        for (const BlockKey& key : it->second) {
          const M& m = merged_.at(key);
          ++s.case_products[0];
          me().case_ = 0;
          const M x1 = mm(mm(Op::H, C.row_basis.transfer[key.row], Op::N, m), C.col_basis.transfer[key.col].conjugate());
          me().case_ = -1;
          const Target& tg = *find_target(v, key.col);
          if (tg.st != TargetStatus::admissible && tg.st != TargetStatus::inside_admissible)
            throw InvariantError("mmp: merged coupling with an impossible target");
          deposit(tg, x1);
        }
      for (const auto& [j, kind_a] : row_in_order(i, level))
        for (const auto& [k, kind_b] : rows_[j]) {
          const bool na = kind_a == BlockKind::subdivided, nb = kind_b == BlockKind::subdivided;
          if (na && nb) continue;
          const int ci = na ? 1 : (nb ? 2 : 3);
          ++s.case_products[ci];
          me().case_ = ci;
          M x2;
          if (na) x2 = mm(mm(ca_.at({i, j}), B.coupling.at({j, k})), pb_[k]);
          else if (nb) x2 = mm(mm(pa_[i], A.coupling.at({i, j})), cb_.at({j, k}));
          else x2 = mm(mm(mm(mm(pa_[i], A.coupling.at({i, j})), bp_[j]), B.coupling.at({j, k})), pb_[k]);
          me().case_ = -1;
          deposit(*find_target(v, k), x2);
        }
    });
    merge_stats(st, part);
  }

  // ---- top-down split (mmp.cpp:617-659) ----------------------------------
  void split_down() {
    for (int level = 1; level < T.depth; ++level) {
      std::vector<BlockKey> keys;
      for (const auto& [key, m] : nl_)
        if (T.clusters[key.row].level == level) keys.push_back(key);
      // child NL slots (created lazily by the reference) resolved serially; every child
      // block has exactly one parent key, so the tasks write disjoint blocks
      struct Dst {
        M* nl[2][2];
      };
      std::vector<Dst> dst(keys.size());
      for (size_t q = 0; q < keys.size(); ++q) {
        const Cluster& ci = T.clusters[keys[q].row];
        const Cluster& ck = T.clusters[keys[q].col];
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) {
            dst[q].nl[a][b] = nullptr;
            const int ic = ci.child[a], kc = ck.child[b];
            if (BT.kind(ic, kc).value() == BlockKind::subdivided) {
              M& slot = nl_[{ic, kc}];
              if (slot.size() == 0) slot = M(kcr(ic), kcc(kc));
              dst[q].nl[a][b] = &slot;
            }
          }
      }
      pfor(keys.size(), [&](std::int64_t q) {
        const BlockKey& key = keys[q];
        const M& s = nl_.at(key);
        const Cluster& ci = T.clusters[key.row];
        const Cluster& ck = T.clusters[key.col];
        const M& tr = C.row_basis.transfer[key.row];
        const M& tc = C.col_basis.transfer[key.col];
        Index ro = 0;
        for (int a = 0; a < 2; ++a) {
          const int ic = ci.child[a];
          const Index kr = kcr(ic);
          Index co = 0;
          for (int b = 0; b < 2; ++b) {
            const int kc = ck.child[b];
            const Index kk = kcc(kc);
            const M x = mm(Op::N, mm(tr.rows_range(ro, kr), s), Op::T, tc.rows_range(co, kk));
            switch (BT.kind(ic, kc).value()) {
              case BlockKind::admissible: C.coupling.at({ic, kc}) += x; break;
              case BlockKind::subdivided: *dst[q].nl[a][b] += x; break;
              case BlockKind::inadmissible_leaf:
                C.full.at({ic, kc}) += mm(Op::N, mm(C.row_basis.leaf[ic], x), Op::T, C.col_basis.leaf[kc]);
                break;
            }
            co += kk;
          }
          ro += kr;
        }
      });
      for (const BlockKey& key : keys) nl_.erase(key);
    }
  }

  const H2Matrix<S>& A;
  const H2Matrix<S>& B;
  const ClusterTree& T;
  const BlockTree& BT;
  double eps_;
  bool adaptive_;
  MmpOptions opt_;
  int threads_ = 1;
  std::vector<Tally> tl_;
  std::unique_ptr<Pool> pool_;
  H2Matrix<S> C;
  MmpReport rep_;
  std::vector<std::vector<std::pair<int, BlockKind>>> rows_, cols_;
  std::vector<int> pos_;
  std::vector<M> bp_, pa_, pb_;
  std::map<BlockKey, M> ca_, cb_, pending_, nl_, merged_, asm_a_, asm_b_;
  std::map<std::tuple<int, int, int>, M> ff_;
  std::int64_t ff_bytes_ = 0;
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
