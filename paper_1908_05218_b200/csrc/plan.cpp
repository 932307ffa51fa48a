// Structure plan builder (see plan.hpp).  Host C++, multi-threaded over rows.
#include "plan.hpp"

#include <algorithm>
#include <mutex>
#include <exception>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <stdexcept>
#include <string>
#include <thread>

namespace h2b {

namespace {

struct InvariantError : std::logic_error {
  using std::logic_error::logic_error;
};

template <class F>
void parallel_for(int n, int threads, F&& f) {
  threads = std::max(1, std::min(threads, n));
  if (threads <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex em;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      try {
        for (;;) {
          const int i = next.fetch_add(1);
          if (i >= n) break;
          f(i);
        }
      } catch (...) {  // rethrown on the calling thread (structure errors -> C-ABI error codes)
        std::lock_guard<std::mutex> g(em);
        if (!err) err = std::current_exception();
        next = n;
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

enum Status : uint8_t { kFullTarget = 0, kAdmTarget = 1, kSubTarget = 2, kInside = 3 };

struct Triple {
  int32_t k, j, a, b;  // target column, middle, A block, B block
};

// one row's triples, sorted by (k, j)
struct RowTriples {
  std::vector<Triple> t;
};

int find_block(const LevelPlan& L, int i, int k) {
  const int32_t* b = L.bcol.data() + L.row_ptr[i];
  const int32_t* e = L.bcol.data() + L.row_ptr[i + 1];
  const int32_t* it = std::lower_bound(b, e, k);
  if (it != e && *it == k) return L.row_ptr[i] + static_cast<int>(it - b);
  return -1;
}

// block_tree.cpp:61-85 restated over level positions: parent of position p is
// p >> 1 (complete binary tree of uniform depth, children at 2p and 2p+1).
Status status_of(const std::vector<LevelPlan>& lv, int l, int i, int k) {
  int a = i, c = k;
  for (int m = l; m >= 0; --m, a >>= 1, c >>= 1) {
    const int b = find_block(lv[m], a, c);
    if (b < 0) continue;
    const uint8_t kind = lv[m].bkind[b];
    if (m != l) {
      if (kind != kAdm) throw InvariantError("cluster pair below a non-admissible block");
      return kInside;
    }
    return kind == kAdm ? kAdmTarget : (kind == kFull ? kFullTarget : kSubTarget);
  }
  throw InvariantError("cluster pair not covered by the block tree");
}

void finish_csr(Csr& c, int n_out, const std::vector<int32_t>& owner) {
  // owner[e] = output of entry e; entries already in the wanted per-output order
  if (owner.size() > size_t(INT32_MAX))  // row pointers are int32 on the device
    throw std::length_error("structure plan: " + std::to_string(owner.size()) +
                            " entries in one CSR list exceed the int32 index range");
  c.ptr.assign(n_out + 1, 0);
  for (int32_t o : owner) c.ptr[o + 1]++;
  for (int o = 0; o < n_out; ++o) c.ptr[o + 1] += c.ptr[o];
  std::vector<int32_t> li(c.li.size()), ri(c.ri.size()), fill(c.ptr.begin(), c.ptr.end() - 1);
  for (size_t e = 0; e < owner.size(); ++e) {
    const int32_t at = fill[owner[e]]++;
    li[at] = c.li[e];
    ri[at] = c.ri[e];
  }
  c.li.swap(li);
  c.ri.swap(ri);
}

struct Builder {
  Csr csr;
  std::vector<int32_t> owner;
  void add(int32_t o, int32_t l, int32_t r) {
    owner.push_back(o);
    csr.li.push_back(l);
    csr.ri.push_back(r);
  }
  void append(const Builder& b) {
    owner.insert(owner.end(), b.owner.begin(), b.owner.end());
    csr.li.insert(csr.li.end(), b.csr.li.begin(), b.csr.li.end());
    csr.ri.insert(csr.ri.end(), b.csr.ri.begin(), b.csr.ri.end());
  }
  Csr done(int n_out) {
    finish_csr(csr, n_out, owner);
    owner.clear();
    return std::move(csr);
  }
};

}  // namespace

Plan build_plan(const h2c_tree& tree, const h2c_blocks& blocks, int threads) {
  const auto t0 = std::chrono::steady_clock::now();
  Plan P;
  P.depth = tree.depth;
  P.n_points = tree.n_points;
  P.n_clusters = tree.n_clusters;
  const int D = tree.depth;
  if (blocks.depth != D) throw std::invalid_argument("block structure depth does not match the tree");
  P.lv.resize(D + 1);
  P.pos_of.assign(tree.n_clusters, -1);

  // ---- level positions (ordered by begin, cluster_tree.cpp:90-92)
  for (int id = 0; id < tree.n_clusters; ++id) {
    const int l = tree.level[id];
    if (l < 0 || l > D) throw std::invalid_argument("cluster level out of range");
    P.lv[l].id.push_back(id);
  }
  for (int l = 0; l <= D; ++l) {
    LevelPlan& L = P.lv[l];
    L.level = l;
    std::sort(L.id.begin(), L.id.end(), [&](int a, int b) { return tree.begin[a] < tree.begin[b]; });
    L.n = static_cast<int>(L.id.size());
    if (L.n != (1 << l)) throw std::invalid_argument("cluster tree is not a complete binary tree of uniform depth");
    L.size.resize(L.n);
    for (int p = 0; p < L.n; ++p) {
      P.pos_of[L.id[p]] = p;
      L.size[p] = tree.end[L.id[p]] - tree.begin[L.id[p]];
    }
  }
  for (int l = 0; l < D; ++l)
    for (int p = 0; p < P.lv[l].n; ++p) {
      const int id = P.lv[l].id[p];
      if (P.pos_of[tree.child0[id]] != 2 * p || P.pos_of[tree.child1[id]] != 2 * p + 1)
        throw std::invalid_argument("children are not at positions 2p, 2p+1");
    }

  // ---- blocks per level, (row, col) order, kind-local indices, CSRs
  for (int l = 0; l <= D; ++l) {
    LevelPlan& L = P.lv[l];
    std::vector<int64_t> g;
    for (int64_t b = blocks.level_ptr[l]; b < blocks.level_ptr[l + 1]; ++b) g.push_back(b);
    std::sort(g.begin(), g.end(), [&](int64_t a, int64_t b) {
      const int ra = P.pos_of[blocks.row[a]], rb = P.pos_of[blocks.row[b]];
      return ra < rb || (ra == rb && P.pos_of[blocks.col[a]] < P.pos_of[blocks.col[b]]);
    });
    const int nb = static_cast<int>(g.size());
    L.bglobal = g;
    L.brow.resize(nb);
    L.bcol.resize(nb);
    L.bkind.resize(nb);
    L.kidx.resize(nb);
    for (int b = 0; b < nb; ++b) {
      L.brow[b] = P.pos_of[blocks.row[g[b]]];
      L.bcol[b] = P.pos_of[blocks.col[g[b]]];
      if (tree.level[blocks.row[g[b]]] != l || tree.level[blocks.col[g[b]]] != l)
        throw std::invalid_argument("block pairs clusters of another level");
      L.bkind[b] = blocks.kind[g[b]];
      if (L.bkind[b] == kAdm) {
        L.kidx[b] = static_cast<int32_t>(L.adm.size());
        L.adm.push_back(b);
      } else {
        if ((L.bkind[b] == kFull) != (l == D))
          throw std::invalid_argument("inadmissible leaves only at the leaf level, subdivided blocks above");
        L.kidx[b] = static_cast<int32_t>(L.nearb.size());
        L.nearb.push_back(b);
      }
    }
    L.row_ptr.assign(L.n + 1, 0);
    L.col_ptr.assign(L.n + 1, 0);
    for (int b = 0; b < nb; ++b) {
      L.row_ptr[L.brow[b] + 1]++;
      L.col_ptr[L.bcol[b] + 1]++;
    }
    for (int p = 0; p < L.n; ++p) {
      L.row_ptr[p + 1] += L.row_ptr[p];
      L.col_ptr[p + 1] += L.col_ptr[p];
    }
    L.col_blk.resize(nb);
    std::vector<int32_t> fill(L.col_ptr.begin(), L.col_ptr.end() - 1);
    for (int b = 0; b < nb; ++b) L.col_blk[fill[L.bcol[b]]++] = b;  // rows ascending within a column
  }

  const bool trace = std::getenv("H2B_PLAN_TRACE") != nullptr;
  auto stamp = [&](const char* what) {
    if (trace)
      std::fprintf(stderr, "[plan] %-28s %.3f s\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  };
  stamp("levels + blocks");
  // ---- pass 1 (bottom-up): triples per level, pending and merged sets
  std::vector<std::vector<RowTriples>> rows(D + 1);
  std::vector<std::vector<std::pair<int, int>>> pend(D + 1);  // (row, col) pending pairs
  std::vector<std::vector<uint8_t>> trip_status(D + 1);
  for (int l = D; l >= 1 || (l == 0 && D == 0); --l) {
    LevelPlan& L = P.lv[l];
    const bool leaf = l == D;
    rows[l].resize(L.n);
    parallel_for(L.n, threads, [&](int i) {
      // bucket (counting) sort by target column k: row i's blocks come in ascending j, so each
      // bucket fills in ascending j — the (k, j) order without sorting the triples themselves
      thread_local std::vector<int32_t> at;
      thread_local std::vector<int32_t> touched;
      if (at.size() < size_t(L.n)) at.assign(L.n, 0);
      touched.clear();
      auto each = [&](auto&& f) {
        for (int ba = L.row_ptr[i]; ba < L.row_ptr[i + 1]; ++ba) {
          const int j = L.bcol[ba];
          for (int bb = L.row_ptr[j]; bb < L.row_ptr[j + 1]; ++bb) {
            if (!leaf && L.bkind[ba] == kSub && L.bkind[bb] == kSub) continue;  // mmp.cpp:593
            f(L.bcol[bb], j, ba, bb);
          }
        }
      };
      each([&](int k, int, int, int) {
        if (at[k]++ == 0) touched.push_back(k);
      });
      std::sort(touched.begin(), touched.end());
      int32_t total = 0;
      for (int k : touched) {
        const int32_t c = at[k];
        at[k] = total;
        total += c;
      }
      auto& out = rows[l][i].t;
      out.resize(total);
      each([&](int k, int j, int ba, int bb) { out[at[k]++] = {k, j, ba, bb}; });
      for (int k : touched) at[k] = 0;
    });
    // case counters (mmp.cpp:307-308, 594-595), per row in parallel
    std::vector<std::array<int64_t, 4>> cc(L.n);
    parallel_for(L.n, threads, [&](int i) {
      cc[i] = {0, 0, 0, 0};
      for (const Triple& t : rows[l][i].t) {
        const bool fa = L.bkind[t.a] != kAdm, fb = L.bkind[t.b] != kAdm;
        cc[i][leaf ? (fa ? (fb ? 0 : 1) : (fb ? 2 : 3)) : (fa ? 1 : (fb ? 2 : 3))]++;
      }
    });
    for (int i = 0; i < L.n; ++i)
      for (int c = 0; c < 4; ++c) {
        L.case_products[c] += cc[i][c];
        P.total_triples += cc[i][c];
      }
    // pending candidates from triples (per row in parallel, concatenated in row order)
    std::vector<std::vector<std::pair<int, int>>> cand_row(L.n);
    std::atomic<bool> full_target{false};
    parallel_for(L.n, threads, [&](int i) {
      int last = -1;
      for (const Triple& t : rows[l][i].t) {
        if (t.k == last) continue;
        last = t.k;
        const Status s = status_of(P.lv, l, i, t.k);
        if (s == kInside) cand_row[i].push_back({i, t.k});
        if (!leaf && s == kFullTarget) full_target = true;
      }
    });
    if (full_target) throw InvariantError("mmp: coupling contribution aimed at a full block");
    std::vector<std::pair<int, int>> cand;
    for (auto& v : cand_row) cand.insert(cand.end(), v.begin(), v.end());
    cand_row.clear();
    // merged pairs of the children's pending couplings (mmp.cpp:344-365)
    if (!leaf) {
      const LevelPlan& C = P.lv[l + 1];
      (void)C;
      std::vector<std::pair<int, int>> par;
      for (const auto& [ci, ck] : pend[l + 1]) par.push_back({ci >> 1, ck >> 1});
      std::sort(par.begin(), par.end());
      par.erase(std::unique(par.begin(), par.end()), par.end());
      L.merged_row.resize(par.size());
      L.merged_col.resize(par.size());
      L.merged_quad.assign(4 * par.size(), -1);
      for (size_t m = 0; m < par.size(); ++m) {
        L.merged_row[m] = par[m].first;
        L.merged_col[m] = par[m].second;
        const Status s = status_of(P.lv, l, par[m].first, par[m].second);
        if (s != kAdmTarget && s != kInside)
          throw InvariantError("mmp: merged coupling with an impossible target");
        if (s == kInside) cand.push_back(par[m]);
      }
      LevelPlan& Ch = P.lv[l + 1];
      Ch.pend_mq.assign(pend[l + 1].size(), -1);
      for (size_t q = 0; q < pend[l + 1].size(); ++q) {
        const auto [ci, ck] = pend[l + 1][q];
        const auto it = std::lower_bound(par.begin(), par.end(), std::make_pair(ci >> 1, ck >> 1));
        const int32_t mq = static_cast<int32_t>(4 * (it - par.begin()) + 2 * (ci & 1) + (ck & 1));
        L.merged_quad[mq] = static_cast<int32_t>(q);
        Ch.pend_mq[q] = mq;
      }
    }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    pend[l] = cand;
    L.pend_row.resize(cand.size());
    L.pend_col.resize(cand.size());
    for (size_t q = 0; q < cand.size(); ++q) {
      L.pend_row[q] = cand[q].first;
      L.pend_col[q] = cand[q].second;
    }
    if (l == 0) break;
  }
  if (D > 0 && !pend[1].empty())
    throw InvariantError("mmp: pending couplings left after the bottom-up pass");

  stamp("pass 1 (triples, pending)");
  // ---- pass 2 (top-down): which subdivided blocks hold NL couplings
  for (int l = 1; l < D; ++l) {
    LevelPlan& L = P.lv[l];
    std::vector<uint8_t> has(L.brow.size(), 0);
    parallel_for(L.n, threads, [&](int i) {  // block (i, k) belongs to row i: rows write disjoint flags
      int last = -1;
      for (const Triple& t : rows[l][i].t) {
        if (t.k == last) continue;
        last = t.k;
        if (status_of(P.lv, l, i, t.k) == kSubTarget) has[find_block(L, i, t.k)] = 1;
      }
    });
    if (l > 1) {  // children of the parent level's NL blocks (mmp.cpp:641-645)
      const LevelPlan& U = P.lv[l - 1];
      for (int32_t b : U.nl_block)
        for (int q = 0; q < 4; ++q) {
          const int cb = find_block(L, 2 * U.brow[b] + (q >> 1), 2 * U.bcol[b] + (q & 1));
          if (cb >= 0 && L.bkind[cb] == kSub) has[cb] = 1;
        }
    }
    L.nl_of_block.assign(L.brow.size(), -1);
    for (size_t b = 0; b < has.size(); ++b)
      if (has[b]) {
        L.nl_of_block[b] = static_cast<int32_t>(L.nl_block.size());
        L.nl_block.push_back(static_cast<int32_t>(b));
      }
  }
  for (int l = 0; l <= D; ++l)
    if (P.lv[l].nl_of_block.empty()) P.lv[l].nl_of_block.assign(P.lv[l].brow.size(), -1);

  stamp("pass 2 (NL blocks)");
  // ---- pass 3: CSRs with final target numbering
  for (int l = D; l >= 1 || (l == 0 && D == 0); --l) {
    LevelPlan& L = P.lv[l];
    const bool leaf = l == D;
    const int na = static_cast<int>(L.adm.size());
    const int np = static_cast<int>(L.pend_row.size());
    const int nt = L.n_targets();
    L.target_row.resize(nt);
    L.target_col.resize(nt);
    for (int a = 0; a < na; ++a) {
      L.target_row[a] = L.brow[L.adm[a]];
      L.target_col[a] = L.bcol[L.adm[a]];
    }
    for (int q = 0; q < np; ++q) {
      L.target_row[na + q] = L.pend_row[q];
      L.target_col[na + q] = L.pend_col[q];
    }
    for (size_t q = 0; q < L.nl_block.size(); ++q) {
      L.target_row[na + np + q] = L.brow[L.nl_block[q]];
      L.target_col[na + np + q] = L.bcol[L.nl_block[q]];
    }
    auto slot_of = [&](int i, int k, Status s) -> int {
      if (s == kAdmTarget) return L.kidx[find_block(L, i, k)];
      if (s == kInside) {
        const auto it = std::lower_bound(pend[l].begin(), pend[l].end(), std::make_pair(i, k));
        return na + static_cast<int>(it - pend[l].begin());
      }
      if (s == kSubTarget) return na + np + L.nl_of_block[find_block(L, i, k)];
      return -1;
    };
    const int nnear = static_cast<int>(L.nearb.size());
    // rows in T contiguous chunks with private builders, concatenated in chunk (= row) order:
    // the entries of every output come from its own row, so the lists equal the serial ones
    struct Part {
      Builder ly, lyr, lyn, xr, ww, ff, fr, rf, rr, hq;
      std::vector<std::array<int, 3>> hqc;  // (B near, i, A near)
    };
    const int T = std::max(1, std::min(threads, L.n));
    std::vector<Part> parts(T);
    parallel_for(T, T, [&](int pt) {
      Part& Pt = parts[pt];
      const int i0 = static_cast<int>(int64_t(L.n) * pt / T), i1 = static_cast<int>(int64_t(L.n) * (pt + 1) / T);
      for (int i = i0; i < i1; ++i) {
        const auto& tr = rows[l][i].t;
        size_t s0 = 0;
        while (s0 < tr.size()) {
          size_t s1 = s0;
          while (s1 < tr.size() && tr[s1].k == tr[s0].k) ++s1;
          const int k = tr[s0].k;
          const Status st = status_of(P.lv, l, i, k);
          if (st == kFullTarget) {
            const int o = L.kidx[find_block(L, i, k)];
            for (size_t e = s0; e < s1; ++e) {
              const Triple& t = tr[e];
              const bool fa = L.bkind[t.a] == kFull, fb = L.bkind[t.b] == kFull;
              if (fa && fb) Pt.ff.add(o, L.kidx[t.a], L.kidx[t.b]);
              else if (fa) Pt.fr.add(o, L.kidx[t.a], L.kidx[t.b]);
              else if (fb) Pt.rf.add(o, L.kidx[t.a], L.kidx[t.b]);
              else Pt.rr.add(o, L.kidx[t.a], L.kidx[t.b]);
            }
          } else {
            const int o = slot_of(i, k, st);
            for (size_t e = s0; e < s1; ++e) {
              const Triple& t = tr[e];
              const bool ra = L.bkind[t.a] == kAdm, rb = L.bkind[t.b] == kAdm;
              if (rb) {
                Pt.ly.add(o, t.a, L.kidx[t.b]);
                if (ra) Pt.lyr.add(o, L.kidx[t.a], L.kidx[t.b]);
                else Pt.lyn.add(o, t.a, L.kidx[t.b]);
              }
              else if (ra) Pt.xr.add(o, L.kidx[t.a], t.b);
              else {  // full x full at the leaf level (NL x NL never reaches here)
                Pt.ww.add(o, L.kidx[t.a], L.kidx[t.b]);
                if (st == kAdmTarget || st == kInside) {
                  Pt.hq.add(L.kidx[t.a], L.kidx[t.b], 0);
                  Pt.hqc.push_back({L.kidx[t.b], i, L.kidx[t.a]});
                }
              }
            }
          }
          s0 = s1;
        }
      }
    });
    if (trace) stamp("    parts");
    Builder hqc;
    std::vector<std::vector<std::pair<int, int>>> hqc_rows;  // per B near: (i, A near)
    if (leaf) {
      hqc_rows.resize(nnear);
      for (Part& Pt : parts)
        for (const auto& h : Pt.hqc) hqc_rows[h[0]].push_back({h[1], h[2]});
    }
    // the ten lists: concatenated in row order and counting-sorted by output, one per thread
    Builder Part::*which[10] = {&Part::ly, &Part::lyr, &Part::lyn, &Part::xr, &Part::ww,
                                &Part::ff, &Part::fr, &Part::rf, &Part::rr, &Part::hq};
    Csr* dst[10] = {&L.ly, &L.lyr, &L.lyn, &L.xr, &L.ww, &L.ff, &L.fr, &L.rf, &L.rr, &L.hq};
    const int nout[10] = {nt, nt, nt, nt, nt, nnear, nnear, nnear, nnear, nnear};
    // Every list but hq is owned by targets numbered in (row, col) order inside three ranges
    // (admissible, pending, NL; one range for the full-target lists), and every target's entries
    // come from its own row, i.e. from one part: each part copies its entries of range c straight
    // to the final position (ranges in order, parts in row order inside a range) and counts its
    // own targets' row pointers — no concatenation, no sort, parallel over parts.
    for (int w = 0; w < (leaf ? 9 : 5); ++w) {
      const int no = nout[w];
      const int c0 = w < 5 ? na : no, c1 = w < 5 ? na + np : no;
      auto cat = [&](int32_t o) { return o < c0 ? 0 : (o < c1 ? 1 : 2); };
      std::vector<std::array<size_t, 3>> cnt(T);
      parallel_for(T, threads, [&](int pt) {
        cnt[pt] = {0, 0, 0};
        for (int32_t o : (parts[pt].*which[w]).owner) cnt[pt][cat(o)]++;
      });
      std::vector<std::array<size_t, 3>> at(T);
      size_t run = 0;
      for (int c = 0; c < 3; ++c)
        for (int pt = 0; pt < T; ++pt) {
          at[pt][c] = run;
          run += cnt[pt][c];
        }
      if (run > size_t(INT32_MAX))
        throw std::length_error("structure plan: " + std::to_string(run) +
                                " entries in one CSR list exceed the int32 index range");
      Csr& out = *dst[w];
      out.li.resize(run);
      out.ri.resize(run);
      out.ptr.assign(no + 1, 0);
      parallel_for(T, threads, [&](int pt) {
        Builder& B = parts[pt].*which[w];
        auto pos = at[pt];
        for (size_t e = 0; e < B.owner.size(); ++e) {
          const size_t d = pos[cat(B.owner[e])]++;
          out.li[d] = B.csr.li[e];
          out.ri[d] = B.csr.ri[e];
          out.ptr[B.owner[e] + 1]++;  // the target's entries all come from this part
        }
        B = Builder{};
      });
      for (int o = 0; o < no; ++o) out.ptr[o + 1] += out.ptr[o];
    }
    if (leaf) {  // hq is owned by A's near block (i, j): not ordered along the rows -> general sort
      Builder all;
      for (Part& Pt : parts) {
        all.append(Pt.hq);
        Pt.hq = Builder{};
      }
      L.hq = all.done(nnear);
    }
    parts.clear();
    if (trace) {
      stamp("    lists");
      for (int w = 0; w < (leaf ? 10 : 5); ++w) std::fprintf(stderr, "      list %d: %zu entries\n", w, dst[w]->li.size());
    }
    if (leaf) {
      // hq entries per A near block were added in (i, k asc, j asc) order:
      // per (i,j) the k's are ascending
      for (int b = 0; b < nnear; ++b) {
        auto& v = hqc_rows[b];
        std::sort(v.begin(), v.end());
        for (const auto& [i, an] : v) hqc.add(b, an, 0);
      }
      L.hqc = hqc.done(nnear);
    }
    if (trace && leaf) stamp("  leaf hqc");
    // per-cluster near blocks by row / column (block order)
    {
      Builder rn, cn;
      for (int b : L.nearb) rn.add(L.brow[b], L.kidx[b], L.kidx[b]);
      for (int p = 0; p < L.n; ++p)
        for (int c = L.col_ptr[p]; c < L.col_ptr[p + 1]; ++c) {
          const int b = L.col_blk[c];
          if (L.bkind[b] != kAdm) cn.add(p, L.kidx[b], L.kidx[b]);
        }
      L.row_near = rn.done(L.n);
      L.col_near = cn.done(L.n);
    }
    if (trace) stamp("    near");
    if (!leaf) {
      const int nm = static_cast<int>(L.merged_row.size());
      L.merged_target.resize(nm);
      Builder mg, rm, cm;
      parallel_for(nm, threads, [&](int m) {
        const Status s = status_of(P.lv, l, L.merged_row[m], L.merged_col[m]);
        L.merged_target[m] = slot_of(L.merged_row[m], L.merged_col[m], s);
      });
      for (int m = 0; m < nm; ++m) {
        mg.add(L.merged_target[m], m, L.merged_col[m]);
        rm.add(L.merged_row[m], m, m);
      }
      // merged by column, rows ascending
      std::vector<int> idx(nm);
      for (int m = 0; m < nm; ++m) idx[m] = m;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return L.merged_col[a] < L.merged_col[b]; });
      for (int m : idx) cm.add(L.merged_col[m], m, m);
      L.mg = mg.done(nt);
      const int na_ = static_cast<int>(L.adm.size()), np_ = static_cast<int>(L.pend_row.size());
      for (int m = 0; m < nm; ++m) {
        const int t = L.merged_target[m];
        const bool adm_t = t < na_;
        if (!adm_t && t >= na_ + np_) throw InvariantError("mmp: merged coupling into a non-leaf target");
        LevelPlan::MergedInto& z = adm_t ? L.mz_adm : L.mz_pend;
        z.row.push_back(L.merged_row[m]);
        z.col.push_back(L.merged_col[m]);
        z.m.push_back(m);
        z.out.push_back(adm_t ? t : L.pend_mq[t - na_]);
      }
      L.row_merged = rm.done(L.n);
      L.col_merged = cm.done(L.n);
      if (trace) stamp("    merged");
      // children of subdivided blocks
      const LevelPlan& C = P.lv[l + 1];
      L.sub_child.assign(4 * nnear, -1);
      for (int s = 0; s < nnear; ++s) {
        const int b = L.nearb[s];
        for (int q = 0; q < 4; ++q) {
          const int cb = find_block(C, 2 * L.brow[b] + (q >> 1), 2 * L.bcol[b] + (q & 1));
          if (cb < 0) throw InvariantError("subdivided block without its four children");
          L.sub_child[4 * s + q] = cb;
        }
      }
      // split lists (mmp.cpp:617-659)
      for (size_t q = 0; q < L.nl_block.size(); ++q) {
        const int b = L.nl_block[q];
        for (int s = 0; s < 4; ++s) {
          L.split_src[s].push_back(static_cast<int32_t>(q));
          L.split_dst[s].push_back(L.sub_child[4 * L.kidx[b] + s]);
        }
      }
    }
    rows[l].clear();
    rows[l].shrink_to_fit();
    if (trace) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "  level %d done", l);
      stamp(buf);
    }
    if (l == 0) break;
  }
  stamp("pass 3 (CSRs)");
  P.build_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return P;
}

}  // namespace h2b
