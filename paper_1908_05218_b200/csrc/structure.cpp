// Cluster tree and block tree builders of the drop-in API (host C++).
//
// Same rules as the reference so C's structure is identical:
//  - uniform depth d = min{d : ceil(N/2^d) <= leafsize}, longest bounding-box
//    axis, median split with ceil(size/2) points on the left, ties on the
//    coordinate broken by original index (cluster_tree.cpp:29-93);
//  - strong admissibility max(diam t, diam s) <= eta * gap(t, s) with a
//    positive gap (cluster_tree.cpp:95-109), recursive subdivision from
//    (root, root) (block_tree.cpp:9-53), blocks sorted by (row, col) per level,
//    C_sp over rows and columns per level.
#include "structure.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <unordered_map>

namespace h2b {

namespace {

double len3(double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); }

struct TB {
  const double* xyz;
  Structure& S;
  int depth;

  int make(int begin, int end, int level, int parent) {
    const int id = static_cast<int>(S.parent.size());
    S.parent.push_back(parent);
    S.child0.push_back(-1);
    S.child1.push_back(-1);
    S.level.push_back(level);
    S.begin.push_back(begin);
    S.end.push_back(end);
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = xyz[3 * S.perm[begin] + a];
    for (int p = begin; p < end; ++p)
      for (int a = 0; a < 3; ++a) {
        const double v = xyz[3 * S.perm[p] + a];
        lo[a] = std::min(lo[a], v);
        hi[a] = std::max(hi[a], v);
      }
    for (int a = 0; a < 3; ++a) S.bbox.push_back(lo[a]);
    for (int a = 0; a < 3; ++a) S.bbox.push_back(hi[a]);
    if (level >= depth) return id;
    const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    int axis = 0;
    if (ext[1] > ext[0]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    std::sort(S.perm.begin() + begin, S.perm.begin() + end, [&](int a, int b) {
      const double pa = xyz[3 * a + axis], pb = xyz[3 * b + axis];
      return pa < pb || (pa == pb && a < b);
    });
    const int mid = begin + (end - begin + 1) / 2;
    const int l = make(begin, mid, level + 1, id);
    const int r = make(mid, end, level + 1, id);
    S.child0[id] = l;
    S.child1[id] = r;
    return id;
  }
};

struct BB {
  Structure& S;
  double eta;
  std::vector<std::vector<std::tuple<int, int, uint8_t>>> lv;

  double diam(int c) const {
    const double* b = &S.bbox[6 * c];
    return len3(b[3] - b[0], b[4] - b[1], b[5] - b[2]);
  }
  bool admissible(int t, int s) const {
    const double* a = &S.bbox[6 * t];
    const double* b = &S.bbox[6 * s];
    double g[3];
    for (int k = 0; k < 3; ++k) g[k] = std::max(std::max(a[k] - b[k + 3], b[k] - a[k + 3]), 0.0);
    const double dist = len3(g[0], g[1], g[2]);
    return dist > 0.0 && std::max(diam(t), diam(s)) <= eta * dist;
  }
  void sub(int t, int s) {
    uint8_t k;
    const bool lt = S.child0[t] < 0, ls = S.child0[s] < 0;
    if (admissible(t, s)) k = H2C_ADMISSIBLE;
    else if (lt && ls) k = H2C_INADMISSIBLE_LEAF;
    else k = H2C_SUBDIVIDED;
    lv[S.level[t]].push_back({t, s, k});
    if (k != H2C_SUBDIVIDED) return;
    if (lt || ls) throw std::logic_error("uneven block subdivision; trees are not level-uniform");
    for (int a : {S.child0[t], S.child1[t]})
      for (int b : {S.child0[s], S.child1[s]}) sub(a, b);
  }
};

}  // namespace

std::unique_ptr<Structure> build_structure(const double* xyz, int n, int leafsize, double eta) {
  if (leafsize < 1) throw std::invalid_argument("leafsize must be >= 1");
  if (n < 1) throw std::invalid_argument("cannot build a cluster tree over no points");
  if (eta <= 0) throw std::invalid_argument("eta must be positive");
  auto S = std::make_unique<Structure>();
  S->n_points = n;
  S->leafsize = leafsize;
  S->perm.resize(n);
  std::iota(S->perm.begin(), S->perm.end(), 0);
  int depth = 0;
  while ((n + (1 << depth) - 1) / (1 << depth) > leafsize) ++depth;
  S->depth = depth;
  TB tb{xyz, *S, depth};
  tb.make(0, n, 0, -1);
  BB bb{*S, eta, {}};
  bb.lv.resize(depth + 1);
  bb.sub(0, 0);
  S->eta = eta;
  S->level_ptr.push_back(0);
  S->c_sp = 0;
  for (auto& L : bb.lv) {
    std::sort(L.begin(), L.end());
    std::unordered_map<int, int> pr, pc;
    for (const auto& [t, s, k] : L) {
      S->row.push_back(t);
      S->col.push_back(s);
      S->kind.push_back(k);
      S->c_sp = std::max({S->c_sp, ++pr[t], ++pc[s]});
    }
    S->level_ptr.push_back(static_cast<int64_t>(S->row.size()));
  }
  return S;
}

void Structure::tree_desc(h2c_tree* d) const {
  d->n_points = n_points;
  d->depth = depth;
  d->leafsize = leafsize;
  d->n_clusters = static_cast<int32_t>(parent.size());
  d->parent = parent.data();
  d->child0 = child0.data();
  d->child1 = child1.data();
  d->level = level.data();
  d->begin = begin.data();
  d->end = end.data();
  d->bbox = bbox.data();
  d->perm = perm.data();
}

void Structure::blocks_desc(h2c_blocks* d) const {
  d->depth = depth;
  d->c_sp = c_sp;
  d->eta = eta;
  d->n_blocks = static_cast<int64_t>(row.size());
  d->level_ptr = level_ptr.data();
  d->row = row.data();
  d->col = col.data();
  d->kind = kind.data();
}

// block_tree.cpp:61-85 over cluster ids, with a per-call hash of the blocks
int target_status(const h2c_tree& t, const h2c_blocks& b, int ti, int si) {
  std::unordered_map<int64_t, uint8_t> kind;
  kind.reserve(static_cast<size_t>(b.n_blocks) * 2);
  for (int64_t k = 0; k < b.n_blocks; ++k) kind[(int64_t(b.row[k]) << 32) | uint32_t(b.col[k])] = b.kind[k];
  for (int x = ti, y = si; x >= 0 && y >= 0; x = t.parent[x], y = t.parent[y]) {
    auto it = kind.find((int64_t(x) << 32) | uint32_t(y));
    if (it == kind.end()) continue;
    if (x != ti) {
      if (it->second != H2C_ADMISSIBLE) throw std::logic_error("cluster pair below a non-admissible block");
      return 3;
    }
    return it->second == H2C_ADMISSIBLE ? 1 : (it->second == H2C_INADMISSIBLE_LEAF ? 0 : 2);
  }
  throw std::logic_error("cluster pair not covered by the block tree");
}

}  // namespace h2b
