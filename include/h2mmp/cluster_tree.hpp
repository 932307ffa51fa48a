// ClusterTree of proj/core/include/h2mmp/cluster_tree.hpp:12-48, same fields
// and semantics, built by the B200 library's host code (h2c_build_structure).
// The tree also owns the flat descriptor the C-ABI consumes, so every H2Matrix
// sharing this tree passes the same descriptor address (mmp.cpp:59 identity).
#pragma once

#include <array>
#include <cmath>
#include <algorithm>
#include <memory>
#include <vector>

#include "h2mmp/geometry.hpp"

namespace h2mmp {

struct Cluster {
  int id = -1;
  int parent = -1;
  int level = 0;
  int begin = 0;
  int end = 0;
  std::array<int, 2> child{-1, -1};
  std::array<double, 3> bbox_min{0, 0, 0};
  std::array<double, 3> bbox_max{0, 0, 0};
  bool is_leaf() const { return child[0] < 0; }
  int size() const { return end - begin; }
  double diameter() const {
    const double x = bbox_max[0] - bbox_min[0], y = bbox_max[1] - bbox_min[1], z = bbox_max[2] - bbox_min[2];
    return std::sqrt((x * x + y * y) + z * z);
  }
};

struct ClusterTree {
  std::vector<Cluster> clusters;
  std::vector<std::vector<int>> levels;
  std::vector<int> perm;
  std::vector<int> inv_perm;
  int depth = 0;
  int leafsize = 0;
  int size() const { return static_cast<int>(perm.size()); }
  const Cluster& root() const { return clusters.front(); }

  // ---- flat form for the C-ABI (filled by build_cluster_tree) ----
  std::vector<int32_t> f_parent, f_child0, f_child1, f_level, f_begin, f_end, f_perm;
  std::vector<double> f_bbox;
  std::vector<double> points;  // original points, kept for build_block_tree
  h2c_tree desc{};
};

namespace detail {
inline void tree_from_structure(const h2c_structure* s, ClusterTree& t) {
  h2c_tree d;
  h2c_structure_tree(s, &d);
  t.depth = d.depth;
  t.leafsize = d.leafsize;
  const int nc = d.n_clusters;
  t.f_parent.assign(d.parent, d.parent + nc);
  t.f_child0.assign(d.child0, d.child0 + nc);
  t.f_child1.assign(d.child1, d.child1 + nc);
  t.f_level.assign(d.level, d.level + nc);
  t.f_begin.assign(d.begin, d.begin + nc);
  t.f_end.assign(d.end, d.end + nc);
  t.f_bbox.assign(d.bbox, d.bbox + 6 * nc);
  t.f_perm.assign(d.perm, d.perm + d.n_points);
  t.clusters.resize(nc);
  for (int i = 0; i < nc; ++i) {
    Cluster& c = t.clusters[i];
    c.id = i;
    c.parent = d.parent[i];
    c.level = d.level[i];
    c.begin = d.begin[i];
    c.end = d.end[i];
    c.child = {d.child0[i], d.child1[i]};
    for (int a = 0; a < 3; ++a) {
      c.bbox_min[a] = d.bbox[6 * i + a];
      c.bbox_max[a] = d.bbox[6 * i + 3 + a];
    }
  }
  t.perm.assign(d.perm, d.perm + d.n_points);
  t.inv_perm.assign(d.n_points, 0);
  for (int i = 0; i < d.n_points; ++i) t.inv_perm[t.perm[i]] = i;
  t.levels.assign(t.depth + 1, {});
  for (const Cluster& c : t.clusters) t.levels[c.level].push_back(c.id);
  for (auto& lv : t.levels)
    std::sort(lv.begin(), lv.end(), [&](int a, int b) { return t.clusters[a].begin < t.clusters[b].begin; });
  t.desc = h2c_tree{d.n_points, d.depth, d.leafsize, nc, t.f_parent.data(), t.f_child0.data(), t.f_child1.data(),
                    t.f_level.data(), t.f_begin.data(), t.f_end.data(), t.f_bbox.data(), t.f_perm.data()};
}
}  // namespace detail

/// cluster_tree.cpp:66-93
inline ClusterTree build_cluster_tree(const PointSet& pts, int leafsize) {
  if (leafsize < 1) throw ConfigError("leafsize must be >= 1");
  if (pts.size() == 0) throw ConfigError("cannot build a cluster tree over no points");
  ClusterTree t;
  t.points.resize(3 * static_cast<size_t>(pts.size()));
  for (int i = 0; i < pts.size(); ++i)
    for (int a = 0; a < 3; ++a) t.points[3 * i + a] = pts.points[i][a];
  h2c_structure* s = h2c_build_structure(t.points.data(), pts.size(), leafsize, 1.0);
  if (!s) throw ConfigError(h2c_last_error(nullptr));
  detail::tree_from_structure(s, t);
  h2c_structure_free(s);
  return t;
}

inline double bbox_distance(const Cluster& t, const Cluster& s) {
  double g[3];
  for (int a = 0; a < 3; ++a) g[a] = std::max(std::max(t.bbox_min[a] - s.bbox_max[a], s.bbox_min[a] - t.bbox_max[a]), 0.0);
  return std::sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
}

inline bool is_admissible(const Cluster& t, const Cluster& s, double eta) {
  const double dist = bbox_distance(t, s);
  return dist > 0.0 && std::max(t.diameter(), s.diameter()) <= eta * dist;
}

}  // namespace h2mmp
