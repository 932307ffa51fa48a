// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// Restatement of the reference's input side of the MMP path: geometry
// generators (geometry.cpp), dense kernel assembly, the uniform-depth
// bisection cluster tree (cluster_tree.cpp) and the strong-admissibility
// block tree with target classification (block_tree.cpp).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <string>

#include "model.hpp"

namespace h2o {

// ---------------------------------------------------------------------------
// geometry.cpp:39-52 — points uniform in [0,1)^3 from mt19937_64, 53-bit
// mantissa conversion so the stream is library independent.
static PointSet random_cloud(const GeometrySpec& g) {
  PointSet out;
  std::mt19937_64 eng(g.seed);
  auto u01 = [&eng] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  out.points.reserve(g.n);
  for (int i = 0; i < g.n; ++i) {
    Vec3 p;
    p.x = u01();
    p.y = u01();
    p.z = u01();
    out.points.push_back(p);
  }
  return out;
}

// geometry.cpp:12-17,54-95 — two crossing layers of square-section bars,
// lateral surface sampled on a (axial station) x (perimeter point) lattice.
static PointSet bus(const GeometrySpec& g) {
  const int m = g.bus_count, d = g.samples_per_meter;
  const double len = 2.0 * m + 1.0;
  const int stations = std::max(1, static_cast<int>(std::lround(len * d)));
  const int ring = 4 * std::max(1, d);
  auto perimeter = [](double u, double& a, double& b) {
    if (u < 1.0) { a = u; b = 0.0; }
    else if (u < 2.0) { a = 1.0; b = u - 1.0; }
    else if (u < 3.0) { a = 3.0 - u; b = 1.0; }
    else { a = 0.0; b = 4.0 - u; }
  };
  PointSet out;
  for (int layer = 0; layer < 2; ++layer)
    for (int c = 0; c < m; ++c)
      for (int i = 0; i < stations; ++i) {
        const double ax = (i + 0.5) / stations * len;
        for (int j = 0; j < ring; ++j) {
          double a, b;
          perimeter((j + 0.5) / ring * 4.0, a, b);
          Vec3 p;
          if (layer == 0) { p.x = ax; p.y = 2.0 * c + a; p.z = b; }
          else { p.x = 2.0 * c + a; p.y = ax; p.z = 2.0 + b; }
          out.points.push_back(p);
        }
      }
  return out;
}

// geometry.cpp:97-107
static PointSet slab(const GeometrySpec& g) {
  PointSet out;
  for (int ix = 0; ix < g.slab_width; ++ix)
    for (int iy = 0; iy < g.slab_width; ++iy)
      for (int iz = 0; iz < g.slab_thickness; ++iz) out.points.push_back({ix * 0.1, iy * 0.1, iz * 0.1});
  return out;
}

// geometry.cpp:109-137
static PointSet cube_array(const GeometrySpec& g) {
  const double edge = 0.3, pitch = 0.6;
  const int a = g.array_edge, q = g.cube_points;
  const double step = q > 1 ? edge / (q - 1) : 0.0;
  const double center = q > 1 ? 0.0 : edge / 2.0;
  PointSet out;
  for (int cx = 0; cx < a; ++cx)
    for (int cy = 0; cy < a; ++cy)
      for (int cz = 0; cz < a; ++cz)
        for (int ix = 0; ix < q; ++ix)
          for (int iy = 0; iy < q; ++iy)
            for (int iz = 0; iz < q; ++iz)
              out.points.push_back({cx * pitch + (center + ix * step),
                                    cy * pitch + (center + iy * step),
                                    cz * pitch + (center + iz * step)});
  return out;
}

PointSet generate_geometry(const GeometrySpec& g) {
  switch (g.family) {
    case Family::random_cloud:
      if (g.n < 1) throw ConfigError("random_cloud: n must be positive");
      return random_cloud(g);
    case Family::bus:
      if (g.bus_count < 1 || g.samples_per_meter < 1) throw ConfigError("bus: bad parameters");
      return bus(g);
    case Family::slab:
      if (g.slab_width < 1 || g.slab_thickness < 1) throw ConfigError("slab: bad parameters");
      return slab(g);
    case Family::cube_array:
      if (g.array_edge < 1 || g.cube_points < 1) throw ConfigError("cube_array: bad parameters");
      return cube_array(g);
  }
  throw ConfigError("unknown geometry family");
}

// geometry.cpp:185-233 — 1/r or exp(i k r)/r off the diagonal; diagonal from
// the kernel or twice the largest first-row magnitude.
template <class S>
Mat<S> assemble_dense(const PointSet& pts, const Kernel& k) {
  const int n = pts.size();
  if (n == 0) throw ConfigError("assemble_dense: empty point set");
  if ((k.kind == KernelKind::laplace) != !is_complex_v<S>)
    throw ConfigError("kernel kind does not match the scalar type");
  Mat<S> out(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      const Vec3& a = pts.points[i];
      const Vec3& b = pts.points[j];
      const double r = norm3(a.x - b.x, a.y - b.y, a.z - b.z);
      if (r == 0.0) throw AssemblyError("duplicate points");
      if constexpr (is_complex_v<S>) out(i, j) = std::polar(1.0 / r, k.wavenumber * r);
      else out(i, j) = 1.0 / r;
    }
  double diag;
  if (k.diagonal_value) {
    diag = *k.diagonal_value;
  } else {
    double mx = 0.0;
    for (int j = 1; j < n; ++j) mx = std::max(mx, std::abs(out(0, j)));
    diag = 2.0 * mx;
  }
  for (int i = 0; i < n; ++i) out(i, i) = S(diag);
  return out;
}
template Mat<Real> assemble_dense<Real>(const PointSet&, const Kernel&);
template Mat<Complex> assemble_dense<Complex>(const PointSet&, const Kernel&);

// ---------------------------------------------------------------------------
// cluster_tree.cpp:12-93 — recursive longest-axis median bisection to the
// uniform depth d = min{d : ceil(N/2^d) <= leafsize}; ids in DFS pre-order;
// the left child receives ceil(size/2) points; ties on the split coordinate
// are broken by original index.
namespace {
struct TreeBuilder {
  const PointSet& pts;
  ClusterTree& t;
  int depth;

  void bbox(Cluster& c) {
    Vec3 lo = pts.points[t.perm[c.begin]], hi = lo;
    for (int p = c.begin; p < c.end; ++p) {
      const Vec3& x = pts.points[t.perm[p]];
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], x[a]);
        hi[a] = std::max(hi[a], x[a]);
      }
    }
    c.bbox_min = lo;
    c.bbox_max = hi;
  }

  int make(int begin, int end, int level, int parent) {
    const int id = static_cast<int>(t.clusters.size());
    Cluster c;
    c.id = id;
    c.parent = parent;
    c.level = level;
    c.begin = begin;
    c.end = end;
    bbox(c);
    t.clusters.push_back(c);
    if (level >= depth) return id;
    const Vec3 ext{c.bbox_max.x - c.bbox_min.x, c.bbox_max.y - c.bbox_min.y,
                   c.bbox_max.z - c.bbox_min.z};
    int axis = 0;
    if (ext.y > ext.x) axis = 1;
    if (ext.z > ext[axis]) axis = 2;
    std::sort(t.perm.begin() + begin, t.perm.begin() + end, [&](int a, int b) {
      const double pa = pts.points[a][axis], pb = pts.points[b][axis];
      return pa < pb || (pa == pb && a < b);
    });
    const int mid = begin + (end - begin + 1) / 2;
    const int l = make(begin, mid, level + 1, id);
    const int r = make(mid, end, level + 1, id);
    t.clusters[id].child = {l, r};
    return id;
  }
};
}  // namespace

ClusterTree build_cluster_tree(const PointSet& pts, int leafsize) {
  if (leafsize < 1) throw ConfigError("leafsize must be >= 1");
  if (pts.size() == 0) throw ConfigError("cannot build a cluster tree over no points");
  const int n = pts.size();
  ClusterTree t;
  t.leafsize = leafsize;
  t.perm.resize(n);
  std::iota(t.perm.begin(), t.perm.end(), 0);
  int depth = 0;
  while ((n + (1 << depth) - 1) / (1 << depth) > leafsize) ++depth;
  t.depth = depth;
  TreeBuilder b{pts, t, depth};
  b.make(0, n, 0, -1);
  t.inv_perm.resize(n);
  for (int i = 0; i < n; ++i) t.inv_perm[t.perm[i]] = i;
  t.levels.assign(depth + 1, {});
  for (const Cluster& c : t.clusters) t.levels[c.level].push_back(c.id);
  for (auto& lv : t.levels)
    std::sort(lv.begin(), lv.end(),
              [&](int a, int b) { return t.clusters[a].begin < t.clusters[b].begin; });
  return t;
}

// cluster_tree.cpp:95-109 — bounding-box gap distance; admissible iff the gap
// is positive and max(diam) <= eta * gap.
double bbox_distance(const Cluster& t, const Cluster& s) {
  double g[3];
  for (int a = 0; a < 3; ++a)
    g[a] = std::max(std::max(t.bbox_min[a] - s.bbox_max[a], s.bbox_min[a] - t.bbox_max[a]), 0.0);
  return norm3(g[0], g[1], g[2]);
}
bool is_admissible(const Cluster& t, const Cluster& s, double eta) {
  const double diam = std::max(t.diameter(), s.diameter());
  const double dist = bbox_distance(t, s);
  return dist > 0.0 && diam <= eta * dist;
}

// ---------------------------------------------------------------------------
// block_tree.cpp:9-53 — recursive subdivision from (root, root).
BlockTree::BlockTree(std::shared_ptr<const ClusterTree> rows,
                     std::shared_ptr<const ClusterTree> cols, double eta)
    : rows_(std::move(rows)), cols_(std::move(cols)), eta_(eta) {
  if (eta_ <= 0) throw ConfigError("eta must be positive");
  if (rows_->size() != cols_->size())
    throw ConfigError("block tree requires trees over the same unknown count");
  if (rows_->depth != cols_->depth) throw ConfigError("block tree requires trees of equal depth");
  level_blocks_.assign(rows_->depth + 1, {});
  subdivide(0, 0);
  finish();
}

BlockTree::BlockTree(std::shared_ptr<const ClusterTree> tree, double eta,
                     std::vector<std::vector<BlockEntry>> level_blocks)
    : rows_(tree), cols_(tree), eta_(eta), level_blocks_(std::move(level_blocks)) {
  for (const auto& lv : level_blocks_)
    for (const BlockEntry& e : lv) kind_.emplace(e.key, e.kind);
  finish();
}

void BlockTree::finish() {
  for (auto& lv : level_blocks_)
    std::sort(lv.begin(), lv.end(),
              [](const BlockEntry& a, const BlockEntry& b) { return a.key < b.key; });
  // block_tree.cpp:24-31 — sparsity constant over rows and columns per level
  c_sp_ = 0;
  for (const auto& lv : level_blocks_) {
    std::map<int, int> per_row, per_col;
    for (const BlockEntry& e : lv) {
      c_sp_ = std::max(c_sp_, ++per_row[e.key.row]);
      c_sp_ = std::max(c_sp_, ++per_col[e.key.col]);
    }
  }
}

void BlockTree::subdivide(int t, int s) {
  const Cluster& ct = rows_->clusters[t];
  const Cluster& cs = cols_->clusters[s];
  BlockKind k;
  if (is_admissible(ct, cs, eta_)) k = BlockKind::admissible;
  else if (ct.is_leaf() && cs.is_leaf()) k = BlockKind::inadmissible_leaf;
  else k = BlockKind::subdivided;
  kind_.emplace(BlockKey{t, s}, k);
  level_blocks_[ct.level].push_back({BlockKey{t, s}, k});
  if (k != BlockKind::subdivided) return;
  if (ct.is_leaf() || cs.is_leaf())
    throw InvariantError("uneven block subdivision; trees are not level-uniform");
  for (int a : ct.child)
    for (int b : cs.child) subdivide(a, b);
}

std::optional<BlockKind> BlockTree::kind(int t, int s) const {
  auto it = kind_.find(BlockKey{t, s});
  if (it == kind_.end()) return std::nullopt;
  return it->second;
}

// block_tree.cpp:61-85 — walk ancestor pairs until a block is found.
TargetStatus BlockTree::target_status(int t, int s) const {
  for (int a = t, b = s; a >= 0 && b >= 0;
       a = rows_->clusters[a].parent, b = cols_->clusters[b].parent) {
    auto it = kind_.find(BlockKey{a, b});
    if (it == kind_.end()) continue;
    if (a != t) {
      if (it->second != BlockKind::admissible)
        throw InvariantError("cluster pair below a non-admissible block");
      return TargetStatus::inside_admissible;
    }
    switch (it->second) {
      case BlockKind::admissible: return TargetStatus::admissible;
      case BlockKind::inadmissible_leaf: return TargetStatus::full_block;
      case BlockKind::subdivided: return TargetStatus::subdivided;
    }
  }
  throw InvariantError("cluster pair not covered by the block tree");
}

std::int64_t BlockTree::admissible_count() const {
  std::int64_t n = 0;
  for (const auto& [k, v] : kind_) n += v == BlockKind::admissible;
  return n;
}
std::int64_t BlockTree::inadmissible_count() const {
  std::int64_t n = 0;
  for (const auto& [k, v] : kind_) n += v == BlockKind::inadmissible_leaf;
  return n;
}

}  // namespace h2o
