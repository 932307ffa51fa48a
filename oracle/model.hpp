// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/dense.hpp).
//
// CPU restatement of the reference's data model and algorithms on the MMP
// path.  Each declaration cites the reference symbol it restates.
#pragma once

#include <array>
#include <functional>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <tuple>
#include <vector>

#include "dense.hpp"

namespace h2o {

// ---- errors (errors.hpp:9-29) ---------------------------------------------
struct ConfigError : std::invalid_argument {
  explicit ConfigError(const std::string& w) : std::invalid_argument(w) {}
};
struct InvariantError : std::logic_error {
  explicit InvariantError(const std::string& w) : std::logic_error(w) {}
};
struct AssemblyError : std::runtime_error {
  explicit AssemblyError(const std::string& w) : std::runtime_error(w) {}
};

// ---- geometry (geometry.hpp:15-78) ----------------------------------------
struct Vec3 {
  double x = 0, y = 0, z = 0;
  double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  double& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
};
inline double norm3(double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); }

struct PointSet {
  std::vector<Vec3> points;
  int size() const { return static_cast<int>(points.size()); }
};

enum class Family { random_cloud = 0, bus = 1, slab = 2, cube_array = 3 };
struct GeometrySpec {
  Family family = Family::random_cloud;
  std::uint64_t seed = 0;
  int n = 0;
  int bus_count = 0;
  int samples_per_meter = 1;
  int slab_width = 0;
  int slab_thickness = 2;
  int array_edge = 0;
  int cube_points = 3;
};
PointSet generate_geometry(const GeometrySpec& spec);  // geometry.cpp:159-181

enum class KernelKind { laplace = 0, helmholtz = 1 };
struct Kernel {
  KernelKind kind = KernelKind::laplace;
  double wavenumber = 0.0;
  std::optional<double> diagonal_value;
};
template <class S>
Mat<S> assemble_dense(const PointSet& pts, const Kernel& kernel);  // geometry.cpp:200-233

// ---- cluster tree (cluster_tree.hpp:12-41) --------------------------------
struct Cluster {
  int id = -1, parent = -1, level = 0, begin = 0, end = 0;
  std::array<int, 2> child{-1, -1};
  Vec3 bbox_min, bbox_max;
  bool is_leaf() const { return child[0] < 0; }
  int size() const { return end - begin; }
  double diameter() const {
    return norm3(bbox_max.x - bbox_min.x, bbox_max.y - bbox_min.y, bbox_max.z - bbox_min.z);
  }
};
struct ClusterTree {
  std::vector<Cluster> clusters;
  std::vector<std::vector<int>> levels;
  std::vector<int> perm, inv_perm;
  int depth = 0;
  int leafsize = 0;
  int size() const { return static_cast<int>(perm.size()); }
};
ClusterTree build_cluster_tree(const PointSet& pts, int leafsize);  // cluster_tree.cpp:66-93
double bbox_distance(const Cluster& t, const Cluster& s);          // cluster_tree.cpp:95-102
bool is_admissible(const Cluster& t, const Cluster& s, double eta);  // cluster_tree.cpp:104-109

// ---- block tree (block_tree.hpp:13-73) ------------------------------------
enum class BlockKind : unsigned char { admissible = 0, inadmissible_leaf = 1, subdivided = 2 };
enum class TargetStatus : unsigned char { full_block, admissible, subdivided, inside_admissible };
struct BlockKey {
  int row = -1, col = -1;
  friend bool operator<(const BlockKey& a, const BlockKey& b) {
    return a.row < b.row || (a.row == b.row && a.col < b.col);
  }
  friend bool operator==(const BlockKey& a, const BlockKey& b) {
    return a.row == b.row && a.col == b.col;
  }
};
struct BlockEntry {
  BlockKey key;
  BlockKind kind;
};
class BlockTree {
 public:
  BlockTree(std::shared_ptr<const ClusterTree> rows, std::shared_ptr<const ClusterTree> cols,
            double eta);
  // Rebuild from flat lists (used when the structure comes over the C-ABI).
  BlockTree(std::shared_ptr<const ClusterTree> tree, double eta,
            std::vector<std::vector<BlockEntry>> level_blocks);
  const ClusterTree& rows() const { return *rows_; }
  const ClusterTree& cols() const { return *cols_; }
  double eta() const { return eta_; }
  int depth() const { return rows_->depth; }
  int c_sp() const { return c_sp_; }
  const std::vector<BlockEntry>& level_blocks(int l) const { return level_blocks_[l]; }
  std::optional<BlockKind> kind(int t, int s) const;
  TargetStatus target_status(int t, int s) const;  // block_tree.cpp:61-85
  std::int64_t admissible_count() const;
  std::int64_t inadmissible_count() const;

 private:
  void subdivide(int t, int s);
  void finish();
  std::shared_ptr<const ClusterTree> rows_, cols_;
  double eta_;
  int c_sp_ = 0;
  std::vector<std::vector<BlockEntry>> level_blocks_;
  std::map<BlockKey, BlockKind> kind_;
};

// ---- truncation (truncation.hpp:7-19) -------------------------------------
template <class S>
struct TruncatedBasis {
  Mat<S> basis;
  bool degenerate = false;
  std::vector<double> eigenvalues;  // ascending, clamped (diagnostic: threshold margins)
};
template <class S>
TruncatedBasis<S> svd_truncate_gram(const Mat<S>& gram, double eps);  // truncation.cpp:9-47

// ---- H^2 format (h2_matrix.hpp:19-48) -------------------------------------
template <class S>
struct ClusterBasis {
  std::vector<Mat<S>> leaf, transfer;
  std::vector<Index> rank;
  std::vector<char> degenerate;
  void resize(size_t n) {
    leaf.assign(n, {});
    transfer.assign(n, {});
    rank.assign(n, 0);
    degenerate.assign(n, 0);
  }
};
template <class S>
struct H2Matrix {
  std::shared_ptr<const ClusterTree> tree;
  std::shared_ptr<const BlockTree> structure;
  ClusterBasis<S> row_basis, col_basis;
  std::map<BlockKey, Mat<S>> coupling, full;
  int size() const { return tree ? tree->size() : 0; }
};

template <class S>
H2Matrix<S> build_h2(const Mat<S>& dense, std::shared_ptr<const BlockTree> structure,
                     double eps_h2);  // h2_matrix.cpp:141-181
template <class S>
Mat<S> h2_to_dense(const H2Matrix<S>& h);  // h2_matrix.cpp:183-211
template <class S>
std::vector<S> mvp(const H2Matrix<S>& h, const std::vector<S>& x);  // h2_matrix.cpp:213-278
template <class S>
std::int64_t memory_footprint(const H2Matrix<S>& h);  // h2_matrix.cpp:280-292
template <class S>
Mat<S> materialized_row_basis(const H2Matrix<S>& h, int cluster);  // h2_matrix.cpp:294-297
template <class S>
Mat<S> materialized_col_basis(const H2Matrix<S>& h, int cluster);  // h2_matrix.cpp:299-302

// ---- MMP (mmp.hpp:16-74) --------------------------------------------------
struct LevelStats {
  int level = 0;
  Index max_row_rank = 0, max_col_rank = 0;
  std::array<std::int64_t, 4> case_products{0, 0, 0, 0};
  int max_case1_terms = 0, max_case2_terms = 0, max_case3_terms = 0;
};
struct MmpReport {
  double eps_trunc = 0.0;
  bool adaptive = true;
  std::vector<LevelStats> levels;
  std::int64_t flops = 0;
  std::array<std::int64_t, 4> case_flops{0, 0, 0, 0};
  double wall_seconds = 0.0;
  int pending_after_split = 0;
  // oracle diagnostics: per truncation, the smallest relative distance of an
  // eigenvalue to the threshold eps*lambda_max (rank-flip margins)
  double min_threshold_margin = 1e300;
};
template <class S>
struct MmpResult {
  H2Matrix<S> product;
  MmpReport report;
};

struct MmpOptions {
  // bytes the leaf F^A F^B cache may occupy (mmp.cpp:127-133); beyond it the
  // oracle recomputes products instead of caching (identical values and
  // counters)
  std::int64_t ff_cache_bytes = std::int64_t(8) << 30;
  // threads of the parallel restatement (1 = the reference's single thread;
  // results are bit-identical for any count, oracle/product_engine.cpp)
  int threads = 1;
  // slice point callback (counted MACs so far); may block or throw
  std::function<void(std::int64_t)> gate;
};

template <class S>
MmpResult<S> mmp(const H2Matrix<S>& a, const H2Matrix<S>& b, double eps,
                 const MmpOptions& opt = {});  // mmp.cpp:688-691
template <class S>
MmpResult<S> formatted_mmp(const H2Matrix<S>& a, const H2Matrix<S>& b,
                           const MmpOptions& opt = {});  // mmp.cpp:716-719
template <class S>
std::vector<Mat<S>> basis_products(const H2Matrix<S>& a, const H2Matrix<S>& b);  // :693-714

// ---- metrics (metrics.hpp:21-57) ------------------------------------------
template <class S>
std::vector<S> random_vector(int n, std::uint64_t seed);  // metrics.cpp:17-35
template <class S>
double relative_error(const H2Matrix<S>& a, const H2Matrix<S>& b, const H2Matrix<S>& c,
                      std::uint64_t seed, bool* reference_was_zero = nullptr);  // :37-55

}  // namespace h2o
