// BlockTree of proj/core/include/h2mmp/block_tree.hpp:13-77 (same enums, keys,
// accessors), built by the B200 library (h2c_build_structure).  The MMP path
// uses square structures over ONE shared cluster tree (mmp.cpp:59), which is
// the only form the drop-in builds.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <vector>

#include "h2mmp/cluster_tree.hpp"

namespace h2mmp {

enum class BlockKind : unsigned char { admissible, inadmissible_leaf, subdivided };
enum class TargetStatus : unsigned char { full_block, admissible, subdivided, inside_admissible };

struct BlockKey {
  int row = -1;
  int col = -1;
  friend bool operator<(const BlockKey& a, const BlockKey& b) {
    return a.row < b.row || (a.row == b.row && a.col < b.col);
  }
  friend bool operator==(const BlockKey& a, const BlockKey& b) { return a.row == b.row && a.col == b.col; }
};

struct BlockEntry {
  BlockKey key;
  BlockKind kind;
};

class BlockTree {
 public:
  BlockTree(std::shared_ptr<const ClusterTree> tree, double eta) : tree_(std::move(tree)), eta_(eta) {
    if (eta_ <= 0) throw ConfigError("eta must be positive");
    h2c_structure* s = h2c_build_structure(tree_->points.data(), tree_->size(), tree_->leafsize, eta_);
    if (!s) throw ConfigError(h2c_last_error(nullptr));
    h2c_blocks d;
    h2c_structure_blocks(s, &d);
    c_sp_ = d.c_sp;
    ptr_.assign(d.level_ptr, d.level_ptr + d.depth + 2);
    row_.assign(d.row, d.row + d.n_blocks);
    col_.assign(d.col, d.col + d.n_blocks);
    kind8_.assign(d.kind, d.kind + d.n_blocks);
    h2c_structure_free(s);
    level_blocks_.assign(tree_->depth + 1, {});
    for (int l = 0; l <= tree_->depth; ++l)
      for (int64_t b = ptr_[l]; b < ptr_[l + 1]; ++b) {
        const BlockEntry e{BlockKey{row_[b], col_[b]}, static_cast<BlockKind>(kind8_[b])};
        level_blocks_[l].push_back(e);
        kind_.emplace(e.key, e.kind);
      }
    desc = h2c_blocks{tree_->depth, c_sp_, eta_, static_cast<int64_t>(row_.size()), ptr_.data(), row_.data(),
                      col_.data(), kind8_.data()};
  }

  const ClusterTree& rows() const { return *tree_; }
  const ClusterTree& cols() const { return *tree_; }
  const std::shared_ptr<const ClusterTree>& rows_ptr() const { return tree_; }
  const std::shared_ptr<const ClusterTree>& cols_ptr() const { return tree_; }
  double eta() const { return eta_; }
  int depth() const { return tree_->depth; }
  int c_sp() const { return c_sp_; }
  const std::vector<BlockEntry>& level_blocks(int level) const { return level_blocks_[level]; }
  std::optional<BlockKind> kind(int t, int s) const {
    auto it = kind_.find(BlockKey{t, s});
    if (it == kind_.end()) return std::nullopt;
    return it->second;
  }
  /// block_tree.cpp:61-85
  TargetStatus target_status(int t, int s) const {
    const int r = h2c_target_status(&tree_->desc, &desc, t, s);
    if (r < 0) throw InvariantError(h2c_last_error(nullptr));
    return static_cast<TargetStatus>(r);
  }
  std::int64_t admissible_count() const { return count(BlockKind::admissible); }
  std::int64_t inadmissible_count() const { return count(BlockKind::inadmissible_leaf); }

  h2c_blocks desc{};
  // index of a block in the flat arrays (level order, (row, col) order)
  int64_t flat_index(const BlockKey& k) const {
    const int l = tree_->clusters[k.row].level;
    for (int64_t b = ptr_[l]; b < ptr_[l + 1]; ++b)
      if (row_[b] == k.row && col_[b] == k.col) return b;
    return -1;
  }

 private:
  std::int64_t count(BlockKind k) const {
    std::int64_t n = 0;
    for (const auto& [key, v] : kind_) n += v == k;
    return n;
  }
  std::shared_ptr<const ClusterTree> tree_;
  double eta_;
  int c_sp_ = 0;
  std::vector<int64_t> ptr_;
  std::vector<int32_t> row_, col_;
  std::vector<uint8_t> kind8_;
  std::vector<std::vector<BlockEntry>> level_blocks_;
  std::map<BlockKey, BlockKind> kind_;
};

/// block_tree.cpp:101-105 (rows and cols must be the same shared tree)
inline std::shared_ptr<const BlockTree> build_block_tree(std::shared_ptr<const ClusterTree> rows,
                                                         std::shared_ptr<const ClusterTree> cols, double eta) {
  if (rows != cols) throw ConfigError("build_block_tree: the B200 MMP path requires one shared cluster tree");
  return std::make_shared<const BlockTree>(std::move(rows), eta);
}

}  // namespace h2mmp
