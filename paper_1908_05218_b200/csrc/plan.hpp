// Structure plan: everything the level-synchronous GPU MMP needs that depends
// only on the cluster tree and block structure (never on ranks or values), so
// it is built once per structure and cached by the context.
//
// It replaces the reference's per-call std::map adjacency and per-triple
// ancestor walks (mmp.cpp:92-103, block_tree.cpp:61-85) with flat, per-level
// CSR lists: blocks by row/column, the (i,j,k) triple lists grouped by target
// (i,k) in ascending j (mmp.cpp:301-339, 587-612; accumulation order of
// mmp.hpp:56-59), the structural sets of pending / merged / non-leaf
// couplings, and the split lists of the top-down pass (mmp.cpp:617-659).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/h2c_types.h"

namespace h2b {

enum : uint8_t { kAdm = 0, kFull = 1, kSub = 2 };

// CSR of (left index, right index) entries grouped by output.
struct Csr {
  std::vector<int32_t> ptr;  // [n_out + 1]
  std::vector<int32_t> li, ri;
  int64_t entries() const { return static_cast<int64_t>(li.size()); }
};

struct LevelPlan {
  int level = 0;
  int n = 0;  // clusters at this level; positions 0..n-1 ordered by begin
  std::vector<int32_t> id;          // position -> cluster id
  std::vector<int32_t> size;        // cluster sizes
  // blocks at this level in (row, col) order
  std::vector<int32_t> brow, bcol;  // level positions
  std::vector<uint8_t> bkind;
  std::vector<int64_t> bglobal;     // index into h2c_blocks arrays
  std::vector<int32_t> kidx;        // index inside its kind (adm list or near list)
  std::vector<int32_t> adm, nearb;  // block indices of admissible / near (full or subdivided)
  std::vector<int32_t> row_ptr;     // CSR over rows: blocks of row p are [row_ptr[p], row_ptr[p+1])
  std::vector<int32_t> col_ptr, col_blk;  // CSR over columns (blocks sorted by row)

  // ---- coupling targets: [0, n_adm) admissible C blocks (adm order),
  //      [n_adm, n_adm + n_pend) pending pairs, then NL (subdivided) blocks
  std::vector<int32_t> pend_row, pend_col;  // pending pairs (inside-admissible), sorted
  std::vector<int32_t> pend_mq;             // pending q -> 4 * (merged idx at level-1) + quadrant
  std::vector<int32_t> nl_block;            // subdivided blocks holding NL content (sorted)
  std::vector<int32_t> nl_of_block;         // block -> nl slot or -1
  int n_targets() const { return static_cast<int>(adm.size() + pend_row.size() + nl_block.size()); }
  std::vector<int32_t> target_row, target_col;  // positions of every coupling target

  // triple groups into coupling targets, entries in ascending middle cluster j
  Csr ly;  // (A block idx, B adm idx) with B admissible, A any (report counters)
  Csr lyr;  // (A adm idx, B adm idx): R x R, summed as S^A B_j S^B (P^A, P^B factored out)
  Csr lyn;  // (A block idx, B adm idx) with A near: coll_a S^B (P^B factored out)
  Csr xr;  // (A adm idx, B block idx) with A admissible, B near
  Csr ww;  // leaf only: (A near idx, B near idx) full x full into a coupling target
  // per-target case ids for the report: counts of case 0..3 contributions
  // leaf only: full targets (C full blocks, near-list order)
  Csr ff;  // (A near idx, B near idx)
  Csr fr;  // (A near idx, B adm idx)
  Csr rf;  // (A adm idx, B near idx)
  Csr rr;  // (A adm idx, B adm idx)

  // merged children couplings at this level (non-leaf): parent pairs of the
  // pending targets of level+1 with the pending slot of each quadrant (-1 = none)
  std::vector<int32_t> merged_row, merged_col;
  std::vector<int32_t> merged_quad;  // [n_merged][4] pending index at level+1 (q = 2*ri + ci)
  std::vector<int32_t> merged_target;  // coupling-target slot at this level
  // case-1 contributions T^C_i^H M conj(T^C_k) written straight into their
  // targets before the triple sums accumulate: merged blocks whose target is
  // admissible (out = Tg slot) and whose target is pending (out = parent's
  // merged quadrant, see pend_mq); per entry: row pos, col pos, merged idx, out
  struct MergedInto {
    std::vector<int32_t> row, col, m, out;
  } mz_adm, mz_pend;
  // case-1 into targets: CSR over coupling targets of merged indices (0 or 1 each)
  Csr mg;  // (merged idx, target col position)

  // leaf Gram support (leaf level only)
  Csr hq;   // per A near (full) block (i,j): B near blocks (j,k) with (i,k) qualifying
  Csr hqc;  // per B near (full) block (j,k): A near blocks (i,j) with (i,k) qualifying
  Csr row_near, col_near;  // per cluster: near blocks in its row / column (block order)
  // non-leaf Gram support
  Csr row_merged, col_merged;  // per cluster: merged indices in its row / column

  // children blocks of each subdivided block (non-leaf level): [n_near][4] block
  // indices at level+1 (q = 2*ti + si)
  std::vector<int32_t> sub_child;

  // top-down split: for each slot pair q = 2*ri + ci, child blocks at level+1
  // receiving from an existing NL block of this level: (nl slot, child block idx)
  std::vector<int32_t> split_src[4], split_dst[4];

  // report counters that depend only on structure
  int64_t case_products[4] = {0, 0, 0, 0};
};

struct Plan {
  int depth = 0;
  int n_points = 0;
  int64_t n_clusters = 0;
  std::vector<LevelPlan> lv;
  std::vector<int32_t> pos_of;    // cluster id -> level position
  double build_seconds = 0;
  int64_t total_triples = 0;
};

// Builds the plan; throws std::invalid_argument / std::logic_error with the
// reference's messages on malformed structure (block_tree.cpp:61-85).
Plan build_plan(const h2c_tree& tree, const h2c_blocks& blocks, int threads);

}  // namespace h2b
