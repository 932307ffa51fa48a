// Owned ClusterTree + BlockTree in the flat layout of h2c_types.h.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "../../include/h2c_types.h"

namespace h2b {

struct Structure {
  int32_t n_points = 0, depth = 0, leafsize = 0, c_sp = 0;
  double eta = 1.0;
  std::vector<int32_t> parent, child0, child1, level, begin, end, perm;
  std::vector<double> bbox;
  std::vector<int64_t> level_ptr;
  std::vector<int32_t> row, col;
  std::vector<uint8_t> kind;
  void tree_desc(h2c_tree* d) const;
  void blocks_desc(h2c_blocks* d) const;
};

std::unique_ptr<Structure> build_structure(const double* xyz, int n, int leafsize, double eta);
int target_status(const h2c_tree& t, const h2c_blocks& b, int ti, int si);

// owned flat H^2 matrix
struct HostH2 {
  int32_t scalar = 0;
  std::vector<int32_t> row_rank, col_rank;
  std::vector<uint8_t> row_dg, col_dg;
  std::vector<int64_t> row_off, col_off, block_off;
  std::vector<double> values;
  void desc(h2c_matrix* d) const;
};

// orders: interpolation order per level (depth + 1 entries)
std::unique_ptr<HostH2> build_chebyshev(const h2c_tree& t, const h2c_blocks& b, const double* xyz, int kernel,
                                        double kappa, double diagonal, const int* orders, double eps_recompress,
                                        int threads);
std::unique_ptr<HostH2> build_fd_laplacian(const h2c_tree& t, const h2c_blocks& b, const double* xyz, double h);

}  // namespace h2b
