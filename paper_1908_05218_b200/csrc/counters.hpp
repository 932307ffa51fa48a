// Reference MmpReport counters from structure + ranks (see counters.cpp).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace h2b {

// per level, per position ranks (int64 to keep the products exact)
struct RankSet {
  std::vector<std::vector<int64_t>> ar, ac, br, bc, cr, cc;
};

struct LevelCount {
  int64_t max_row_rank = 0, max_col_rank = 0;
  std::array<int64_t, 4> case_products{0, 0, 0, 0};
  int max_case1_terms = 0, max_case2_terms = 0, max_case3_terms = 0;
};

struct CountOut {
  int64_t flops = 0;
  std::array<int64_t, 4> case_flops{0, 0, 0, 0};
  std::vector<LevelCount> levels;
};

void count_report(const Plan& P, const RankSet& r, bool adaptive, CountOut& out);

}  // namespace h2b
