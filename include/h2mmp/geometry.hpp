// PointSet of proj/core/include/h2mmp/geometry.hpp:15-22 (Eigen-free: points
// as std::array<double,3>).  The generators and kernels of geometry.cpp are
// input-side and outside the MMP path; make_random_cloud is provided because
// the BASELINE workloads use it (geometry.cpp:39-52).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "../h2c.h"
#include "h2mmp/errors.hpp"

namespace h2mmp {

struct PointSet {
  std::vector<std::array<double, 3>> points;
  std::vector<int> labels;
  int size() const { return static_cast<int>(points.size()); }
};

inline PointSet make_random_cloud(int n, std::uint64_t seed) {
  PointSet p;
  p.points.resize(n);
  if (h2c_random_cloud(n, seed, p.points.empty() ? nullptr : p.points[0].data()) != H2C_OK)
    throw ConfigError(h2c_last_error(nullptr));
  return p;
}

}  // namespace h2mmp
