// Wall time of the C++ drop-in call h2mmp::mmp(a, a, eps) (include/h2mmp/mmp.hpp: flatten the
// std::map blocks -> h2c_mmp -> unflatten the result) at the configs[1] size, cold and warm, next
// to the raw C-ABI call on the same flat descriptors.  Usage: dropin_time [N] [leaf] [order] [eps]
//   g++ -std=c++17 -O2 -Iinclude tools/dropin_time.cpp -Lpaper_1908_05218_b200/lib -lh2mmp_b200 \
//       -Wl,-rpath,$PWD/paper_1908_05218_b200/lib -o /tmp/dropin_time
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "h2mmp/h2mmp.hpp"

using namespace h2mmp;
using clk = std::chrono::steady_clock;
static double since(clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); }

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 65536;
  const int leaf = argc > 2 ? std::atoi(argv[2]) : 64;
  const int order = argc > 3 ? std::atoi(argv[3]) : 4;
  const double eps = argc > 4 ? std::atof(argv[4]) : 1e-8;
  auto t0 = clk::now();
  const PointSet pts = make_random_cloud(n, 1);
  auto tree = std::make_shared<const ClusterTree>(build_cluster_tree(pts, leaf));
  auto structure = build_block_tree(tree, tree, 1.0);
  h2c_h2* raw = h2c_build_chebyshev(&tree->desc, &structure->desc, tree->points.data(), 0, 0.0, 0.0, order, 0.0, 0);
  if (!raw) return 2;
  h2c_matrix d;
  h2c_h2_desc(raw, &d);
  d.tree = &tree->desc;
  d.blocks = &structure->desc;
  const double build_s = since(t0);
  t0 = clk::now();
  const H2Matrix<Real> a = detail::unflatten<Real>(d, tree, structure);
  const double unflat_s = since(t0);

  // raw C-ABI call on the flat descriptors (cold: first call of the process, builds the plan)
  h2c_context* ctx = detail::default_context();
  double cabi[3];
  for (int i = 0; i < 3; ++i) {
    t0 = clk::now();
    h2c_result* res = nullptr;
    if (h2c_mmp(ctx, &d, &d, eps, &res) != 0) return 3;
    cabi[i] = since(t0);
    h2c_result_free(res);
  }
  h2c_h2_free(raw);
  t0 = clk::now();
  const detail::Flat<Real> f = detail::flatten(a);
  const double flat_s = since(t0);
  double cpp[2], dev = 0.0;
  long long flops = 0;
  for (int i = 0; i < 2; ++i) {
    t0 = clk::now();
    const MmpResult<Real> r = mmp(a, a, eps);
    cpp[i] = since(t0);
    flops = r.report.flops;
    dev = r.report.device_seconds;
  }
  std::printf("{\"N\": %d, \"leaf\": %d, \"order\": %d, \"eps\": %g, \"build_seconds\": %.3f, "
              "\"unflatten_operand_seconds\": %.3f, \"flatten_operand_seconds\": %.3f, "
              "\"c_abi_cold_seconds\": %.3f, \"c_abi_warm_seconds\": [%.3f, %.3f], "
              "\"cpp_mmp_seconds\": [%.3f, %.3f], \"device_seconds\": %.3f, \"macs\": %lld, "
              "\"cpp_gflops\": %.1f, \"c_abi_gflops\": %.1f}\n",
              n, leaf, order, eps, build_s, unflat_s, flat_s, cabi[0], cabi[1], cabi[2], cpp[0], cpp[1], dev, flops,
              2.0 * flops / cpp[1] / 1e9, 2.0 * flops / cabi[2] / 1e9);
  return 0;
}
