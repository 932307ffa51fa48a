// Host-only C-ABI entry points (structure, synthetic inputs): see capi_inputs.hpp.
#include <algorithm>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/h2c.h"
#include "capi_inputs.hpp"

using namespace h2b;

namespace h2b {
std::string& capi_error() {
  thread_local std::string e;
  return e;
}
}  // namespace h2b

namespace {
#define g_err (h2b::capi_error())
}  // namespace

#ifdef H2C_INPUTS_ONLY
int h2c_version(void) { return 1; }
const char* h2c_last_error(const h2c_context*) { return g_err.c_str(); }
#endif

h2c_structure* h2c_build_structure(const double* xyz, int n, int leafsize, double eta) {
  try {
    auto* s = new h2c_structure;
    s->s = build_structure(xyz, n, leafsize, eta);
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void h2c_structure_tree(const h2c_structure* s, h2c_tree* out) { s->s->tree_desc(out); }
void h2c_structure_blocks(const h2c_structure* s, h2c_blocks* out) { s->s->blocks_desc(out); }
void h2c_structure_free(h2c_structure* s) { delete s; }

int h2c_target_status(const h2c_tree* tree, const h2c_blocks* blocks, int t, int s) {
  try {
    return target_status(*tree, *blocks, t, s);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int h2c_random_cloud(int n, uint64_t seed, double* xyz) {
  if (n < 1) {
    g_err = "random_cloud: n must be positive";
    return H2C_ERR_CONFIG;
  }
  std::mt19937_64 eng(seed);
  for (int64_t i = 0; i < 3 * int64_t(n); ++i) xyz[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
  return H2C_OK;
}

h2c_h2* h2c_build_chebyshev(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz, int kernel,
                            double kappa, double diagonal, int order, double eps_recompress, int threads) {
  try {
    if (order < 1) throw std::invalid_argument("chebyshev order must be >= 1");
    const std::vector<int> orders(tree->depth + 1, order);
    return h2c_build_chebyshev_orders(tree, blocks, xyz, kernel, kappa, diagonal, orders.data(), eps_recompress,
                                      threads);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

h2c_h2* h2c_build_chebyshev_orders(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz, int kernel,
                                   double kappa, double diagonal, const int* orders, double eps_recompress,
                                   int threads) {
  try {
    auto m = std::make_unique<h2c_h2>();
    m->m = build_chebyshev(*tree, *blocks, xyz, kernel, kappa, diagonal, orders, eps_recompress,
                           threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency())));
    return m.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

h2c_h2* h2c_build_fd_laplacian(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz, double h) {
  try {
    auto* m = new h2c_h2;
    m->m = build_fd_laplacian(*tree, *blocks, xyz, h);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void h2c_h2_desc(const h2c_h2* m, h2c_matrix* out) { m->m->desc(out); }
void h2c_h2_free(h2c_h2* m) { delete m; }

int h2c_random_vector(int n, uint64_t seed, int scalar, double* out) {
  if (n < 0) {
    g_err = "random_vector: negative length";
    return H2C_ERR_CONFIG;
  }
  std::mt19937_64 eng(seed);
  auto u = [&eng] { return 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0; };
  for (int64_t i = 0; i < int64_t(n) * (scalar == H2C_COMPLEX ? 2 : 1); ++i) out[i] = u();
  return H2C_OK;
}

