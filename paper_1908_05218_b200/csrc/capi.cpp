// C-ABI entry points of libh2mmp_b200.so (include/h2c.h).  Errors map to the
// reference's exception classes (errors.hpp:9-29): ConfigError ->
// H2C_ERR_CONFIG, InvariantError -> H2C_ERR_INVARIANT, CUDA failures ->
// H2C_ERR_CUDA.  There is no CPU fallback: without a usable device every MMP
// entry point fails with H2C_ERR_CUDA.
#include <algorithm>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>

#include "../../include/h2c.h"
#include "counters.hpp"
#include "engine.hpp"
#include "structure.hpp"
#include "capi_inputs.hpp"

using namespace h2b;

struct h2c_context {
  std::unique_ptr<Context> ctx;
  std::string err;
};
struct h2c_result {
  HostResult r;
  const h2c_tree* tree = nullptr;
  const h2c_blocks* blocks = nullptr;
};
struct h2c_operand {
  std::shared_ptr<DevOperand> op;
};

namespace {
#define g_err (h2b::capi_error())

int code_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return H2C_ERR_CONFIG;
  if (dynamic_cast<const std::logic_error*>(&e)) return H2C_ERR_INVARIANT;
  if (dynamic_cast<const std::bad_alloc*>(&e)) return H2C_ERR_ALLOC;
  return H2C_ERR_CUDA;
}

template <class F>
int guarded(h2c_context* c, F&& f) {
  try {
    f();
    return H2C_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    if (c) c->err = e.what();
    return code_of(e);
  }
}
}  // namespace

int h2c_version(void) { return 1; }

const char* h2c_last_error(const h2c_context* ctx) { return ctx && !ctx->err.empty() ? ctx->err.c_str() : g_err.c_str(); }

h2c_context* h2c_create(int device) {
  try {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n <= device)
      throw std::runtime_error(std::string("no CUDA device available: ") + cudaGetErrorString(e));
    auto* c = new h2c_context;
    c->ctx = std::make_unique<Context>(device);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void h2c_destroy(h2c_context* ctx) { delete ctx; }

int64_t h2c_kernel_launches(const h2c_context* ctx) { return ctx ? ctx->ctx->last_kernel_launches() : 0; }
void* h2c_stream(const h2c_context* ctx) { return ctx ? ctx->ctx->stream() : nullptr; }
void h2c_set_profile(h2c_context* ctx, int on) {
  if (ctx) ctx->ctx->profile = on != 0;
}
int h2c_profile_count(const h2c_context* ctx) { return ctx ? static_cast<int>(ctx->ctx->last_profile.size()) : 0; }
int64_t h2c_profile_bytes(const h2c_context* ctx, int i) {
  if (!ctx || i < 0 || i >= static_cast<int>(ctx->ctx->last_profile.size())) return -1;
  return ctx->ctx->last_profile[i].bytes;
}
int h2c_profile_get(const h2c_context* ctx, int i, char* name, int cap, int64_t* launches, double* ms,
                    int64_t* macs) {
  if (!ctx || i < 0 || i >= static_cast<int>(ctx->ctx->last_profile.size())) return H2C_ERR_CONFIG;
  const ProfileEntry& e = ctx->ctx->last_profile[i];
  if (name && cap > 0) {
    std::strncpy(name, e.name.c_str(), cap - 1);
    name[cap - 1] = 0;
  }
  if (launches) *launches = e.launches;
  if (ms) *ms = e.ms;
  if (macs) *macs = e.macs;
  return H2C_OK;
}

static int run_mmp(h2c_context* ctx, const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive,
                   h2c_result** out) {
  *out = nullptr;
  if (!ctx) {
    g_err = "h2c_mmp: null context (no CUDA device)";
    return H2C_ERR_CUDA;
  }
  auto res = std::make_unique<h2c_result>();
  const int rc = guarded(ctx, [&] {
    ctx->ctx->mmp(*a, *b, eps, adaptive, res->r);
    res->tree = a->tree;
    res->blocks = a->blocks;
  });
  if (rc == H2C_OK) *out = res.release();
  return rc;
}

int h2c_mmp(h2c_context* ctx, const h2c_matrix* a, const h2c_matrix* b, double eps, h2c_result** out) {
  return run_mmp(ctx, a, b, eps, 1, out);
}
int h2c_formatted_mmp(h2c_context* ctx, const h2c_matrix* a, const h2c_matrix* b, h2c_result** out) {
  return run_mmp(ctx, a, b, 0.0, 0, out);
}

void h2c_result_matrix(const h2c_result* r, h2c_matrix* d) {
  d->tree = r->tree;
  d->blocks = r->blocks;
  d->scalar = r->r.scalar;
  d->row_rank = r->r.row_rank.data();
  d->col_rank = r->r.col_rank.data();
  d->row_degenerate = r->r.row_dg.data();
  d->col_degenerate = r->r.col_dg.data();
  d->row_offset = r->r.row_off.data();
  d->col_offset = r->r.col_off.data();
  d->block_offset = r->r.block_off.data();
  d->values = r->r.values;
  d->n_values = r->r.n_values;
}

void h2c_result_report(const h2c_result* r, h2c_report* d) {
  std::memset(d, 0, sizeof(*d));
  const HostResult& h = r->r;
  d->eps_trunc = h.eps_trunc;
  d->adaptive = h.adaptive;
  d->n_levels = static_cast<int32_t>(h.max_row.size());
  d->flops = h.flops;
  for (int c = 0; c < 4; ++c) d->case_flops[c] = h.case_flops[c];
  d->wall_seconds = h.wall_seconds;
  d->pending_after_split = 0;
  d->max_row_rank = h.max_row.data();
  d->max_col_rank = h.max_col.data();
  d->case_products = h.case_products.data();
  d->max_case1_terms = h.t1.data();
  d->max_case2_terms = h.t2.data();
  d->max_case3_terms = h.t3.data();
  d->flops_exec = h.flops_exec;
  d->device_seconds = h.device_seconds;
  d->plan_seconds = h.plan_seconds;
  d->h2d_bytes = h.h2d_bytes;
  d->d2h_bytes = h.d2h_bytes;
}

void h2c_result_free(h2c_result* r) { delete r; }

int h2c_upload(h2c_context* ctx, const h2c_matrix* m, h2c_operand** out) {
  *out = nullptr;
  if (!ctx) return H2C_ERR_CUDA;
  auto op = std::make_unique<h2c_operand>();
  const int rc = guarded(ctx, [&] { op->op = ctx->ctx->upload(*m); });
  if (rc == H2C_OK) *out = op.release();
  return rc;
}

void h2c_operand_free(h2c_operand* op) { delete op; }

int h2c_mmp_resident(h2c_context* ctx, const h2c_operand* a, const h2c_operand* b, double eps, int adaptive,
                     double* device_seconds, h2c_result** out) {
  if (out) *out = nullptr;
  if (!ctx) return H2C_ERR_CUDA;
  std::unique_ptr<h2c_result> res = out ? std::make_unique<h2c_result>() : nullptr;
  const int rc = guarded(ctx, [&] {
    if (adaptive && !(eps > 0.0 && eps < 1.0)) throw std::invalid_argument("mmp: eps_trunc must be in (0,1)");
    const double s = ctx->ctx->run_resident(a->op, b->op, eps, adaptive, res ? &res->r : nullptr);
    if (device_seconds) *device_seconds = s;
  });
  if (rc == H2C_OK && out) *out = res.release();
  return rc;
}

void* h2c_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    g_err = "cudaMallocHost failed";
    return nullptr;
  }
  return p;
}
void h2c_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int h2c_count_report(const h2c_matrix* a, const h2c_matrix* b, const h2c_matrix* c, int adaptive, double eps,
                     h2c_result** out) {
  *out = nullptr;
  auto res = std::make_unique<h2c_result>();
  const int rc = guarded(nullptr, [&] {
    if (a->tree != b->tree || a->blocks != b->blocks || a->tree != c->tree)
      throw std::invalid_argument("count_report: operands must share cluster trees and block structure");
    const Plan P = build_plan(*a->tree, *a->blocks, 8);
    RankSet rs;
    auto fill = [&](const int32_t* rk, std::vector<std::vector<int64_t>>& dst) {
      dst.resize(P.depth + 1);
      for (int l = 0; l <= P.depth; ++l)
        for (int p = 0; p < P.lv[l].n; ++p) dst[l].push_back(rk[P.lv[l].id[p]]);
    };
    fill(a->row_rank, rs.ar);
    fill(a->col_rank, rs.ac);
    fill(b->row_rank, rs.br);
    fill(b->col_rank, rs.bc);
    fill(c->row_rank, rs.cr);
    fill(c->col_rank, rs.cc);
    CountOut co;
    count_report(P, rs, adaptive != 0, co);
    HostResult& h = res->r;
    h.eps_trunc = adaptive ? eps : 0.0;
    h.adaptive = adaptive;
    h.flops = co.flops;
    h.case_flops = co.case_flops;
    for (const LevelCount& lc : co.levels) {
      h.max_row.push_back(lc.max_row_rank);
      h.max_col.push_back(lc.max_col_rank);
      for (int k = 0; k < 4; ++k) h.case_products.push_back(lc.case_products[k]);
      h.t1.push_back(lc.max_case1_terms);
      h.t2.push_back(lc.max_case2_terms);
      h.t3.push_back(lc.max_case3_terms);
    }
    res->tree = a->tree;
    res->blocks = a->blocks;
  });
  if (rc == H2C_OK) *out = res.release();
  return rc;
}

int h2c_plan_stats(const h2c_tree* tree, const h2c_blocks* blocks, int64_t* out, int cap) {
  try {
    const Plan P = build_plan(*tree, *blocks, 8);
    for (int l = 0; l <= P.depth && l < cap; ++l) {
      const LevelPlan& L = P.lv[l];
      int64_t* o = out + 10 * l;
      o[0] = L.n;
      o[1] = static_cast<int64_t>(L.adm.size());
      o[2] = static_cast<int64_t>(L.nearb.size());
      o[3] = static_cast<int64_t>(L.pend_row.size());
      o[4] = static_cast<int64_t>(L.nl_block.size());
      o[5] = static_cast<int64_t>(L.merged_row.size());
      o[6] = L.lyr.entries();
      o[7] = L.lyn.entries();
      o[8] = L.xr.entries();
      o[9] = L.ww.entries();
    }
    return P.depth + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int h2c_mvp_resident(h2c_context* ctx, const h2c_operand* a, const double* x, int nv, double* y) {
  if (!ctx) return H2C_ERR_CUDA;
  return guarded(ctx, [&] { ctx->ctx->mvp(a->op, x, nv, y); });
}

int h2c_mvp(h2c_context* ctx, const h2c_matrix* a, const double* x, int nv, double* y) {
  if (!ctx) return H2C_ERR_CUDA;
  return guarded(ctx, [&] {
    auto op = ctx->ctx->upload(*a);
    ctx->ctx->mvp(op, x, nv, y);
  });
}

int h2c_to_dense(h2c_context* ctx, const h2c_matrix* a, double* out) {
  if (!ctx) return H2C_ERR_CUDA;
  return guarded(ctx, [&] {
    auto op = ctx->ctx->upload(*a);
    ctx->ctx->to_dense(op, out);
  });
}

int h2c_truncate_gram(h2c_context* ctx, int scalar, const double* gram, int n, double eps, double* basis, int* rank,
                      int* degenerate) {
  if (!ctx) return H2C_ERR_CUDA;
  return guarded(ctx, [&] { ctx->ctx->truncate_gram(scalar, gram, n, eps, basis, rank, degenerate); });
}
