// B200 MMP engine: level-synchronous device pipeline (see engine.cu).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "plan.hpp"

namespace h2b {

struct DevPlan;  // device copies of the plan's index lists

struct ProfileEntry {
  std::string name;  // phase/kernel
  int64_t launches = 0;
  double ms = 0;
  int64_t macs = 0;
  int64_t bytes = 0;  // algorithmic HBM bytes (operands read once per entry, outputs written / accumulated)
};

// Reusable pinned host buffers for product downloads (pinning tens of GB per
// call would dominate the end-to-end time).  Shared by the context and the
// results it hands out, so either may outlive the other.
class PinnedPool {
 public:
  double* take(size_t bytes, size_t* got);
  void give(double* p, size_t bytes);
  ~PinnedPool();

 private:
  std::mutex mu_;
  std::multimap<size_t, double*> free_;
};

// Host-side result of one product (flat layout of include/h2c_types.h).
struct HostResult {
  std::shared_ptr<PinnedPool> pool;
  size_t values_bytes = 0;
  int32_t scalar = 0;
  std::vector<int32_t> row_rank, col_rank;
  std::vector<uint8_t> row_dg, col_dg;
  std::vector<int64_t> row_off, col_off, block_off;
  double* values = nullptr;  // pinned host memory owned by the result
  int64_t n_values = 0;
  // report
  double eps_trunc = 0;
  int adaptive = 1;
  int64_t flops = 0, flops_exec = 0;
  std::array<int64_t, 4> case_flops{0, 0, 0, 0};
  double wall_seconds = 0, device_seconds = 0, plan_seconds = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  std::vector<int64_t> max_row, max_col, case_products;
  std::vector<int32_t> t1, t2, t3;
  ~HostResult();
};

// Operand already resident on the device (padded per-level layout).
struct DevOperand;
struct DevResult;

class Context {
 public:
  explicit Context(int device);
  ~Context();
  const std::string& error() const { return err_; }
  void set_error(const std::string& e) { err_ = e; }

  // plan cache keyed by the structure descriptors' content
  const Plan& plan_for(const h2c_tree& t, const h2c_blocks& b, double* build_seconds);

  // full drop-in call: host descriptors in, host result out
  void mmp(const h2c_matrix& a, const h2c_matrix& b, double eps, int adaptive, HostResult& out);

  // device-resident path (bench `value`): upload once, run many times
  std::shared_ptr<DevOperand> upload(const h2c_matrix& m);
  // runs the pipeline on resident operands; returns device seconds (CUDA events)
  double run_resident(const std::shared_ptr<DevOperand>& a, const std::shared_ptr<DevOperand>& b,
                      double eps, int adaptive, HostResult* download_to);
  // svd_truncate_gram on the device (truncation.cpp:9-47); basis: n x n buffer
  void truncate_gram(int scalar, const double* gram, int n, double eps, double* basis, int* rank, int* degenerate);
  // exact H^2 MVP Y = A X on a resident operand (host X, Y: N x nv, original ordering)
  void mvp(const std::shared_ptr<DevOperand>& a, const double* x, int nv, double* y);
  // h2_to_dense (h2_matrix.cpp:124-137): A * I through the device MVP, N x N host output
  void to_dense(const std::shared_ptr<DevOperand>& a, double* out);
  void* stream() const { return stream_; }
  int device() const { return device_; }
  struct Arena* arena();  // large-buffer arena of the device, shared by every Context (lazy)
  std::recursive_mutex& call_mutex();  // serialises calls on the device (process-wide)
  // side streams.  0: auxiliary stream of
  // the off-critical-path work (leaf full targets, deferred coupling-target
  // sums) at low priority, optionally bound to a green context holding a
  // subset of the SMs (H2B_AUX_SMS) so the critical path keeps SMs of its own;
  // 1: the column eigensolve of a level, concurrent with the row one
  static constexpr int kSideStreams = 2;
  int aux_sms() const { return aux_sms_; }
  void* side_stream(int i);
  void* make_aux_stream(int priority);
  int64_t last_kernel_launches() const { return launches_; }
  std::shared_ptr<PinnedPool> pinned = std::make_shared<PinnedPool>();
  // per (phase, kernel) timings of the last run, filled when profiling is on
  std::vector<ProfileEntry> last_profile;
  bool profile = false;

 private:
  friend struct EngineRun;
  int device_;
  void* stream_ = nullptr;
  std::vector<void*> side_streams_;
  void* green_ctx_ = nullptr;
  void* green_destroy_ = nullptr;
  int aux_sms_ = 0;  // SMs of the auxiliary stream's green context (0: whole device)
  std::string err_;
  uint64_t plan_key_ = 0;
  std::unique_ptr<Plan> plan_;
  std::vector<int32_t> perm_, key_rows_, key_cols_;  // cached structure (confirms a plan-cache hit)
  std::unique_ptr<DevPlan> dplan_;
  int64_t launches_ = 0;
};

uint64_t structure_hash(const h2c_tree& t, const h2c_blocks& b);

}  // namespace h2b
