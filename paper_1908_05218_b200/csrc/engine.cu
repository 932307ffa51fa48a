// Level-synchronous B200 pipeline of the accuracy-controlled H^2-MMP
// (the reference's ProductEngine, proj/core/src/mmp.cpp:13-684), restated as
// batched products over padded per-level device arrays.
//
// Data layout in HBM (per operand X in {A, B, C}, level l, padded ranks
// K = round_up(max rank at l, 8), leaf size NL = round_up(max #t, 8)):
//   leaf bases      V  [n_L][NL x K_L]            column-major, zero padded
//   transfers       T_l[n_l][2K_{l+1} x K_l]      child 0 rows [0,K_{l+1}), child 1 rows [K_{l+1},2K_{l+1})
//   couplings       S_l[n_adm,l][Kr_l x Kc_l]     admissible blocks in (row,col) order
//   full blocks     F  [n_full][NL x NL]
// Zero padding is exact under every product, so padded rows/columns never
// leak into results; ranks are tracked per cluster on the host.
//
// Reassociation (value-neutral up to rounding, counted separately as
// flops_exec): the projections P^A_i, P^B_k of the four product cases depend
// only on the target (i,k), so they are applied once per target after the sum
// over the middle cluster j (see targets()):
//   T_ik = P^A_i [ sum_RR (S^A B_j) S^B + sum_RF S^A coll_b ] + [ sum_FR coll_a S^B ] P^B_k ... * P^B_k
// which costs k_A k_B k_B per R x R triple instead of the reference's
// left-to-right chain (4 k^3, mmp.cpp:329-332) - 16x fewer MACs at the upper
// levels where C's ranks grow to ~300.  Leaf full x full into couplings stays
// sum_j (V^C^H F_ij)(F_jk conj(V^C)), and the leaf Gram
// G1 = sum_{j,k} (F F)(F F)^H is evaluated as sum_j F_ij (sum_k F_jk F_jk^H) F_ij^H.
#include <cuda_runtime.h>
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <exception>
#include <thread>
#include <tuple>

#include "counters.hpp"
#include "engine.hpp"
#include "heev.cuh"
#include "kernels.cuh"

namespace h2b {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct ConfigErr : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " __FILE__ \
                      ":" + std::to_string(__LINE__));                                         \
  } while (0)

static inline int pad8(int64_t r) { return static_cast<int>(std::max<int64_t>(8, (r + 7) / 8 * 8)); }

// ---------------------------------------------------------------------------
// Device memory.  Large buffers of the main stream come from a per-context
// arena (one cudaMalloc, best-fit free list with coalescing, host-side
// immediate free: every user of such a buffer is ordered on the main stream,
// or joined to it before the free).  This avoids the pool growth / physical
// re-mapping that fragmented cudaMallocAsync pools pay for multi-GB,
// differently-sized per-level buffers on every product.  Everything else is
// stream-ordered cudaMallocAsync.
class Arena {
 public:
  bool init(size_t bytes) {
    if (cudaMalloc(&base_, bytes) != cudaSuccess) {
      cudaGetLastError();
      base_ = nullptr;
      return false;
    }
    cap_ = bytes;
    free_.clear();
    free_[0] = bytes;
    return true;
  }
  ~Arena() {
    if (base_) cudaFree(base_);
  }
  // high = long-lived buffer (operands, C's targets / merged blocks / full blocks): taken from the
  // top of the highest free block that fits, so the short-lived per-level scratch (best fit from
  // the bottom) does not interleave with it and fragment the arena
  void* alloc(size_t bytes, bool high = false) {
    bytes = (bytes + 255) & ~size_t(255);
    std::lock_guard<std::mutex> g(mu_);
    reclaim_locked(false);
    auto best = free_.end();
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= bytes &&
          (best == free_.end() || (high ? it->first > best->first : it->second < best->second)))
        best = it;
    if (best == free_.end()) return nullptr;
    const size_t off = best->first, sz = best->second;
    free_.erase(best);
    size_t at = off;
    if (high) {
      at = off + sz - bytes;
      if (sz > bytes) free_[off] = sz - bytes;
    } else if (sz > bytes) {
      free_[off + bytes] = sz - bytes;
    }
    used_[at] = bytes;
    return static_cast<char*>(base_) + at;
  }
  // the exact range [p, p + bytes) if it is free (an evicted buffer returning to its own place,
  // so repeated products see the same layout), else nullptr
  void* alloc_at(void* p, size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    std::lock_guard<std::mutex> g(mu_);
    reclaim_locked(false);
    if (!owns(p)) return nullptr;
    const size_t off = static_cast<char*>(p) - static_cast<char*>(base_);
    auto it = free_.upper_bound(off);
    if (it == free_.begin()) return nullptr;
    --it;
    const size_t b0 = it->first, sz = it->second;
    if (b0 > off || b0 + sz < off + bytes) return nullptr;
    free_.erase(it);
    if (off > b0) free_[b0] = off - b0;
    if (b0 + sz > off + bytes) free_[off + bytes] = b0 + sz - (off + bytes);
    used_[off] = bytes;
    return p;
  }
  // (total free bytes, largest free block)
  std::pair<size_t, size_t> stats() {
    std::lock_guard<std::mutex> g(mu_);
    size_t tot = 0, big = 0;
    for (auto& kv : free_) {
      tot += kv.second;
      big = std::max(big, kv.second);
    }
    return {tot, big};
  }
  size_t capacity() const { return cap_; }
  bool owns(const void* p) const {
    return base_ && p >= base_ && p < static_cast<const char*>(base_) + cap_;
  }
  void free(void* p) {
    std::lock_guard<std::mutex> g(mu_);
    free_locked(p);
  }
  // A block last used on another stream (the auxiliary stream) returns to the
  // free list only once `ev`, recorded there after its last use, has completed
  // (checked on later allocations) or after the main stream has joined it.
  void free_after(void* p, cudaEvent_t ev) {
    std::lock_guard<std::mutex> g(mu_);
    pending_.push_back({p, ev});
  }
  bool has_pending() {
    std::lock_guard<std::mutex> g(mu_);
    return !pending_.empty();
  }
  // all_done: the main stream has waited for everything issued on the other streams
  void reclaim(bool all_done) {
    std::lock_guard<std::mutex> g(mu_);
    reclaim_locked(all_done);
  }

 private:
  void reclaim_locked(bool all_done) {
    size_t k = 0;
    for (size_t i = 0; i < pending_.size(); ++i) {
      if (all_done || cudaEventQuery(pending_[i].second) == cudaSuccess) {
        free_locked(pending_[i].first);
        cudaEventDestroy(pending_[i].second);
      } else {
        pending_[k++] = pending_[i];
      }
    }
    pending_.resize(k);
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not sticky, but clear it
  }
  void free_locked(void* p) {
    size_t off = static_cast<char*>(p) - static_cast<char*>(base_);
    auto u = used_.find(off);
    if (u == used_.end()) return;
    size_t sz = u->second;
    used_.erase(u);
    auto next = free_.lower_bound(off);
    if (next != free_.end() && next->first == off + sz) {  // merge right
      sz += next->second;
      next = free_.erase(next);
    }
    if (next != free_.begin()) {  // merge left
      auto prev = std::prev(next);
      if (prev->first + prev->second == off) {
        prev->second += sz;
        return;
      }
    }
    free_[off] = sz;
  }

  void* base_ = nullptr;
  size_t cap_ = 0;
  std::map<size_t, size_t> free_, used_;
  std::vector<std::pair<void*, cudaEvent_t>> pending_;
  std::mutex mu_;
};

// Per-device state shared by every Context of the process: the arena (one cudaMalloc of
// the free HBM minus a reserve, so it cannot be per context) and the mutex that serialises
// calls on the device (the arena, the plan caches and the pinned pools are not re-entrant).
// It lives until process exit, so buffers released after their Context is gone still
// return to a live arena.
struct DeviceShared {
  std::recursive_mutex call_mu;
  std::mutex init_mu;
  Arena* arena = nullptr;
  bool tried = false;
};
static DeviceShared& device_shared(int dev) {
  static std::mutex m;
  static std::map<int, DeviceShared*> all;
  std::lock_guard<std::mutex> g(m);
  DeviceShared*& p = all[dev];
  if (!p) p = new DeviceShared;  // intentionally never freed (process lifetime)
  return *p;
}

// the arena of the context running on this thread, and its main stream
thread_local Arena* t_arena = nullptr;
thread_local cudaStream_t t_arena_stream = nullptr;
// long-lived allocations (Arena::alloc high) while a HighScope is alive on this thread
thread_local bool t_arena_high = false;
struct HighScope {
  bool prev;
  explicit HighScope(bool on = true) : prev(t_arena_high) { t_arena_high = on; }
  ~HighScope() { t_arena_high = prev; }
};
// the auxiliary stream of the run on this thread: its buffers also come from the
// arena and are returned through Arena::free_after
thread_local cudaStream_t t_aux_stream = nullptr;
// memory-pressure hook of the run on this thread: frees device memory (eviction of buffers the
// rest of the product does not read) and returns true if it did
struct Relief {
  virtual bool relieve() = 0;
  virtual ~Relief() = default;
};
thread_local Relief* t_relief = nullptr;
constexpr size_t kArenaMin = size_t(8) << 20;
// per-buffer scratch bound of the chunked target / full-block / case-1 loops:
// one chunk per level at cfg2, bounded scratch at the larger configurations
constexpr size_t kChunkBytes = size_t(8) << 30;
// the chunk bound actually used: kChunkBytes, or 1/24 of the arena's free bytes when that is
// smaller (large configurations near the HBM capacity)

struct DBuf {
  double* p = nullptr;
  size_t n = 0;  // doubles
  cudaStream_t s = nullptr;
  Arena* arena = nullptr;
  bool aux = false;  // arena block used on the auxiliary stream
  DBuf() = default;
  DBuf(size_t doubles, cudaStream_t st, bool zero = false) { alloc(doubles, st, zero); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      arena = o.arena;
      aux = o.aux;
      o.p = nullptr;
      o.n = 0;
      o.arena = nullptr;
    }
    return *this;
  }
  // takes over an arena block obtained by the caller (Arena::alloc_at)
  void adopt(double* ptr, size_t doubles, cudaStream_t st, Arena* a) {
    release();
    p = ptr;
    n = doubles;
    s = st;
    arena = a;
    aux = false;
  }
  void alloc(size_t doubles, cudaStream_t st, bool zero = false) {
    release();
    s = st;
    n = std::max<size_t>(doubles, 2);
    if (t_arena && (st == t_arena_stream || (st && st == t_aux_stream)) && n * sizeof(double) >= kArenaMin) {
      p = static_cast<double*>(t_arena->alloc(n * sizeof(double), t_arena_high));
      if (!p && t_aux_stream && t_arena->has_pending()) {
        // memory pressure: let the deferred work drain, reclaim its blocks, retry
        CK(cudaStreamSynchronize(t_aux_stream));
        t_arena->reclaim(false);
        p = static_cast<double*>(t_arena->alloc(n * sizeof(double), t_arena_high));
      }
      while (!p && t_relief && t_relief->relieve())  // evict what the rest of the product does not read
        p = static_cast<double*>(t_arena->alloc(n * sizeof(double), t_arena_high));
      if (p) {
        arena = t_arena;
        aux = st != t_arena_stream;
      }
    }
    if (!p) {
      const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(double), s);
      if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        std::string msg = "device allocation of " + std::to_string(n * sizeof(double) >> 20) + " MiB failed (" +
                          cudaGetErrorString(e) + ")";
        if (t_arena) {
          const auto st = t_arena->stats();
          msg += "; arena " + std::to_string(t_arena->capacity() >> 20) + " MiB, free " + std::to_string(st.first >> 20) +
                 " MiB, largest free block " + std::to_string(st.second >> 20) + " MiB";
        }
        throw CudaError(msg);
      }
    }
    if (zero) CK(cudaMemsetAsync(p, 0, n * sizeof(double), s));
  }
  void release() {
    if (p) {
      if (arena && aux) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, s));
        arena->free_after(p, ev);
      } else if (arena) {
        arena->free(p);
      } else {
        cudaFreeAsync(p, s);
      }
    }
    p = nullptr;
    n = 0;
    arena = nullptr;
    aux = false;
  }
  ~DBuf() { release(); }
  operator double*() const { return p; }
};

template <class T>
struct DVec {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DVec() = default;
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  DVec(DVec&& o) noexcept { *this = std::move(o); }
  DVec& operator=(DVec&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
    }
    return *this;
  }
  void upload(const std::vector<T>& v, cudaStream_t st) {
    release();
    s = st;
    n = v.size();
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(1, n) * sizeof(T), s));
    if (n) CK(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void alloc(size_t cnt, cudaStream_t st) {
    release();
    s = st;
    n = cnt;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(1, n) * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  ~DVec() { release(); }
};

// ---------------------------------------------------------------------------
// device copy of the plan
struct DevCsr {
  const int* ptr = nullptr;
  const int* li = nullptr;
  const int* ri = nullptr;
  int n_out = 0;
  int64_t entries = 0;
};

struct DevLevel {
  DevCsr lyr, lyn, xr, ww, ff, fr, rf, rr, mg, hq, hqc, row_near, col_near, row_merged, col_merged;
  const int *target_row = nullptr, *target_col = nullptr;
  DevCsr adm_by_row;   // per row position: (adm idx, col position)   (MVP coupling products)
  DevCsr near_by_row;  // per row position: (near idx, col position)  (MVP near field)
  const int *near_row = nullptr, *near_col = nullptr, *adm_row = nullptr, *adm_col = nullptr;
  const int *nearb = nullptr, *adm = nullptr, *merged_row = nullptr, *merged_quad = nullptr;
  const int *sub_child = nullptr, *nl_col = nullptr;
  const int* subq[4] = {};  // per quadrant q = 2*ri + ci: sub_child[4 t + q] (child block index)
  const int* pend_mq = nullptr;  // pending target -> 4 * merged idx (level-1) + quadrant
  struct MZ {
    const int *row = nullptr, *col = nullptr, *m = nullptr, *out = nullptr;
    int n = 0;
  } mz_adm, mz_pend;  // LevelPlan::MergedInto
  // split from this level into level+1, per quadrant
  const int *sp_src[4] = {}, *sp_prow[4] = {}, *sp_omap[4] = {};
  int sp_n[4] = {0, 0, 0, 0};
  const int *sf_src[4] = {}, *sf_prow[4] = {}, *sf_near[4] = {}, *sf_crow[4] = {}, *sf_ccol[4] = {};
  int sf_n[4] = {0, 0, 0, 0};
};

struct DevPlan {
  std::vector<DevLevel> lv;
  const int* even = nullptr;  // p -> 2p
  const int* odd = nullptr;   // p -> 2p+1
  const int* iota = nullptr;  // e -> e (block indices of chunked outputs written densely)
  DVec<int32_t> blob;
};

static std::unique_ptr<DevPlan> upload_plan(const Plan& P, cudaStream_t s) {
  auto D = std::make_unique<DevPlan>();
  std::vector<int32_t> blob;
  std::vector<std::pair<const int**, size_t>> fix;
  auto put = [&](const int** dst, const std::vector<int32_t>& v) {
    fix.push_back({dst, blob.size()});
    blob.insert(blob.end(), v.begin(), v.end());
    blob.push_back(0);  // keep every array non-empty
  };
  auto put_csr = [&](DevCsr& d, const Csr& c) {
    put(&d.ptr, c.ptr);
    put(&d.li, c.li);
    put(&d.ri, c.ri);
    d.n_out = c.ptr.empty() ? 0 : static_cast<int>(c.ptr.size()) - 1;
    d.entries = c.entries();
  };
  D->lv.resize(P.depth + 1);
  int maxn = 1;
  for (int l = 0; l <= P.depth; ++l) {
    const LevelPlan& L = P.lv[l];
    DevLevel& Q = D->lv[l];
    maxn = std::max(maxn, L.n);
    put_csr(Q.lyr, L.lyr);
    put_csr(Q.lyn, L.lyn);
    put(&Q.target_row, L.target_row);
    put(&Q.target_col, L.target_col);
    put_csr(Q.xr, L.xr);
    put_csr(Q.ww, L.ww);
    put_csr(Q.ff, L.ff);
    put_csr(Q.fr, L.fr);
    put_csr(Q.rf, L.rf);
    put_csr(Q.rr, L.rr);
    put_csr(Q.mg, L.mg);
    put_csr(Q.hq, L.hq);
    put_csr(Q.hqc, L.hqc);
    put_csr(Q.row_near, L.row_near);
    put_csr(Q.col_near, L.col_near);
    put_csr(Q.row_merged, L.row_merged);
    put_csr(Q.col_merged, L.col_merged);
    std::vector<int32_t> nr, nc, ar, ac, nlc;
    for (int b : L.nearb) {
      nr.push_back(L.brow[b]);
      nc.push_back(L.bcol[b]);
    }
    for (int b : L.adm) {
      ar.push_back(L.brow[b]);
      ac.push_back(L.bcol[b]);
    }
    for (int b : L.nl_block) nlc.push_back(L.bcol[b]);
    put(&Q.near_row, nr);
    put(&Q.near_col, nc);
    put(&Q.adm_row, ar);
    put(&Q.adm_col, ac);
    put(&Q.nearb, L.nearb);
    put(&Q.adm, L.adm);
    put(&Q.merged_row, L.merged_row);
    put(&Q.merged_quad, L.merged_quad);
    put(&Q.pend_mq, L.pend_mq);
    auto put_mz = [&](DevLevel::MZ& d, const LevelPlan::MergedInto& z) {
      put(&d.row, z.row);
      put(&d.col, z.col);
      put(&d.m, z.m);
      put(&d.out, z.out);
      d.n = static_cast<int>(z.m.size());
    };
    put_mz(Q.mz_adm, L.mz_adm);
    put_mz(Q.mz_pend, L.mz_pend);
    put(&Q.sub_child, L.sub_child);
    for (int q = 0; q < 4; ++q) {
      std::vector<int32_t> v(L.sub_child.size() / 4);
      for (size_t t = 0; t < v.size(); ++t) v[t] = L.sub_child[4 * t + q];
      put(&Q.subq[q], v);
    }
    put(&Q.nl_col, nlc);
    {
      Csr ar, nr;
      ar.ptr.assign(L.n + 1, 0);
      nr.ptr.assign(L.n + 1, 0);
      for (int p = 0; p < L.n; ++p) {
        for (int b = L.row_ptr[p]; b < L.row_ptr[p + 1]; ++b) {
          if (L.bkind[b] == kAdm) {
            ar.li.push_back(L.kidx[b]);
            ar.ri.push_back(L.bcol[b]);
          } else if (L.bkind[b] == kFull) {
            nr.li.push_back(L.kidx[b]);
            nr.ri.push_back(L.bcol[b]);
          }
        }
        ar.ptr[p + 1] = static_cast<int32_t>(ar.li.size());
        nr.ptr[p + 1] = static_cast<int32_t>(nr.li.size());
      }
      put_csr(Q.adm_by_row, ar);
      put_csr(Q.near_by_row, nr);
    }
    if (l < P.depth) {
      const LevelPlan& C = P.lv[l + 1];
      const int cna = static_cast<int>(C.adm.size());
      for (int q = 0; q < 4; ++q) {
        std::vector<int32_t> src, prow, omap, fsrc, fprow, fnear, fcrow, fccol;
        for (size_t e = 0; e < L.split_src[q].size(); ++e) {
          const int nl = L.split_src[q][e];
          const int cb = L.split_dst[q][e];
          const int pr = L.brow[L.nl_block[nl]];
          if (C.bkind[cb] == kFull) {
            fsrc.push_back(nl);
            fprow.push_back(pr);
            fnear.push_back(C.kidx[cb]);
            fcrow.push_back(C.brow[cb]);
            fccol.push_back(C.bcol[cb]);
          } else {
            src.push_back(nl);
            prow.push_back(pr);
            // compacted target store of level+1: [admissible | non-leaf] (pending dropped)
            omap.push_back(C.bkind[cb] == kAdm ? C.kidx[cb] : cna + C.nl_of_block[cb]);
          }
        }
        Q.sp_n[q] = static_cast<int>(src.size());
        Q.sf_n[q] = static_cast<int>(fsrc.size());
        put(&Q.sp_src[q], src);
        put(&Q.sp_prow[q], prow);
        put(&Q.sp_omap[q], omap);
        put(&Q.sf_src[q], fsrc);
        put(&Q.sf_prow[q], fprow);
        put(&Q.sf_near[q], fnear);
        put(&Q.sf_crow[q], fcrow);
        put(&Q.sf_ccol[q], fccol);
      }
    }
  }
  std::vector<int32_t> ev(maxn), od(maxn);
  for (int p = 0; p < maxn; ++p) {
    ev[p] = 2 * p;
    od[p] = 2 * p + 1;
  }
  put(&D->even, ev);
  put(&D->odd, od);
  size_t maxz = 1;
  for (int l = 0; l <= P.depth; ++l) maxz = std::max(maxz, P.lv[l].mz_pend.m.size());
  std::vector<int32_t> io(maxz);
  for (size_t e = 0; e < maxz; ++e) io[e] = static_cast<int32_t>(e);
  put(&D->iota, io);
  D->blob.upload(blob, s);
  for (auto& [dst, off] : fix) *dst = D->blob.p + off;
  return D;
}

// ---------------------------------------------------------------------------
// operands resident on the device
struct DevOperand {
  uint64_t key = 0;
  int scalar = 0;
  int depth = 0, NL = 8;
  std::vector<int> Kr, Kc;                          // padded ranks per level
  std::vector<std::vector<int64_t>> rr, rc;         // ranks per level / position
  std::vector<std::vector<uint8_t>> dgr, dgc;       // degenerate flags
  std::vector<DVec<uint8_t>> dgr_d, dgc_d;
  std::vector<DVec<int32_t>> rr_d, rc_d;
  DBuf Vr, Vc, F;
  std::vector<DBuf> Tr, Tc, S;
};

// scalars per host<->device staging batch (H2B_STAGE_SCALARS overrides; tests use a tiny value
// to exercise the batching)
static int64_t stage_scalars() {
  const char* e = std::getenv("H2B_STAGE_SCALARS");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? v : (int64_t(1) << 27);
}

struct CopyList {
  std::vector<CopyJob> jobs;
  void add(const double* src, double* dst, int rows, int cols, int sld, int dld) {
    if (rows > 0 && cols > 0) jobs.push_back({src, dst, rows, cols, sld, dld});
  }
  void run(cudaStream_t s, int W, int64_t* launches) {
    if (jobs.empty()) return;
    DVec<CopyJob> d;
    d.upload(jobs, s);
    const size_t chunk = 1u << 30;
    for (size_t o = 0; o < jobs.size(); o += chunk) {
      const unsigned nb = static_cast<unsigned>(std::min(chunk, jobs.size() - o));
      copy_jobs_kernel<<<nb, 128, 0, s>>>(d.p + o, W);
      CK(cudaGetLastError());
      (*launches)++;
    }
  }
};

static std::shared_ptr<DevOperand> upload_operand(const Plan& P, const h2c_matrix& m,
                                                  cudaStream_t s, int64_t* launches) {
  auto X = std::make_shared<DevOperand>();
  const int D = P.depth;
  const int W = m.scalar == H2C_COMPLEX ? 2 : 1;
  X->scalar = m.scalar;
  X->depth = D;
  int maxleaf = 1;
  for (int p = 0; p < P.lv[D].n; ++p) maxleaf = std::max(maxleaf, P.lv[D].size[p]);
  X->NL = pad8(maxleaf);
  X->Kr.assign(D + 1, 8);
  X->Kc.assign(D + 1, 8);
  X->rr.resize(D + 1);
  X->rc.resize(D + 1);
  X->dgr.resize(D + 1);
  X->dgc.resize(D + 1);
  for (int l = 0; l <= D; ++l) {
    const LevelPlan& L = P.lv[l];
    int64_t mr = 0, mc = 0;
    for (int p = 0; p < L.n; ++p) {
      const int id = L.id[p];
      X->rr[l].push_back(m.row_rank[id]);
      X->rc[l].push_back(m.col_rank[id]);
      X->dgr[l].push_back(m.row_degenerate ? m.row_degenerate[id] : 0);
      X->dgc[l].push_back(m.col_degenerate ? m.col_degenerate[id] : 0);
      mr = std::max<int64_t>(mr, m.row_rank[id]);
      mc = std::max<int64_t>(mc, m.col_rank[id]);
    }
    X->Kr[l] = pad8(mr);
    X->Kc[l] = pad8(mc);
  }
  X->dgr_d.resize(D + 1);
  X->dgc_d.resize(D + 1);
  X->rr_d.resize(D + 1);
  X->rc_d.resize(D + 1);
  for (int l = 0; l <= D; ++l) {
    X->dgr_d[l].upload(X->dgr[l], s);
    X->dgc_d[l].upload(X->dgc[l], s);
    std::vector<int32_t> a(X->rr[l].begin(), X->rr[l].end()), b(X->rc[l].begin(), X->rc[l].end());
    X->rr_d[l].upload(a, s);
    X->rc_d[l].upload(b, s);
  }
  const int NL = X->NL;
  const LevelPlan& LL = P.lv[D];
  HighScope operand_is_long_lived;
  X->Vr.alloc(size_t(LL.n) * NL * X->Kr[D] * W, s, true);
  X->Vc.alloc(size_t(LL.n) * NL * X->Kc[D] * W, s, true);
  X->F.alloc(size_t(LL.nearb.size()) * NL * NL * W, s, true);
  X->Tr.resize(D + 1);
  X->Tc.resize(D + 1);
  X->S.resize(D + 1);
  for (int l = 1; l < D; ++l) {
    X->Tr[l].alloc(size_t(P.lv[l].n) * 2 * X->Kr[l + 1] * X->Kr[l] * W, s, true);
    X->Tc[l].alloc(size_t(P.lv[l].n) * 2 * X->Kc[l + 1] * X->Kc[l] * W, s, true);
  }
  for (int l = 0; l <= D; ++l)
    X->S[l].alloc(size_t(P.lv[l].adm.size()) * X->Kr[l] * X->Kc[l] * W, s, true);

  // copy jobs with HOST source offsets (scalars into m.values), executed in staged chunks below
  struct HJob {
    int64_t off;
    double* dst;
    int rows, cols, sld, dld;
  };
  std::vector<HJob> hj;
  struct {
    std::vector<HJob>* v;
    void add(int64_t off, double* dst, int rows, int cols, int sld, int dld) {
      if (rows > 0 && cols > 0) v->push_back({off, dst, rows, cols, sld, dld});
    }
  } cl{&hj};
  auto src = [&](int64_t off) { return off; };
  for (int p = 0; p < LL.n; ++p) {
    const int id = LL.id[p];
    if (m.row_offset[id] >= 0)
      cl.add(src(m.row_offset[id]), X->Vr.p + size_t(p) * NL * X->Kr[D] * W, LL.size[p], m.row_rank[id], LL.size[p], NL);
    if (m.col_offset[id] >= 0)
      cl.add(src(m.col_offset[id]), X->Vc.p + size_t(p) * NL * X->Kc[D] * W, LL.size[p], m.col_rank[id], LL.size[p], NL);
  }
  for (int l = 1; l < D; ++l) {
    const LevelPlan& L = P.lv[l];
    for (int p = 0; p < L.n; ++p) {
      for (int side = 0; side < 2; ++side) {
        const int id = L.id[p];
        const int32_t* rk = side == 0 ? m.row_rank : m.col_rank;
        const int64_t off = side == 0 ? m.row_offset[id] : m.col_offset[id];
        if (off < 0) continue;
        const int K1 = side == 0 ? X->Kr[l + 1] : X->Kc[l + 1];
        const int K0 = side == 0 ? X->Kr[l] : X->Kc[l];
        double* base = (side == 0 ? X->Tr[l].p : X->Tc[l].p) + size_t(p) * 2 * K1 * K0 * W;
        const int c0 = rk[P.lv[l + 1].id[2 * p]], c1 = rk[P.lv[l + 1].id[2 * p + 1]];
        cl.add(src(off), base, c0, rk[id], c0 + c1, 2 * K1);
        cl.add(src(off + c0), base + size_t(K1) * W, c1, rk[id], c0 + c1, 2 * K1);
      }
    }
  }
  for (int l = 0; l <= D; ++l) {
    const LevelPlan& L = P.lv[l];
    for (size_t a = 0; a < L.adm.size(); ++a) {
      const int b = L.adm[a];
      const int64_t off = m.block_offset[L.bglobal[b]];
      const int rr = m.row_rank[L.id[L.brow[b]]], rc = m.col_rank[L.id[L.bcol[b]]];
      if (off >= 0) cl.add(src(off), X->S[l].p + a * size_t(X->Kr[l]) * X->Kc[l] * W, rr, rc, rr, X->Kr[l]);
    }
  }
  for (size_t q = 0; q < LL.nearb.size(); ++q) {
    const int b = LL.nearb[q];
    const int64_t off = m.block_offset[LL.bglobal[b]];
    const int nr = LL.size[LL.brow[b]], nc = LL.size[LL.bcol[b]];
    if (off >= 0) cl.add(src(off), X->F.p + q * size_t(NL) * NL * W, nr, nc, nr, NL);
  }
  // Stage the host values through a bounded device buffer (<= 1 GiB per batch of jobs sorted by
  // source offset) instead of one copy of the whole operand: the padded layout is all that stays
  // resident, and no allocation of the operand's full size is needed twice (2^20-point operands
  // are ~35 GB).
  std::sort(hj.begin(), hj.end(), [](const HJob& x, const HJob& y) { return x.off < y.off; });
  const int64_t cap = stage_scalars();  // scalars per staging batch (1 GiB real)
  auto extent = [](const HJob& j) { return int64_t(j.cols - 1) * j.sld + j.rows; };
  int64_t span_max = 0;
  for (const HJob& j : hj) span_max = std::max(span_max, extent(j));
  HighScope staging_is_short_lived(false);
  DBuf stage(size_t(std::max(cap, span_max)) * W, s);
  for (size_t i = 0; i < hj.size();) {
    const int64_t o0 = hj[i].off;
    int64_t o1 = o0 + extent(hj[i]);
    size_t e = i + 1;
    while (e < hj.size() && std::max(o1, hj[e].off + extent(hj[e])) - o0 <= std::max(cap, span_max)) {
      o1 = std::max(o1, hj[e].off + extent(hj[e]));
      ++e;
    }
    CK(cudaMemcpyAsync(stage.p, m.values + o0 * W, size_t(o1 - o0) * W * sizeof(double), cudaMemcpyHostToDevice, s));
    CopyList dl;
    for (size_t q = i; q < e; ++q)
      dl.add(stage.p + (hj[q].off - o0) * W, hj[q].dst, hj[q].rows, hj[q].cols, hj[q].sld, hj[q].dld);
    dl.run(s, W, launches);
    CK(cudaStreamSynchronize(s));  // the staging buffer is reused by the next batch
    i = e;
  }
  return X;
}

// ---------------------------------------------------------------------------
struct Ref {
  const double* p;
  long long s;    // stride between matrices (scalars)
  long long off;  // view offset (scalars)
  int ld;
  int op;
  const double* const* ch = nullptr;  // chunked storage (Chunked::table), see SegGroup::Lch
  int sh = 0;
};

// A per-level store of many equal blocks kept as power-of-two block chunks of <= 4 GiB
// (the merged 2x2 blocks: 55-70 GB at the 64^3 grid of configs[3]) so it needs no single
// contiguous region of the arena; the kernels address block b at table[b >> shift].
struct Chunked {
  std::vector<DBuf> parts;
  DVec<double*> table;
  int shift = 0;
  bool empty() const { return parts.empty(); }
  void alloc(long long nblocks, long long block_doubles, cudaStream_t st, bool zero) {
    release();
    const long long cap = (long long)(size_t(4) << 30) / 8;  // doubles per chunk
    shift = 0;
    while ((2LL << shift) * block_doubles <= cap && (1LL << shift) < nblocks) ++shift;
    const long long bpc = 1LL << shift;
    std::vector<double*> ptrs;
    for (long long b0 = 0; b0 < std::max<long long>(nblocks, 1); b0 += bpc) {
      parts.emplace_back(size_t(std::min(bpc, std::max<long long>(nblocks, 1) - b0) * block_doubles), st, zero);
      ptrs.push_back(parts.back().p);
    }
    table.upload(ptrs, st);
  }
  void release() {
    parts.clear();
    table.release();
  }
};
struct Grp {
  Ref L, R;
  int K;
  const DevCsr* csr;
  const int* li;
  const int* ri;
};

struct EngineRun : Relief {
  Context& ctx;
  const Plan& P;
  const DevPlan& DP;
  const DevOperand& A;
  const DevOperand& B;
  double eps;
  bool adaptive;
  bool cplx;
  int W;
  cudaStream_t s;
  int D, NL;
  int64_t exec_macs = 0;
  std::atomic<int64_t> launches{0};
  // optional per-launch profiling (CUDA events on the engine stream)
  struct ProfRec {
    std::string phase;
    const char* kernel;
    int64_t macs;
    int64_t bytes;
    cudaEvent_t a, b;
  };
  bool profiling = false;
  // H2B_PROF_SHAPES=1: profile entries keyed by launch shape too (M x N, inner dims, entries)
  const bool prof_shapes = std::getenv("H2B_PROF_SHAPES") != nullptr;
  std::string shape_tag;
  std::string phase = "setup";
  std::vector<ProfRec> prof;
  // H2B_NVTX=1: one NVTX range "<phase>:<kernel>" per launch, so ncu can select the
  // launches of one phase (ncu --nvtx --nvtx-include "L9.targets:seg_gemm]")
  const bool nvtx = std::getenv("H2B_NVTX") != nullptr;
  int nvtx_depth = 0;
  void pre(const char* kernel, int64_t macs, int64_t bytes = 0) {
    if (nvtx) {
      nvtxRangePushA((phase + ":" + kernel).c_str());
      ++nvtx_depth;
    }
    if (!profiling) return;
    ProfRec r{phase + shape_tag, kernel, macs, bytes, nullptr, nullptr};
    shape_tag.clear();
    CK(cudaEventCreate(&r.a));
    CK(cudaEventCreate(&r.b));
    CK(cudaEventRecord(r.a, s));
    prof.push_back(r);
  }
  // phase boundary on the main stream: in profiling mode an event pair per
  // phase measures its wall time on the device, gaps included
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  std::chrono::steady_clock::time_point host_t0 = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> host_marks;
  const bool mem_trace = std::getenv("H2B_MEM_TRACE") != nullptr;
  void mark(const std::string& name) {
    phase = name;
    if (mem_trace && t_arena) {
      const auto st = t_arena->stats();
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      std::fprintf(stderr, "[mem] %-24s arena free %7zu MiB (largest %7zu MiB) of %7zu MiB; device free %7zu MiB\n",
                   name.c_str(), st.first >> 20, st.second >> 20, t_arena->capacity() >> 20, fr >> 20);
    }
    if (profiling)
      host_marks.push_back({name, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count()});
    if (!profiling) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, s));
    marks.push_back({name, e});
  }
  void post() {
    if (debug_sync) {  // H2B_DEBUG_SYNC=1: locate a faulting launch by phase
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error in phase ") + phase + ": " + cudaGetErrorString(e));
    }
    if (nvtx_depth > 0) {
      nvtxRangePop();
      --nvtx_depth;
    }
    if (!profiling) return;
    CK(cudaEventRecord(prof.back().b, s));
  }
  const bool debug_sync = std::getenv("H2B_DEBUG_SYNC") != nullptr;
  const bool debug_check = std::getenv("H2B_DEBUG_CHECK") != nullptr;

  // C
  std::vector<int> KCr, KCc;
  std::vector<std::vector<int64_t>> rcr, rcc;
  std::vector<DVec<uint8_t>> dgr, dgc;
  DBuf Vr, Vc, F;
  // Tg: [adm | NL] coupling targets per level; Mg[l]: merged 2x2 blocks of level l,
  // written directly by level l+1's pending targets (mmp.cpp:344-365)
  std::vector<DBuf> Tr, Tc, Tg;
  std::vector<Chunked> Mg;
  // H2B_NO_DEFER=1: admissible / NL targets on the main stream (A/B runs)
  const bool no_defer_env = std::getenv("H2B_NO_DEFER") != nullptr;
  bool defer_targets = true;  // set in run(): off when profiling or H2B_NO_DEFER
  // per-level intermediates
  std::vector<DBuf> Bp, PA, PB, LA, RB;
  // auxiliary stream for the C-independent leaf full targets
  cudaStream_t s_aux = nullptr, prev_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_full = nullptr, ev_side = nullptr;
  bool joined = true;  // nothing queued on the auxiliary stream yet
  std::vector<DBuf> hold;
  // A main-stream buffer the main stream no longer needs but deferred work on
  // the auxiliary stream (all of it already issued) may still read: an arena
  // block returns to the free list once the auxiliary stream passes this point
  // (main-stream reuse is ordered by the stream, auxiliary reuse by the next
  // fork); anything else waits for join().
  void retire(DBuf&& x) {
    if (!x.p) return;
    if (joined) {
      x.release();
      return;
    }
    if (x.arena && !x.aux) {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CK(cudaEventRecord(ev, s_aux));
      x.arena->free_after(x.p, ev);
      x.p = nullptr;
      x.n = 0;
      x.arena = nullptr;
      return;
    }
    hold.push_back(std::move(x));
  }
  void join() {
    if (joined) return;
    CK(cudaEventRecord(ev_full, s_aux));  // everything queued on the auxiliary stream so far
    CK(cudaStreamWaitEvent(s, ev_full, 0));
    if (t_arena) t_arena->reclaim(true);
    hold.clear();  // frees on the main stream, ordered after the join
    joined = true;
  }
  // ---- memory pressure (configs[3] at the 64^3 grid): buffers the upper levels do not read
  // move to pinned host memory and come back when needed: the operands' full blocks once the
  // leaf phase is done (restored at the end of the product), C's full blocks and leaf targets
  // once the deferred leaf work has finished (restored for the split).  Off unless an
  // allocation fails.
  struct Evicted {
    DBuf* buf;
    double* host;
    size_t bytes, n;
    bool operand;
    double* home;  // where the buffer lived in the arena (nullptr: not an arena block)
  };
  std::vector<Evicted> evicted;
  bool leaf_done = false;
  bool splitting = false;
  bool restore_operands = true;  // false: the operands were uploaded for this call only
  Relief* prev_relief = nullptr;
  bool evict(DBuf& b, bool operand) {
    if (!b.p) return false;
    for (auto& e : evicted)
      if (e.buf == &b) return false;
    if (!operand) {  // C's stores are written by the deferred (auxiliary-stream) work
      if (s_aux) CK(cudaStreamSynchronize(s_aux));
    }
    CK(cudaStreamSynchronize(s));
    Evicted e{&b, nullptr, b.n * sizeof(double), b.n, operand, b.arena ? b.p : nullptr};
    size_t got = 0;
    e.host = ctx.pinned->take(e.bytes, &got);
    CK(cudaMemcpyAsync(e.host, b.p, e.bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    e.bytes = got;
    b.release();
    if (t_arena) t_arena->reclaim(false);
    evicted.push_back(e);
    if (std::getenv("H2B_MEM_TRACE"))
      std::fprintf(stderr, "[mem] evicted %zu MiB to pinned host memory (%s)\n", (e.n * 8) >> 20,
                   operand ? "operand full blocks" : "C leaf stores");
    return true;
  }
  bool relieve() override {
    if (!leaf_done) return false;
    if (evict(const_cast<DBuf&>(A.F), true)) return true;
    if (evict(const_cast<DBuf&>(B.F), true)) return true;
    if (splitting) return false;  // the split accumulates into C's leaf stores
    if (evict(F, false)) return true;
    if (evict(Tg[D], false)) return true;
    return false;
  }
  void restore(bool operands) {
    for (size_t i = 0; i < evicted.size();) {
      Evicted& e = evicted[i];
      if (e.operand != operands) {
        ++i;
        continue;
      }
      // back to its own place when that is free again, so the next product on these operands
      // finds the arena laid out as the first one did (a drifting operand fragmented it: the
      // fourth consecutive configs[3] product at 64^3 failed to place a 21 GB target store)
      void* home = (e.home && t_arena) ? t_arena->alloc_at(e.home, e.n * sizeof(double)) : nullptr;
      if (home) {
        e.buf->adopt(static_cast<double*>(home), e.n, s, t_arena);
      } else {
        HighScope long_lived;
        e.buf->alloc(e.n, s);
      }
      CK(cudaMemcpyAsync(e.buf->p, e.host, e.n * sizeof(double), cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
      ctx.pinned->give(e.host, e.bytes);
      evicted.erase(evicted.begin() + i);
    }
  }
  // every device buffer of the product itself (C's stores, bases, per-level factors)
  void release_product() {
    Vr.release();
    Vc.release();
    F.release();
    for (auto* v : {&Tr, &Tc, &Tg, &Bp, &PA, &PB, &LA, &RB, &hold})
      for (DBuf& b : *v) b.release();
    for (Chunked& m : Mg) m.release();
  }
  ~EngineRun() {
    // deferred work may still read held buffers (error paths): drain it first
    if (s_aux) cudaStreamSynchronize(s_aux);
    try {
      // Evicted operand blocks come back only now, after the product's own buffers are gone
      // (the result has been downloaded by then): their home blocks are free again, so the
      // operands stay where they were uploaded and the next product on them finds the arena
      // laid out as this one did.
      if (!evicted.empty()) {
        bool operands = false;
        for (const Evicted& e : evicted) operands |= e.operand;
        if (operands && restore_operands) {
          release_product();
          cudaStreamSynchronize(s);
          if (t_arena) t_arena->reclaim(true);
        }
      }
      if (!restore_operands) {  // per-call operands (h2c_mmp): they are freed next, nothing to bring back
        for (size_t i = 0; i < evicted.size();) {
          if (evicted[i].operand) {
            ctx.pinned->give(evicted[i].host, evicted[i].bytes);
            evicted.erase(evicted.begin() + i);
          } else {
            ++i;
          }
        }
      }
      restore(true);  // operands stay resident across calls
      restore(false);
    } catch (...) {
    }
    t_relief = prev_relief;
    t_aux_stream = prev_aux;
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_full) cudaEventDestroy(ev_full);
    if (ev_side) cudaEventDestroy(ev_side);
  }

  EngineRun(Context& c, const Plan& p, const DevPlan& dp, const DevOperand& a, const DevOperand& b,
            double e, bool ad, cudaStream_t st)
      : ctx(c), P(p), DP(dp), A(a), B(b), eps(e), adaptive(ad), s(st) {
    cplx = a.scalar == H2C_COMPLEX;
    W = cplx ? 2 : 1;
    D = P.depth;
    NL = A.NL;
    KCr.assign(D + 1, 8);
    KCc.assign(D + 1, 8);
    rcr.resize(D + 1);
    rcc.resize(D + 1);
    dgr.resize(D + 1);
    dgc.resize(D + 1);
    Tr.resize(D + 1);
    Tc.resize(D + 1);
    Tg.resize(D + 1);
    Mg.resize(D + 1);
    Bp.resize(D + 1);
    PA.resize(D + 1);
    PB.resize(D + 1);
    LA.resize(D + 2);
    RB.resize(D + 2);
    s_aux = static_cast<cudaStream_t>(c.side_stream(0));
    prev_aux = t_aux_stream;
    t_aux_stream = s_aux;
    prev_relief = t_relief;
    t_relief = this;
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_full, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
  }

  size_t sz(size_t count, int r, int c) const { return count * size_t(r) * c * W; }

  // ---- launchers -----------------------------------------------------------
  // seg_gemm3 (kernels.cuh): cp.async pipeline of 8-deep k-chunks x 4 stages; every
  // inner dimension is a multiple of the k-chunk (the padded layout guarantees it)
  template <int TM, int TN, bool CX, int KC, int ST, int WM = 2, int WN = 2>
  void launch_v3_cfg(const SegParams& sp, dim3 grid) {
    constexpr int sm = Seg2Cfg<TM, TN, CX, KC, ST, WM, WN>::SMEM;
    if constexpr (CX) {
      if (cplx3m) {
        static bool attr3 = false;
        if (!attr3) {
          CK(cudaFuncSetAttribute(seg_gemm3_kernel<TM, TN, CX, KC, ST, WM, WN, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          attr3 = true;
        }
        seg_gemm3_kernel<TM, TN, CX, KC, ST, WM, WN, true><<<grid, 32 * WM * WN, sm, s>>>(sp);
        return;
      }
    }
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(seg_gemm3_kernel<TM, TN, CX, KC, ST, WM, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              sm));
      attr = true;
    }
    seg_gemm3_kernel<TM, TN, CX, KC, ST, WM, WN><<<grid, 32 * WM * WN, sm, s>>>(sp);
  }
  // complex products with 3 real DMMAs per complex MAC (Gauss; cfg5s 0.416 -> 0.377 s,
  // profiles/r01/ab_3m_cfg5s.txt); H2B_CPLX4M=1 restores the 4-product form
  const bool cplx3m = std::getenv("H2B_CPLX4M") == nullptr;
  // 8-wide tile classes: outputs with a padded dimension of 8, e.g. the rank-1 (padded 8)
  // FD operand of cfg4, would waste half a 16-wide tile
  template <int TM, int TN, int WM, int WN>
  void launch_seg8(const SegParams& sp, int tiles) {
    dim3 grid(sp.n_out, tiles);
    if (cplx) launch_v3_cfg<TM, TN, true, 8, 4, WM, WN>(sp, grid);
    else launch_v3_cfg<TM, TN, false, 8, 4, WM, WN>(sp, grid);
    CK(cudaGetLastError());
    launches++;
  }
  template <int TM, int TN>
  void launch_seg(const SegParams& sp, int tiles) {
    for (int g = 0; g < sp.ngroups; ++g)
      if (sp.g[g].K % 8 != 0) throw std::logic_error("seg: inner dimension not a multiple of 8");
    dim3 grid(sp.n_out, tiles);
    if (cplx) launch_v3_cfg<TM, TN, true, 8, 4>(sp, grid);
    else launch_v3_cfg<TM, TN, false, 8, 4>(sp, grid);
    CK(cudaGetLastError());
    launches++;
  }

  // one-shot quadrant scatter for the next seg() (see SegParams::oquad)
  struct Quad {
    const int* mq = nullptr;
    int qm = 0, qn = 0;
  } quad;
  // one-shot chunked output store for the next seg() (see SegParams::och)
  const Chunked* ochunk = nullptr;
  void seg(double* out, long long Os, long long Ooff, int Old, const int* omap, int M, int N, int n_out,
           bool acc, std::initializer_list<Grp> gs, bool sym = false) {
    const Quad qd = quad;
    quad = Quad{};
    const Chunked* oc = ochunk;
    ochunk = nullptr;
    if (n_out <= 0) return;
    SegParams sp{};
    if (oc) {
      sp.och = oc->table.p;
      sp.osh = oc->shift;
    }
    sp.oquad = qd.mq;
    sp.qm = qd.qm;
    sp.qn = qd.qn;
    sp.sym = sym ? 1 : 0;
    sp.out = out;
    sp.Os = Os;
    sp.Ooff = Ooff;
    sp.Old = Old;
    sp.omap = omap;
    sp.M = M;
    sp.N = N;
    sp.n_out = n_out;
    sp.accumulate = acc ? (c_prefetch ? 3 : 1) : 0;
    int ng = 0;
    for (const Grp& g : gs) {
      const int64_t entries = g.csr ? g.csr->entries : n_out;
      if (entries == 0) continue;
      if (ng >= kMaxGroups) throw std::logic_error("seg: too many groups");
      SegGroup& G = sp.g[ng++];
      G.L = g.L.p;
      G.Lch = g.L.ch;
      G.Lsh = g.L.sh;
      G.Rch = g.R.ch;
      G.Rsh = g.R.sh;
      G.Ls = g.L.s;
      G.Loff = g.L.off;
      G.Lld = g.L.ld;
      G.opL = g.L.op;
      G.R = g.R.p;
      G.Rs = g.R.s;
      G.Roff = g.R.off;
      G.Rld = g.R.ld;
      G.opR = g.R.op;
      G.K = g.K;
      if (g.csr) {
        G.ptr = g.csr->ptr;
        G.li = g.csr->li;
        G.ri = g.csr->ri;
      } else {
        G.ptr = nullptr;
        G.li = g.li;
        G.ri = g.ri;
      }
      exec_macs += entries * int64_t(M) * N * g.K / (sym ? 2 : 1);
    }
    sp.ngroups = ng;
    if (ng == 0 && acc) return;
    int64_t macs = 0;
    for (const Grp& g : gs) macs += (g.csr ? g.csr->entries : n_out) * int64_t(M) * N * g.K;
    if (sym) macs = macs / 2 + macs / (2 * ((M + 63) / 64));
    if (profiling && prof_shapes) {
      shape_tag = " [" + std::to_string(M) + "x" + std::to_string(N) + " K";
      int64_t ent = 0;
      for (const Grp& g : gs) {
        shape_tag += ":" + std::to_string(g.K);
        ent += g.csr ? g.csr->entries : n_out;
      }
      shape_tag += " e/out " + std::to_string(ent / std::max(1, n_out)) + " out " + std::to_string(n_out) + "]";
    }
    int64_t bytes = int64_t(n_out) * M * N * 8 * W * (acc ? 2 : 1);
    for (const Grp& g : gs) {
      const int64_t ent = g.csr ? g.csr->entries : n_out;
      bytes += ent * (int64_t(M) * g.K + int64_t(g.K) * N) * 8 * W;
    }
    {
      double ch = 0;
      for (const Grp& g : gs) ch += double(g.csr ? g.csr->entries : n_out) * (g.K / 8);
      cur_chunks = ch / n_out;
    }
    pre("seg_gemm", macs, bytes);
    if (sym && (M != N || acc)) throw std::logic_error("seg: symmetric launch needs a square, fresh output");
    // Outputs wider than one 64 tile whose last tile row / column would be at
    // most half full (e.g. a padded rank of 208 = 3*64 + 16): the full 64-tiles
    // and the remainder strip run as separate launches on shifted views, the
    // strip with a 16/32-wide tile class instead of a mostly-padding 64 tile.
    const int rm = M % 64, rn = N % 64;
    // outputs of 33..48 rows / columns as a 32-strip + a remainder strip (40 = 32 + 8) instead of
    // one mostly-padding 64 tile (profiles/r01/ab_strips_small.txt; H2B_NO_STRIPS_SMALL=1
    // disables, H2B_STRIPS_SMALL_MAX sets the largest remainder); H2B_STRIPS_24=1 also 17..24 as
    // 16 + remainder
    auto small_cut = [&](int X) {
      if (!strips_small || sym) return 0;
      if (X > 32 && X - 32 <= strips_small_max) return 32;
      if (strips_24 && X > 16 && X < 32 && X - 16 <= 8) return 16;
      return 0;
    };
    const int scM = small_cut(M), scN = small_cut(N);
    const bool smM = scM > 0, smN = scN > 0;
    const bool splitM = smM || (!sym && !no_strips && M > 64 && rm > 0 && rm <= 32);
    const bool splitN = smN || (!sym && !no_strips && N > 64 && rn > 0 && rn <= 32);
    if (!splitM && !splitN) {
      launch_tiles(sp);
    } else {
      const int cutM = smM ? scM : M - rm, cutN = smN ? scN : N - rn;
      const int mcuts[3] = {0, splitM ? cutM : M, M}, ncuts[3] = {0, splitN ? cutN : N, N};
      for (int a = 0; a < (splitM ? 2 : 1); ++a)
        for (int b = 0; b < (splitN ? 2 : 1); ++b) {
          const int r0 = mcuts[a], r1 = splitM ? mcuts[a + 1] : M;
          const int c0 = ncuts[b], c1 = splitN ? ncuts[b + 1] : N;
          SegParams q = sp;
          q.M = r1 - r0;
          q.N = c1 - c0;
          q.Ooff = sp.Ooff + r0 + (long long)c0 * sp.Old;
          for (int g = 0; g < q.ngroups; ++g) {
            SegGroup& G = q.g[g];
            const bool lt = G.opL == OP_T || G.opL == OP_H, rt = G.opR == OP_T || G.opR == OP_H;
            G.Loff += lt ? (long long)r0 * G.Lld : r0;
            G.Roff += rt ? c0 : (long long)c0 * G.Rld;
          }
          launch_tiles(q);
        }
    }
    post();
  }
  // accumulating launches prefetch their output tile to L2 (H2B_NO_CPREFETCH=1: A/B)
  const bool c_prefetch = std::getenv("H2B_NO_CPREFETCH") == nullptr;
  const bool no_strips = std::getenv("H2B_NO_STRIPS") != nullptr;  // A/B: single launch per product
  const bool strips_small = std::getenv("H2B_NO_STRIPS_SMALL") == nullptr;
  const bool strips_24 = std::getenv("H2B_STRIPS_24") != nullptr;
  // largest remainder split off a 33..63-wide output (H2B_STRIPS_SMALL_MAX, default 16: 48 = 32 + 16)
  const int strips_small_max = [] {
    const char* e = std::getenv("H2B_STRIPS_SMALL_MAX");
    return e ? std::atoi(e) : 16;
  }();
  // Hermitian (Gram) outputs cannot be cut into strips; their square tile is chosen by
  // lower-triangle tile area / relative tile efficiency (64: 1, 32: 0.75): e.g. an 80 x 80 Gram
  // takes 6 tiles of 32 (6,144 padded elements) instead of 3 of 64 (12,288, 26 % useful).
  // H2B_SYM_T64=1 restores the plain rule.
  const bool sym_t64 = std::getenv("H2B_SYM_T64") != nullptr;
  // relative efficiency assumed for the 32-tile kernel: 0.75 for real products (round 1, neutral
  // either way); 1.0 for complex ones - the 3-product 64 x 64 instantiation runs 2 CTAs per SM at
  // 249 registers, the 32 x 32 one 5, and lower triangles of 32-tiles carry up to 25 % less padding:
  // configs[4] 1.566 -> 1.538 s (profiles/r02/ab_small_maxch_sym_tile.json).  H2B_SYM_EFF32: A/B.
  static int sym_tile(int M, bool cplx) {
    if (M <= 32) return M <= 16 ? 16 : 32;
    static const double eff_env = [] {
      const char* e = std::getenv("H2B_SYM_EFF32");
      return e ? std::atof(e) : 0.0;
    }();
    const double eff32 = eff_env > 0.0 ? eff_env : (cplx ? 1.0 : 0.75);
    auto cost = [&](int T, double eff) {
      const double t = (M + T - 1) / T;
      return t * (t + 1) / 2 * T * T / eff;
    };
    return cost(32, eff32) < cost(64, 1.0) ? 32 : 64;
  }
  // seg_small (kernels.cuh): one warp per output, for outputs of at most 12 m8n8 fragments (e.g.
  // 24 x 32; a 32 x 32 output needs 126 registers per lane and measured slower than seg_gemm3).
  // Real products: sums of at most 4 8-deep k-chunks per output on average (48 for outputs of one
  // or two fragments) - beyond that seg_gemm3's asynchronous pipeline wins; complex products
  // (16-byte fragment loads): every such output.  profiles/r02/ab_seg_small.txt;
  // H2B_SMALL_MAXCH overrides the chunk bound (0 disables the kernel).
  const int small_max_chunks = [] {
    const char* e = std::getenv("H2B_SMALL_MAXCH");
    return e ? std::atoi(e) : -1;
  }();
  bool use_small(const SegParams& sp) const {
    const int M = sp.M, N = sp.N;
    if (sp.sym || M > 32 || N > 32 || M % 8 != 0 || N % 8 != 0 || M * N > 32 * 24) return false;
    if (small_max_chunks >= 0) return cur_chunks <= small_max_chunks;
    if (cplx) return true;
    return cur_chunks <= (M * N <= 128 ? 48 : 4);
  }
  double cur_chunks = 1e30;  // average k-chunks per output of the launch being issued
  template <int FM, int FN>
  void launch_small_cfg(const SegParams& sp) {
    const dim3 grid((sp.n_out + 3) / 4);
    if (cplx) seg_small_kernel<FM, FN, true><<<grid, 128, 0, s>>>(sp);
    else seg_small_kernel<FM, FN, false><<<grid, 128, 0, s>>>(sp);
    CK(cudaGetLastError());
    launches++;
  }
  template <int FM>
  void launch_small_n(const SegParams& sp) {
    switch (sp.N / 8) {
      case 1: launch_small_cfg<FM, 1>(sp); break;
      case 2: launch_small_cfg<FM, 2>(sp); break;
      case 3: launch_small_cfg<FM, 3>(sp); break;
      default: launch_small_cfg<FM, 4>(sp); break;
    }
  }
  void launch_tiles(const SegParams& sp) {
    const int M = sp.M, N = sp.N;
    if (use_small(sp)) {
      switch (M / 8) {
        case 1: launch_small_n<1>(sp); break;
        case 2: launch_small_n<2>(sp); break;
        case 3: launch_small_n<3>(sp); break;
        default: launch_small_n<4>(sp); break;
      }
      return;
    }
    int TM = M <= 8 ? 8 : M <= 16 ? 16 : (M <= 32 ? 32 : 64);
    int TN = N <= 8 ? 8 : N <= 16 ? 16 : (N <= 32 ? 32 : 64);
    if (sp.sym && !sym_t64 && M > 32) TM = TN = sym_tile(M, cplx);
    const int tm_ = (M + TM - 1) / TM;
    const int tiles = sp.sym ? tm_ * (tm_ + 1) / 2 : tm_ * ((N + TN - 1) / TN);
    if (TM == 8 || TN == 8) {
      if (TM == 8 && TN == 8) launch_seg8<8, 8, 1, 1>(sp, tiles);
      else if (TM == 8 && TN == 16) launch_seg8<8, 16, 1, 2>(sp, tiles);
      else if (TM == 8 && TN == 32) launch_seg8<8, 32, 1, 4>(sp, tiles);
      else if (TM == 8) launch_seg8<8, 64, 1, 4>(sp, tiles);
      else if (TM == 16) launch_seg8<16, 8, 2, 1>(sp, tiles);
      else if (TM == 32) launch_seg8<32, 8, 4, 1>(sp, tiles);
      else launch_seg8<64, 8, 4, 1>(sp, tiles);
      return;
    }
    if (TM == 16 && TN == 16) launch_seg<16, 16>(sp, tiles);
    else if (TM == 16 && TN == 32) launch_seg<16, 32>(sp, tiles);
    else if (TM == 16 && TN == 64) launch_seg<16, 64>(sp, tiles);
    else if (TM == 32 && TN == 16) launch_seg<32, 16>(sp, tiles);
    else if (TM == 32 && TN == 32) launch_seg<32, 32>(sp, tiles);
    else if (TM == 32 && TN == 64) launch_seg<32, 64>(sp, tiles);
    else if (TM == 64 && TN == 16) launch_seg<64, 16>(sp, tiles);
    else if (TM == 64 && TN == 32) launch_seg<64, 32>(sp, tiles);
    else launch_seg<64, 64>(sp, tiles);
  }
  // convenience: densely stored output [n_out][M x N]
  void segd(double* out, int M, int N, int n_out, std::initializer_list<Grp> gs) {
    seg(out, (long long)M * N, 0, M, nullptr, M, N, n_out, false, gs);
  }
  // Hermitian outputs (Gram sums): lower tiles only, mirrored in the epilogue
  void segh(double* out, int M, int n_out, std::initializer_list<Grp> gs) {
    seg(out, (long long)M * M, 0, M, nullptr, M, M, n_out, false, gs, true);
  }

  static Ref ref(const double* p, long long stride, int ld, int op, long long off = 0) {
    return Ref{p, stride, off, ld, op};
  }
  static Ref cref(const Chunked& c, long long stride, int ld, int op, long long off = 0) {
    return Ref{nullptr, stride, off, ld, op, c.table.p, c.shift};
  }

  void seg_add(double* out, long long Os, const double* in, long long Is, const DevCsr& c, long long elems) {
    if (c.n_out <= 0) return;
    const int chunks = static_cast<int>(std::min<long long>(8, (elems / 2 + 255) / 256));
    pre("seg_add", 0, (c.entries + c.n_out) * elems * 8 * W);
    seg_add_kernel<<<dim3(c.n_out, std::max(1, chunks)), 256, 0, s>>>(out, Os * W, in, Is * W, c.ptr, c.li,
                                                                      elems * W, 0);
    CK(cudaGetLastError());
    post();
    launches++;
  }

  // combine three Grams and truncate; returns device arrays of ranks/flags and
  // the sorted eigenvector buffer (n x n per cluster)
  struct Trunc {
    DBuf vec, val;
    DVec<int32_t> rank;
    DVec<uint8_t> degen;
    DBuf G;  // eigensolve input (deferred library solve / kept until the solve is joined)
    DBuf hV, hZ, hSlab;  // heev workspaces
    DVec<int> fail;      // heev: a QL iteration did not converge
    bool side = false;   // solved on side stream 1 (joined in finish_side)
    int n = 0, count = 0;
  };
  Trunc truncate(DBuf& g1, DBuf& g2, DBuf& g3, int count, int n, const DVec<uint8_t>& opdeg, bool defer = false) {
    Trunc t;
    DBuf G(sz(count, n, n), s);
    t.degen.alloc(count, s);
    pre("gram_combine", 0, 4LL * count * n * n * 8 * W);
    // few large Grams (upper levels): spread each over P CTAs (two passes)
    const int P = static_cast<int>(std::min<long long>(std::max(1, 1184 / std::max(count, 1)),
                                                       std::max<long long>(1, (long long)n * n * W / 4096)));
    if (P > 1) {
      DBuf part(size_t(count) * P * 3, s);
      const dim3 grid(count, P);
      if (cplx) {
        gram_norm_partial_kernel<true><<<grid, 256, 0, s>>>(g1, g2, g3, (long long)n * n, n * n, part.p);
        gram_combine_grid_kernel<true><<<grid, 256, 0, s>>>(g1, g2, g3, G, (long long)n * n, n * n, part.p, opdeg.p,
                                                            t.degen.p);
      } else {
        gram_norm_partial_kernel<false><<<grid, 256, 0, s>>>(g1, g2, g3, (long long)n * n, n * n, part.p);
        gram_combine_grid_kernel<false><<<grid, 256, 0, s>>>(g1, g2, g3, G, (long long)n * n, n * n, part.p, opdeg.p,
                                                             t.degen.p);
      }
      launches++;
    } else if (cplx) {
      gram_combine_kernel<true><<<count, 256, 0, s>>>(g1, g2, g3, G, (long long)n * n, n * n, opdeg.p, nullptr, t.degen.p);
    } else {
      gram_combine_kernel<false><<<count, 256, 0, s>>>(g1, g2, g3, G, (long long)n * n, n * n, opdeg.p, nullptr, t.degen.p);
    }
    CK(cudaGetLastError());
    post();
    launches++;
    g1.release();
    g2.release();
    g3.release();
    t.vec.alloc(sz(count, n, n), s);
    t.val.alloc(size_t(count) * n, s);
    t.rank.alloc(count, s);
    // the engine's own solver (heev.cuh); a deferred (row-side) solve runs on side stream 1,
    // concurrently with the column side, and is joined in finish_side
    cudaStream_t st = s;
    if (defer) {
      st = static_cast<cudaStream_t>(ctx.side_stream(1));
      t.side = true;
    }
    heev(G, count, n, t, st);
    t.G = std::move(G);  // input kept alive until the (possibly deferred) solve is joined
    t.n = n;
    t.count = count;
    return t;
  }

  // the upper levels' row and column truncations run concurrently (side stream 1 + main)
  bool paired_solves = false;

  // Batched Hermitian eigensolver + truncation rule (heev.cuh).  Placement per launch, from
  // tools/heev_bench.cu on the B200 (profiles/r02/heev_*.txt):
  //  * n <= 96 (leaf Grams): one CTA per Gram, Gram in shared memory (2-3 CTAs per SM);
  //  * 12 Grams or more (the batched middle levels): the Gram in a global (L2-resident) slab and
  //    ~20-50 KB of shared memory, one CTA per Gram when there are enough Grams to fill the SMs,
  //    else a cluster of 2 or 4 CTAs per Gram (column slabs, one wave of CTAs);
  //  * few large Grams: a cluster of CS CTAs per Gram (CS the smallest power of two whose
  //    column slabs fit the CTAs' shared memory, <= 16; global slabs beyond).
  // Workspaces come from the main-stream arena before the fork.
  void heev(const DBuf& G, int count, int n, Trunc& t, cudaStream_t st) {
    constexpr int kMaxSmem = 232448;
    int CS = 0;
    bool smem = true;
    for (int cs : {1, 2, 4, 8, 16}) {
      if (HeevLayout(n, cs, cplx, true).total * 8 <= kMaxSmem) {
        CS = cs;
        break;
      }
    }
    if (!CS) {
      CS = 16;
      smem = false;
    }
    // the row and column solves of a level run concurrently: size the decision on both.
    // From 12 Grams on, global slabs with the largest power-of-two cluster of at most 4 CTAs that
    // still gives one wave of CTAs (eff * CS <= 160): e.g. 32 Grams of n = 624 take 26 ms with
    // CS = 4 against 63 ms on 16-CTA shared-memory clusters and 79 ms with one CTA each; 64 Grams
    // of n = 576 41 ms with CS = 2 against 72 ms with CS = 1; 16 Grams of n = 464 13 ms with CS = 4
    // against 18 ms with CS = 8 and 22 ms on 16-CTA shared-memory clusters (8-CTA global-slab
    // clusters never won; profiles/r02/heev_sweep.txt, heev_sweep2.txt).
    const int eff = paired_solves ? 2 * count : count;
    if (n > 96 && eff >= 12) {
      CS = 1;
      while (CS < 4 && eff * CS * 2 <= 160) CS *= 2;
      smem = false;
    }
    const HeevLayout L(n, CS, cplx, smem);
    const int nt = n <= 64 ? 128 : (n <= 192 ? 256 : 512);
    const size_t bytes = size_t(L.total) * 8;
    t.hV.alloc(sz(count, n, n), s);
    t.hZ.alloc(size_t(count) * n * n, s);
    if (!smem) t.hSlab.alloc(size_t(count) * CS * L.ncl * L.ld * W, s);
    t.fail.alloc(1, s);
    CK(cudaMemsetAsync(t.fail.p, 0, sizeof(int), s));
    if (st != s) {
      CK(cudaEventRecord(ev_fork, s));
      CK(cudaStreamWaitEvent(st, ev_fork, 0));
    }
    HeevParams hp{};
    hp.G = G.p;
    hp.V = t.hV.p;
    hp.Zs = t.hZ.p;
    hp.slab = t.hSlab.p;
    hp.vec_out = t.vec.p;
    hp.val_out = t.val.p;
    hp.rank_out = t.rank.p;
    hp.degen_io = t.degen.p;
    hp.fail = t.fail.p;
    hp.n = n;
    hp.eps = jp_eps();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(count) * CS);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    auto go = [&](auto kern) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CK(cudaLaunchKernelEx(&cfg, kern, hp));
    };
    const bool main = st == s;
    // profile estimate: ~8/3 n^3 MACs per Gram (tridiagonalisation + back-transformation) over
    // ~n^3 scalars of trailing-matrix traffic (two reads and one write per Householder step):
    // 0.67 flop/B, a memory-bound kernel by the roofline model (its passes are L2 / latency bound)
    if (main)
      pre("heev", int64_t(count) * int64_t(8.0 / 3.0 * double(n) * n * n),
          int64_t(count) * int64_t(double(n) * n * n) * 8 * W);
    if (cplx) {
      if (smem) go(heev_kernel<true, true>);
      else go(heev_kernel<true, false>);
    } else {
      if (smem) go(heev_kernel<false, true>);
      else go(heev_kernel<false, false>);
    }
    CK(cudaGetLastError());
    if (main) post();
    launches++;
  }

  // Runs a deferred library eigensolve on side stream 1 in a host thread, so
  // the row and column eigensolves of a level overlap (cuSOLVER's batched
  // solver is launch-latency bound).
  // joins the row-side eigensolve (heev on side stream 1): the main stream waits for it
  void finish_side(Trunc& t) {
    if (t.side) {
      CK(cudaEventRecord(ev_side, static_cast<cudaStream_t>(ctx.side_stream(1))));
      CK(cudaStreamWaitEvent(s, ev_side, 0));
      t.side = false;
    }
    t.G.release();
  }
  double jp_eps() const { return adaptive ? eps : 0.5; }

  // H2B_DEBUG_CHECK=1: host check of the truncation output (orthonormal kept columns)
  void check_trunc(const Trunc& t, int count, int n) {
    std::vector<double> v(sz(count, n, n));
    std::vector<int> r(count);
    std::vector<double> ev(size_t(count) * n);
    CK(cudaMemcpyAsync(ev.data(), t.val.p, ev.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v.data(), t.vec.p, v.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(r.data(), t.rank.p, count * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double worst = 0;
    int rmin = 1 << 30, rmax = 0;
    for (int b = 0; b < count; ++b) {
      rmin = std::min(rmin, r[b]);
      rmax = std::max(rmax, r[b]);
      const double* V = v.data() + size_t(b) * n * n * W;
      for (int i = 0; i < r[b]; ++i)
        for (int j = 0; j <= i; ++j) {
          double re = 0, im = 0;
          for (int k = 0; k < n; ++k) {
            if (W == 1) re += V[k + size_t(i) * n] * V[k + size_t(j) * n];
            else {
              const double ar = V[2 * (k + size_t(i) * n)], ai = V[2 * (k + size_t(i) * n) + 1];
              const double br = V[2 * (k + size_t(j) * n)], bi = V[2 * (k + size_t(j) * n) + 1];
              re += ar * br + ai * bi;
              im += ar * bi - ai * br;
            }
          }
          worst = std::max(worst, std::hypot(re - (i == j ? 1.0 : 0.0), im));
        }
    }
    double margin = 1e300;
    const double e_ = jp_eps();
    for (int b = 0; b < count; ++b) {
      const double top = ev[size_t(b) * n];
      for (int i = 0; i < n; ++i) {
        const double l = ev[size_t(b) * n + i];
        if (l > 0 && top > 0) margin = std::min(margin, std::abs(l - e_ * top) / (e_ * top));
      }
    }
    std::fprintf(stderr, "[check] %s n=%d count=%d rank[%d,%d] orth_defect=%.3e min_margin=%.3e\n", phase.c_str(), n,
                 count, rmin, rmax, worst, margin);
  }

  // ranks to host, padded width (and the solver's convergence flag)
  int fetch_ranks(const Trunc& t, int count, std::vector<int64_t>& out) {
    const DVec<int32_t>& r = t.rank;
    std::vector<int32_t> h(count);
    int failed = 0;
    CK(cudaMemcpyAsync(h.data(), r.p, count * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (t.fail.p) CK(cudaMemcpyAsync(&failed, t.fail.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (failed) throw std::logic_error("svd_truncate_gram: eigendecomposition failed (QL iteration did not converge)");
    out.assign(h.begin(), h.end());
    int64_t mx = 0;
    for (auto v : out) mx = std::max(mx, v);
    return pad8(mx);
  }

  void pack(const Trunc& t, int count, int n, DBuf& out, int rows, int kc) {
    if (debug_check) check_trunc(t, count, n);
    out.alloc(sz(count, rows, kc), s);
    pre("pack_basis", 0);
    pack_basis_kernel<<<count, 256, 0, s>>>(t.vec, n, out, rows, kc, t.rank.p, W);
    CK(cudaGetLastError());
    post();
    launches++;
  }

  void identity(DBuf& out, int count, int n, const DVec<int32_t>& rank) {
    out.alloc(sz(count, n, n), s);
    set_identity_kernel<<<count, 256, 0, s>>>(out, n, n, rank.p, W);
    CK(cudaGetLastError());
    launches++;
  }

  void copy_dev(DBuf& dst, const DBuf& src) {
    dst.alloc(src.n, s);
    CK(cudaMemcpyAsync(dst.p, src.p, src.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }

  // ---- basis products B_j = (V^A_col,j)^T V^B_row,j (mmp.cpp:106-124) --------
  void basis_products() {
    mark("basis_products");
    const LevelPlan& LL = P.lv[D];
    Bp[D].alloc(sz(LL.n, A.Kc[D], B.Kr[D]), s);
    segd(Bp[D], A.Kc[D], B.Kr[D], LL.n,
         {Grp{ref(A.Vc, (long long)NL * A.Kc[D], NL, OP_T), ref(B.Vr, (long long)NL * B.Kr[D], NL, OP_N), NL,
              nullptr, nullptr, nullptr}});
    for (int l = D - 1; l >= 1; --l) {
      const int n = P.lv[l].n;
      const int ka1 = A.Kc[l + 1], kb1 = B.Kr[l + 1], ka = A.Kc[l], kb = B.Kr[l];
      DBuf tmp(sz(2 * size_t(n), ka, kb1), s);
      for (int c = 0; c < 2; ++c)  // tmp_c = (T^A_col[c])^T B_child(c)
        seg(tmp.p, (long long)ka * kb1, (long long)c * n * ka * kb1, ka, nullptr, ka, kb1, n, false,
            {Grp{ref(A.Tc[l], 2LL * ka1 * ka, 2 * ka1, OP_T, (long long)c * ka1),
                 ref(Bp[l + 1], (long long)ka1 * kb1, ka1, OP_N), ka1, nullptr, nullptr, c ? DP.odd : DP.even}});
      Bp[l].alloc(sz(n, ka, kb), s);
      segd(Bp[l], ka, kb, n,
           {Grp{ref(tmp, (long long)ka * kb1, ka, OP_N), ref(B.Tr[l], 2LL * kb1 * kb, 2 * kb1, OP_N), kb1, nullptr,
                nullptr, nullptr},
            Grp{ref(tmp, (long long)ka * kb1, ka, OP_N, (long long)n * ka * kb1),
                ref(B.Tr[l], 2LL * kb1 * kb, 2 * kb1, OP_N, kb1), kb1, nullptr, nullptr, nullptr}});
    }
  }

  // ---- admissible-block factors shared by leaf and upper levels --------------
  // SB = S^A B_j, LA = P^A SB ; BS = B_i S^B, RB = BS P^B  (mmp.cpp:325-332,389-390)
  // SB = S^A B_j per admissible block (independent of C)
  void make_sb(int l, DBuf& SB) {
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int na = static_cast<int>(L.adm.size());
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l];
    SB.alloc(sz(na, KAr, KBr), s);
    segd(SB, KAr, KBr, na,
         {Grp{ref(A.S[l], (long long)KAr * KAc, KAr, OP_N), ref(Bp[l], (long long)KAc * KBr, KAc, OP_N), KAc, nullptr,
              nullptr, Q.adm_col}});
  }

  void adm_factors(int l, DBuf& SB) {
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int na = static_cast<int>(L.adm.size());
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l], KBc = B.Kc[l], Kr = KCr[l], Kc = KCc[l];
    if (!SB.p) make_sb(l, SB);
    seg(LA[l], (long long)Kr * KBr, 0, Kr, Q.adm, Kr, KBr, na, false,
        {Grp{ref(PA[l], (long long)Kr * KAr, Kr, OP_N), ref(SB, (long long)KAr * KBr, KAr, OP_N), KAr, nullptr,
             Q.adm_row, nullptr}});
    DBuf BS(sz(na, KAc, KBc), s);
    segd(BS, KAc, KBc, na,
         {Grp{ref(Bp[l], (long long)KAc * KBr, KAc, OP_N), ref(B.S[l], (long long)KBr * KBc, KBr, OP_N), KBr, nullptr,
              Q.adm_row, nullptr}});
    seg(RB[l], (long long)KAc * Kc, 0, KAc, Q.adm, KAc, Kc, na, false,
        {Grp{ref(BS, (long long)KAc * KBc, KAc, OP_N), ref(PB[l], (long long)KBc * Kc, KBc, OP_N), KBc, nullptr,
             nullptr, Q.adm_col}});
  }

  // ---- coupling targets (mmp.cpp:319-334, 573-612) ----------------------------
  // The projections depend only on the target, so they leave the sum over j:
  //   T_ik = P^A_i (sum_RR S^A B_j S^B + ...) P^B_k
  //        = P^A_i [V1 P^B_k + U2] + U1 P^B_k (+ merged + leaf F x F)
  //   V1 = sum_{A,B adm} SB_ij S^B_jk,  U1 = sum_{A near} coll_a_ij S^B_jk,
  //   U2 = sum_{A adm, B near} S^A_ij coll_b_jk
  // Target slots of a level: [0, na) admissible, [na, na + np) pending, then NL.
  // The pending targets feed the parent level's merge (critical path) and run
  // on the main stream into Tp[l]; the admissible and NL targets are only read
  // by split() and the download, so they run on the low-priority auxiliary
  // stream into the compact store Tg[l] = [adm | NL], overlapping the parent
  // levels' Gram / eigensolver / collect chain.
  // output stores of level l's targets: Tg[l] = [adm | NL] and, for pending
  // targets, the parent's merged blocks Mg[l-1] (zero where a quadrant has no
  // child).  zero_tg: the targets accumulate onto case-1 values written first.
  void alloc_targets(int l, bool zero_tg) {
    alloc_tg(l, zero_tg);
    alloc_parent_merged(l);
  }
  void alloc_tg(int l, bool zero_tg) {
    const LevelPlan& L = P.lv[l];
    const int na = static_cast<int>(L.adm.size()), nl = static_cast<int>(L.nl_block.size());
    // the leaf targets sit with the other long-lived buffers at the top of the arena; an upper
    // level's targets are allocated from the bottom: the only long-lived buffer created since
    // this level's merged blocks is then below them, and the hole those leave when released
    // joins the free middle of the arena (the parent's merged blocks are the largest buffers
    // of a product: 70 GB at the 64^3 grid of configs[3])
    HighScope targets_placement(l == D);
    Tg[l].alloc(sz(na + nl, KCr[l], KCc[l]), s, zero_tg);
  }
  void alloc_parent_merged(int l) {
    if (P.lv[l].pend_row.empty()) return;
    const int nm = static_cast<int>(P.lv[l - 1].merged_row.size());
    HighScope merged_blocks_are_long_lived;
    Mg[l - 1].alloc(nm, (long long)sz(1, 2 * KCr[l], 2 * KCc[l]), s, true);
  }

  // case 1 of the upper levels (mmp.cpp:573-585): T^C_i^H M conj(T^C_k) of every
  // merged block, written into its target before the triple sums accumulate onto it; in
  // chunks (Zc = T^C_i^H M scratch).  pend = false: admissible targets, straight into their
  // Tg slots; pend = true: pending targets, into the compact store CP[e] (entry e of
  // mz_pend), which scatter_pending() later copies into the parent's merged quadrants —
  // so the merged blocks of this level are freed before the parent's are allocated
  // (at the 64^3 grid, configs[3], the two would not fit next to each other).
  void merged_into_targets(int l, const Chunked& M, bool pend, Chunked* CP) {
    const DevLevel& Q = DP.lv[l];
    const int Kn = KCr[l + 1], Kq = KCc[l + 1], Kr = KCr[l], Kc = KCc[l];
    const long long MM = 4LL * Kn * Kq;
    const DevLevel::MZ& z = pend ? Q.mz_pend : Q.mz_adm;
    if (z.n == 0) return;
    if (pend) CP->alloc(z.n, (long long)sz(1, Kr, Kc), s, false);
    const size_t per = sz(1, Kr, 2 * Kq) * sizeof(double);
    const int step = static_cast<int>(std::max<size_t>(4096, chunk_bytes() / per));
    for (int e0 = 0; e0 < z.n; e0 += step) {
      const int cnt = std::min(step, z.n - e0);
      DBuf Zc(sz(cnt, Kr, 2 * Kq), s);
      segd(Zc, Kr, 2 * Kq, cnt,
           {Grp{ref(Tr[l], 2LL * Kn * Kr, 2 * Kn, OP_H), cref(M, MM, 2 * Kn, OP_N), 2 * Kn, nullptr, z.row + e0,
                z.m + e0}});
      const Grp g{ref(Zc, 2LL * Kr * Kq, Kr, OP_N), ref(Tc[l], 2LL * Kq * Kc, 2 * Kq, OP_C), 2 * Kq, nullptr, nullptr,
                  z.col + e0};
      if (pend) {
        ochunk = CP;
        seg(nullptr, (long long)Kr * Kc, 0, Kr, DP.iota + e0, Kr, Kc, cnt, false, {g});
      }
      else seg(Tg[l], (long long)Kr * Kc, 0, Kr, z.out + e0, Kr, Kc, cnt, false, {g});
    }
  }
  // the compact pending case-1 values into their quadrants of the parent's merged blocks
  void scatter_pending(int l, const Chunked& CP) {
    const DevLevel::MZ& z = DP.lv[l].mz_pend;
    if (z.n == 0) return;
    pre("scatter_quad", 0, 2LL * z.n * KCr[l] * KCc[l] * 8 * W);
    scatter_quad_kernel<<<z.n, 256, 0, s>>>(Mg[l - 1].table.p, Mg[l - 1].shift, CP.table.p, CP.shift, z.out,
                                            KCr[l], KCc[l], W);
    CK(cudaGetLastError());
    post();
    launches++;
  }

  // acc: accumulate onto the stores (upper levels, after merged_into_targets)
  void targets(int l, const DBuf& SB, const DBuf* WA, const DBuf* WB, bool acc) {
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int na = static_cast<int>(L.adm.size()), np = static_cast<int>(L.pend_row.size());
    const int nl = static_cast<int>(L.nl_block.size());
    if (np > 0)  // pending targets straight into the parent's merged blocks (critical path)
      chunks(l, na, np, [&](int t0, int cnt) {
        targets_range(l, t0, cnt, nullptr, 0, SB, WA, WB, acc, Q.pend_mq + (t0 - na), &Mg[l - 1]);
      });
    auto rest = [&] {
      chunks(l, 0, na, [&](int t0, int cnt) { targets_range(l, t0, cnt, Tg[l], t0, SB, WA, WB, acc); });
      chunks(l, na + np, nl, [&](int t0, int cnt) { targets_range(l, t0, cnt, Tg[l], t0 - np, SB, WA, WB, acc); });
    };
    if (!defer_targets) rest();  // (profiling runs serialise: clean per-kernel timings)
    else on_aux(phase + "_deferred", rest);
  }

  size_t chunk_bytes() const {
    if (!t_arena) return kChunkBytes;
    const size_t fr = t_arena->stats().first;
    return std::max<size_t>(size_t(512) << 20, std::min(kChunkBytes, fr / 24));
  }
  // target ranges in chunks that bound the per-target scratch (V1, U1, U2) to chunk_bytes() each
  template <class Fn>
  void chunks(int l, int t0, int cnt, Fn&& fn) {
    const size_t per = size_t(W) * sizeof(double) *
                       std::max({size_t(A.Kr[l]) * B.Kc[l], size_t(KCr[l]) * B.Kc[l], size_t(A.Kr[l]) * KCc[l]});
    const int step = static_cast<int>(std::max<size_t>(4096, chunk_bytes() / std::max<size_t>(per, 1)));
    for (int c = 0; c < cnt; c += step) fn(t0 + c, std::min(step, cnt - c));
  }

  // run `fn` on the auxiliary stream, ordered after everything issued so far on
  // the main stream; buffers it allocates are stream-ordered on the auxiliary
  // stream, main-stream inputs it reads must stay in `hold` until join().
  template <class Fn>
  void on_aux(const std::string& ph, Fn&& fn) {
    if (profiling) {  // profiled runs are serial: per-kernel event times without overlap
      const std::string keep_phase = phase;
      phase = ph;
      fn();
      phase = keep_phase;
      return;
    }
    CK(cudaEventRecord(ev_fork, s));
    CK(cudaStreamWaitEvent(s_aux, ev_fork, 0));
    cudaStream_t keep = s;
    const std::string keep_phase = phase;
    s = s_aux;
    phase = ph;
    try {
      fn();
    } catch (...) {
      s = keep;
      phase = keep_phase;
      throw;
    }
    s = keep;
    phase = keep_phase;
    joined = false;
  }

  static DevCsr sub_csr(const DevCsr& d, const Csr& h, int t0, int cnt) {
    DevCsr r;
    r.ptr = d.ptr ? d.ptr + t0 : nullptr;
    r.li = d.li;
    r.ri = d.ri;
    r.n_out = cnt;
    r.entries = h.ptr.empty() ? 0 : int64_t(h.ptr[t0 + cnt]) - h.ptr[t0];
    return r;
  }

  // coupling targets t0 .. t0+cnt-1 of level l into out slots slot0.. (mmp.cpp:319-334, 573-612)
  // The projections depend only on the target, so they leave the sum over j:
  //   T_ik = P^A_i (sum_RR S^A B_j S^B + ...) P^B_k
  //        = P^A_i [V1 P^B_k + U2] + U1 P^B_k (+ merged + leaf F x F)
  //   V1 = sum_{A,B adm} SB_ij S^B_jk,  U1 = sum_{A near} coll_a_ij S^B_jk,
  //   U2 = sum_{A adm, B near} S^A_ij coll_b_jk
  // oq: quadrant scatter of the outputs into merged 2x2 blocks (pending targets), else slots slot0..
  void targets_range(int l, int t0, int cnt, double* out, long long slot0, const DBuf& SB, const DBuf* WA,
                     const DBuf* WB, bool acc, const int* oq = nullptr, const Chunked* oc = nullptr) {
    if (cnt <= 0) return;
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l], KBc = B.Kc[l], Kr = KCr[l], Kc = KCc[l];
    const DevCsr lyr = sub_csr(Q.lyr, L.lyr, t0, cnt), lyn = sub_csr(Q.lyn, L.lyn, t0, cnt),
                 xr = sub_csr(Q.xr, L.xr, t0, cnt);
    const int* trow = Q.target_row + t0;
    const int* tcol = Q.target_col + t0;
    const Ref BS_ = ref(B.S[l], (long long)KBr * KBc, KBr, OP_N);
    DBuf V1(sz(cnt, KAr, KBc), s), U1(sz(cnt, Kr, KBc), s), U2(sz(cnt, KAr, Kc), s);
    segd(V1, KAr, KBc, cnt, {Grp{ref(SB, (long long)KAr * KBr, KAr, OP_N), BS_, KBr, &lyr, nullptr, nullptr}});
    segd(U1, Kr, KBc, cnt, {Grp{ref(LA[l], (long long)Kr * KBr, Kr, OP_N), BS_, KBr, &lyn, nullptr, nullptr}});
    segd(U2, KAr, Kc, cnt,
         {Grp{ref(A.S[l], (long long)KAr * KAc, KAr, OP_N), ref(RB[l], (long long)KAc * Kc, KAc, OP_N), KAc, &xr,
              nullptr, nullptr}});
    const Ref PBk = ref(PB[l], (long long)KBc * Kc, KBc, OP_N);
    seg(U2, (long long)KAr * Kc, 0, KAr, nullptr, KAr, Kc, cnt, true,
        {Grp{ref(V1, (long long)KAr * KBc, KAr, OP_N), PBk, KBc, nullptr, nullptr, tcol}});
    V1.release();
    const long long os = oq ? 4LL * Kr * Kc : (long long)Kr * Kc;
    const int old = oq ? 2 * Kr : Kr;
    if (oq) slot0 = 0;
    const Grp gA{ref(PA[l], (long long)Kr * KAr, Kr, OP_N), ref(U2, (long long)KAr * Kc, KAr, OP_N), KAr, nullptr,
                 trow, nullptr};
    const Grp gB{ref(U1, (long long)Kr * KBc, Kr, OP_N), PBk, KBc, nullptr, nullptr, tcol};
    quad = {oq, Kr, Kc};
    ochunk = oc;
    if (WA) {
      const DevCsr ww = sub_csr(Q.ww, L.ww, t0, cnt);
      seg(out, os, slot0 * os, old, nullptr, Kr, Kc, cnt, acc,
          {gA, gB,
           Grp{ref(*WA, (long long)Kr * NL, Kr, OP_N), ref(*WB, (long long)NL * Kc, NL, OP_N), NL, &ww, nullptr,
               nullptr}});
    } else {
      seg(out, os, slot0 * os, old, nullptr, Kr, Kc, cnt, acc, {gA, gB});
    }
  }

  // ---- leaf level (mmp.cpp:245-340) ------------------------------------------
  void leaf_phase() {
    const int l = D;
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int n = L.n, nn = static_cast<int>(L.nearb.size()), na = static_cast<int>(L.adm.size());
    const int nb = static_cast<int>(L.brow.size());
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l], KBc = B.Kc[l];
    const long long NN = (long long)NL * NL;
    const Ref AF = ref(A.F, NN, NL, OP_N), BF = ref(B.F, NN, NL, OP_N);
    auto op = [](Ref r, int o) { r.op = o; return r; };

    // F^A V^B_row,j and (V^A_col,i)^T F^B (reused by Grams, collects, full targets)
    DBuf FV(sz(nn, NL, KBr), s), VF(sz(nn, KAc, NL), s);
    segd(FV, NL, KBr, nn, {Grp{AF, ref(B.Vr, (long long)NL * KBr, NL, OP_N), NL, nullptr, nullptr, Q.near_col}});
    segd(VF, KAc, NL, nn, {Grp{ref(A.Vc, (long long)NL * KAc, NL, OP_T), BF, NL, nullptr, Q.near_row, nullptr}});
    DBuf SB;
    make_sb(l, SB);
    // full targets on the auxiliary stream, overlapping everything until split()
    on_aux("leaf.full_targets", [&] { leaf_full_targets(FV, VF, SB); });

    if (adaptive) {
      mark("leaf.row_gram");
      // row Grams (mmp.cpp:164-200)
      DBuf g1(sz(n, NL, NL), s), g2(sz(n, NL, NL), s), g3(sz(n, NL, NL), s);
      {
        DBuf O(sz(nn, NL, NL), s);
        segh(O, NL, nn, {Grp{BF, op(BF, OP_H), NL, nullptr, nullptr, nullptr}});
        DBuf H(sz(nn, NL, NL), s);
        seg_add(H, NN, O, NN, Q.hq, NN);
        O.release();
        DBuf Y(sz(nn, NL, NL), s);
        segd(Y, NL, NL, nn, {Grp{AF, ref(H, NN, NL, OP_N), NL, nullptr, nullptr, nullptr}});
        segh(g1, NL, n, {Grp{ref(Y, NN, NL, OP_N), op(AF, OP_H), NL, &Q.row_near, nullptr, nullptr}});
      }
      segh(g2, NL, n,
           {Grp{ref(FV, (long long)NL * KBr, NL, OP_N), ref(FV, (long long)NL * KBr, NL, OP_H), KBr, &Q.row_near,
                nullptr, nullptr}});
      segh(g3, NL, n,
           {Grp{ref(A.Vr, (long long)NL * KAr, NL, OP_N), ref(A.Vr, (long long)NL * KAr, NL, OP_H), KAr, nullptr,
                nullptr, nullptr}});
      Trunc tr = truncate(g1, g2, g3, n, NL, A.dgr_d[l]);
      mark("leaf.col_gram");
      // column Grams (mmp.cpp:202-238)
      DBuf c1(sz(n, NL, NL), s), c2(sz(n, NL, NL), s), c3(sz(n, NL, NL), s);
      {
        DBuf Kb(sz(nn, NL, NL), s);
        segh(Kb, NL, nn, {Grp{op(AF, OP_T), op(AF, OP_C), NL, nullptr, nullptr, nullptr}});
        DBuf H(sz(nn, NL, NL), s);
        seg_add(H, NN, Kb, NN, Q.hqc, NN);
        Kb.release();
        DBuf Y(sz(nn, NL, NL), s);
        segd(Y, NL, NL, nn, {Grp{op(BF, OP_T), ref(H, NN, NL, OP_N), NL, nullptr, nullptr, nullptr}});
        segh(c1, NL, n, {Grp{ref(Y, NN, NL, OP_N), op(BF, OP_C), NL, &Q.col_near, nullptr, nullptr}});
      }
      segh(c2, NL, n,
           {Grp{ref(VF, (long long)KAc * NL, KAc, OP_T), ref(VF, (long long)KAc * NL, KAc, OP_C), KAc, &Q.col_near,
                nullptr, nullptr}});
      segh(c3, NL, n,
           {Grp{ref(B.Vc, (long long)NL * KBc, NL, OP_N), ref(B.Vc, (long long)NL * KBc, NL, OP_H), KBc, nullptr,
                nullptr, nullptr}});
      Trunc tc = truncate(c1, c2, c3, n, NL, B.dgc_d[l]);
      mark("leaf.bases");
      KCr[l] = fetch_ranks(tr, n, rcr[l]);
      KCc[l] = fetch_ranks(tc, n, rcc[l]);
      pack(tr, n, NL, Vr, NL, KCr[l]);
      pack(tc, n, NL, Vc, NL, KCc[l]);
      dgr[l] = std::move(tr.degen);
      dgc[l] = std::move(tc.degen);
      // projections (mmp.cpp:275-279)
      PA[l].alloc(sz(n, KCr[l], KAr), s);
      segd(PA[l], KCr[l], KAr, n,
           {Grp{ref(Vr, (long long)NL * KCr[l], NL, OP_H), ref(A.Vr, (long long)NL * KAr, NL, OP_N), NL, nullptr,
                nullptr, nullptr}});
      PB[l].alloc(sz(n, KBc, KCc[l]), s);
      segd(PB[l], KBc, KCc[l], n,
           {Grp{ref(B.Vc, (long long)NL * KBc, NL, OP_T), ref(Vc, (long long)NL * KCc[l], NL, OP_C), NL, nullptr,
                nullptr, nullptr}});
    } else {
      // formatted product: C keeps A's row and B's column bases (mmp.cpp:253-256,265-268)
      formatted_bases(l);
      copy_dev(Vr, A.Vr);
      copy_dev(Vc, B.Vc);
      identity(PA[l], n, KAr, A.rr_d[l]);
      identity(PB[l], n, KBc, B.rc_d[l]);
    }
    const int Kr = KCr[l], Kc = KCc[l];

    mark("leaf.collect");
    // collected full blocks (mmp.cpp:287-298) and W factors of the F x F case
    LA[l].alloc(sz(nb, Kr, KBr), s);
    RB[l].alloc(sz(nb, KAc, Kc), s);
    seg(LA[l], (long long)Kr * KBr, 0, Kr, Q.nearb, Kr, KBr, nn, false,
        {Grp{ref(Vr, (long long)NL * Kr, NL, OP_H), ref(FV, (long long)NL * KBr, NL, OP_N), NL, nullptr, Q.near_row,
             nullptr}});
    seg(RB[l], (long long)KAc * Kc, 0, KAc, Q.nearb, KAc, Kc, nn, false,
        {Grp{ref(VF, (long long)KAc * NL, KAc, OP_N), ref(Vc, (long long)NL * Kc, NL, OP_C), NL, nullptr, nullptr,
             Q.near_col}});
    DBuf WA(sz(nn, Kr, NL), s), WB(sz(nn, NL, Kc), s);
    segd(WA, Kr, NL, nn, {Grp{ref(Vr, (long long)NL * Kr, NL, OP_H), AF, NL, nullptr, Q.near_row, nullptr}});
    segd(WB, NL, Kc, nn, {Grp{BF, ref(Vc, (long long)NL * Kc, NL, OP_C), NL, nullptr, nullptr, Q.near_col}});
    adm_factors(l, SB);

    mark("leaf.coupling_targets");
    alloc_targets(l, false);
    targets(l, SB, &WA, &WB, false);
    retire(std::move(WA));
    retire(std::move(WB));
    // the auxiliary stream still reads these: release after the join
    retire(std::move(FV));
    retire(std::move(VF));
    retire(std::move(SB));

  }

  // ---- leaf full targets (mmp.cpp:310-317) on the auxiliary stream ------------
  // C.full = FF + (sum FV S^B) V^B^T + V^A (sum S^A VF + (sum S^A B S^B) V^B^T).
  // Independent of C's bases, so it overlaps the Gram / eigensolver / upper
  // level pipeline of the main stream; split() joins it.
  void leaf_full_targets(const DBuf& FV, const DBuf& VF, const DBuf& SB) {
    const int l = D;
    const LevelPlan& L = P.lv[l];
    const DevLevel& Q = DP.lv[l];
    const int nn = static_cast<int>(L.nearb.size());
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l], KBc = B.Kc[l];
    const long long NN = (long long)NL * NL;
    const Ref AF = ref(A.F, NN, NL, OP_N), BF = ref(B.F, NN, NL, OP_N);
    phase = "leaf.full_targets";
    const Ref BS = ref(B.S[l], (long long)KBr * KBc, KBr, OP_N);
    {
      HighScope full_blocks_are_long_lived;
      F.alloc(sz(nn, NL, NL), s);
    }
    // in chunks of full blocks: bounded T2 / T4 / U scratch (kChunkBytes each)
    const size_t per = size_t(W) * sizeof(double) * std::max(size_t(NL) * KBc, size_t(KAr) * std::max(KBc, NL));
    const int step = static_cast<int>(std::max<size_t>(4096, chunk_bytes() / per));
    for (int t0 = 0; t0 < nn; t0 += step) {
      const int cnt = std::min(step, nn - t0);
      const DevCsr fr = sub_csr(Q.fr, L.fr, t0, cnt), rr = sub_csr(Q.rr, L.rr, t0, cnt),
                   rf = sub_csr(Q.rf, L.rf, t0, cnt), ff = sub_csr(Q.ff, L.ff, t0, cnt);
      DBuf T2(sz(cnt, NL, KBc), s), T4(sz(cnt, KAr, KBc), s), U(sz(cnt, KAr, NL), s);
      segd(T2, NL, KBc, cnt, {Grp{ref(FV, (long long)NL * KBr, NL, OP_N), BS, KBr, &fr, nullptr, nullptr}});
      segd(T4, KAr, KBc, cnt, {Grp{ref(SB, (long long)KAr * KBr, KAr, OP_N), BS, KBr, &rr, nullptr, nullptr}});
      segd(U, KAr, NL, cnt,
           {Grp{ref(A.S[l], (long long)KAr * KAc, KAr, OP_N), ref(VF, (long long)KAc * NL, KAc, OP_N), KAc, &rf,
                nullptr, nullptr},
            Grp{ref(T4, (long long)KAr * KBc, KAr, OP_N), ref(B.Vc, (long long)NL * KBc, NL, OP_T), KBc, nullptr,
                nullptr, Q.near_col + t0}});
      seg(F, NN, NN * t0, NL, nullptr, NL, NL, cnt, false,
          {Grp{AF, BF, NL, &ff, nullptr, nullptr},
           Grp{ref(T2, (long long)NL * KBc, NL, OP_N), ref(B.Vc, (long long)NL * KBc, NL, OP_T), KBc, nullptr,
               nullptr, Q.near_col + t0},
           Grp{ref(A.Vr, (long long)NL * KAr, NL, OP_N), ref(U, (long long)KAr * NL, KAr, OP_N), KAr, nullptr,
               Q.near_row + t0, nullptr}});
    }
  }

  void formatted_bases(int l) {
    KCr[l] = A.Kr[l];
    KCc[l] = B.Kc[l];
    rcr[l] = A.rr[l];
    rcc[l] = B.rc[l];
    dgr[l].upload(A.dgr[l], s);
    dgc[l].upload(B.dgc[l], s);
  }

  // ---- upper levels (mmp.cpp:555-613) ----------------------------------------
  void upper_level(int l) {
    const LevelPlan& L = P.lv[l];
    const LevelPlan& Lc = P.lv[l + 1];
    const DevLevel& Q = DP.lv[l];
    const int n = L.n, ns = static_cast<int>(L.nearb.size());
    const int nm = static_cast<int>(L.merged_row.size()), nb = static_cast<int>(L.brow.size());
    const int Kn = KCr[l + 1], Kq = KCc[l + 1];
    const int KAr1 = A.Kr[l + 1], KAc1 = A.Kc[l + 1], KBr1 = B.Kr[l + 1], KBc1 = B.Kc[l + 1];
    const int KAr = A.Kr[l], KAc = A.Kc[l], KBr = B.Kr[l], KBc = B.Kc[l];
    const long long MM = 4LL * Kn * Kq;

    mark("L" + std::to_string(l) + ".assemble");
    // merged children couplings and assembled collected blocks (mmp.cpp:344-404)
    Chunked Mg = std::move(this->Mg[l]);  // filled by level l+1's pending targets
    (void)Lc;
    (void)nm;
    // X = asm_a T^B_row (row Gram term 2, collect); Xc = asm_b^T T^A_col.  The 2x2 assembled
    // blocks asm_a / asm_b are never formed: each half of X sums its two quadrant products
    // straight from the children's collects, X rows ri = sum_ci LA[child (ri,ci)] T^B[rows ci]
    // (Xc rows ci = sum_ri RB[child (ri,ci)]^T T^A_col[rows ri]).
    DBuf X(sz(ns, 2 * Kn, KBr), s), Xc(sz(ns, 2 * Kq, KAc), s);
    for (int h = 0; h < 2; ++h) {
      seg(X, 2LL * Kn * KBr, (long long)h * Kn, 2 * Kn, nullptr, Kn, KBr, ns, false,
          {Grp{ref(LA[l + 1], (long long)Kn * KBr1, Kn, OP_N), ref(B.Tr[l], 2LL * KBr1 * KBr, 2 * KBr1, OP_N), KBr1,
               nullptr, Q.subq[2 * h + 0], Q.near_col},
           Grp{ref(LA[l + 1], (long long)Kn * KBr1, Kn, OP_N), ref(B.Tr[l], 2LL * KBr1 * KBr, 2 * KBr1, OP_N, KBr1),
               KBr1, nullptr, Q.subq[2 * h + 1], Q.near_col}});
      seg(Xc, 2LL * Kq * KAc, (long long)h * Kq, 2 * Kq, nullptr, Kq, KAc, ns, false,
          {Grp{ref(RB[l + 1], (long long)KAc1 * Kq, KAc1, OP_T), ref(A.Tc[l], 2LL * KAc1 * KAc, 2 * KAc1, OP_N), KAc1,
               nullptr, Q.subq[0 + h], Q.near_row},
           Grp{ref(RB[l + 1], (long long)KAc1 * Kq, KAc1, OP_T),
               ref(A.Tc[l], 2LL * KAc1 * KAc, 2 * KAc1, OP_N, KAc1), KAc1, nullptr, Q.subq[2 + h], Q.near_row}});
    }
    // still read by level l+1's deferred targets: released after the join
    retire(std::move(LA[l + 1]));
    retire(std::move(RB[l + 1]));

    if (adaptive) {
      mark("L" + std::to_string(l) + ".grams");
      // X3 = blkdiag(P^A_children) T^A_row ; X3c = blkdiag(P^B)^T conj(T^B_col) ; Y3 = blkdiag(P^B)^T T^B_col
      DBuf X3(sz(n, 2 * Kn, KAr), s), X3c(sz(n, 2 * Kq, KBc), s), Y3;
      for (int c = 0; c < 2; ++c) {
        seg(X3, 2LL * Kn * KAr, (long long)c * Kn, 2 * Kn, nullptr, Kn, KAr, n, false,
            {Grp{ref(PA[l + 1], (long long)Kn * KAr1, Kn, OP_N),
                 ref(A.Tr[l], 2LL * KAr1 * KAr, 2 * KAr1, OP_N, (long long)c * KAr1), KAr1, nullptr,
                 c ? DP.odd : DP.even, nullptr}});
        seg(X3c, 2LL * Kq * KBc, (long long)c * Kq, 2 * Kq, nullptr, Kq, KBc, n, false,
            {Grp{ref(PB[l + 1], (long long)KBc1 * Kq, KBc1, OP_T),
                 ref(B.Tc[l], 2LL * KBc1 * KBc, 2 * KBc1, OP_C, (long long)c * KBc1), KBc1, nullptr,
                 c ? DP.odd : DP.even, nullptr}});
      }
      if (cplx) {
        Y3.alloc(sz(n, 2 * Kq, KBc), s);
        for (int c = 0; c < 2; ++c)
          seg(Y3, 2LL * Kq * KBc, (long long)c * Kq, 2 * Kq, nullptr, Kq, KBc, n, false,
              {Grp{ref(PB[l + 1], (long long)KBc1 * Kq, KBc1, OP_T),
                   ref(B.Tc[l], 2LL * KBc1 * KBc, 2 * KBc1, OP_N, (long long)c * KBc1), KBc1, nullptr,
                   c ? DP.odd : DP.even, nullptr}});
      }
      // row transfer Gram (mmp.cpp:406-457)
      DBuf g1(sz(n, 2 * Kn, 2 * Kn), s), g2(sz(n, 2 * Kn, 2 * Kn), s), g3(sz(n, 2 * Kn, 2 * Kn), s);
      segh(g1, 2 * Kn, n,
           {Grp{cref(Mg, MM, 2 * Kn, OP_N), cref(Mg, MM, 2 * Kn, OP_H), 2 * Kq, &Q.row_merged, nullptr, nullptr}});
      segh(g2, 2 * Kn, n,
           {Grp{ref(X, 2LL * Kn * KBr, 2 * Kn, OP_N), ref(X, 2LL * Kn * KBr, 2 * Kn, OP_H), KBr, &Q.row_near,
                nullptr, nullptr}});
      segh(g3, 2 * Kn, n,
           {Grp{ref(X3, 2LL * Kn * KAr, 2 * Kn, OP_N), ref(X3, 2LL * Kn * KAr, 2 * Kn, OP_H), KAr, nullptr, nullptr,
                nullptr}});
      paired_solves = true;
      Trunc tr = truncate(g1, g2, g3, n, 2 * Kn, A.dgr_d[l], /*defer=*/true);
      // column transfer Gram (mmp.cpp:459-512)
      DBuf c1(sz(n, 2 * Kq, 2 * Kq), s), c2(sz(n, 2 * Kq, 2 * Kq), s), c3(sz(n, 2 * Kq, 2 * Kq), s);
      segh(c1, 2 * Kq, n,
           {Grp{cref(Mg, MM, 2 * Kn, OP_T), cref(Mg, MM, 2 * Kn, OP_C), 2 * Kn, &Q.col_merged, nullptr, nullptr}});
      segh(c2, 2 * Kq, n,
           {Grp{ref(Xc, 2LL * Kq * KAc, 2 * Kq, OP_N), ref(Xc, 2LL * Kq * KAc, 2 * Kq, OP_H), KAc, &Q.col_near,
                nullptr, nullptr}});
      segh(c3, 2 * Kq, n,
           {Grp{ref(X3c, 2LL * Kq * KBc, 2 * Kq, OP_N), ref(X3c, 2LL * Kq * KBc, 2 * Kq, OP_H), KBc, nullptr, nullptr,
                nullptr}});
      Trunc tc = truncate(c1, c2, c3, n, 2 * Kq, B.dgc_d[l]);
      finish_side(tr);
      paired_solves = false;
      KCr[l] = fetch_ranks(tr, n, rcr[l]);
      KCc[l] = fetch_ranks(tc, n, rcc[l]);
      pack(tr, n, 2 * Kn, Tr[l], 2 * Kn, KCr[l]);
      pack(tc, n, 2 * Kq, Tc[l], 2 * Kq, KCc[l]);
      dgr[l] = std::move(tr.degen);
      dgc[l] = std::move(tc.degen);
      // projections (mmp.cpp:515-537): P^A = T^C^H X3, P^B = Y3^T conj(T^C_col)
      PA[l].alloc(sz(n, KCr[l], KAr), s);
      segd(PA[l], KCr[l], KAr, n,
           {Grp{ref(Tr[l], 2LL * Kn * KCr[l], 2 * Kn, OP_H), ref(X3, 2LL * Kn * KAr, 2 * Kn, OP_N), 2 * Kn, nullptr,
                nullptr, nullptr}});
      PB[l].alloc(sz(n, KBc, KCc[l]), s);
      const double* y3 = cplx ? Y3.p : X3c.p;
      segd(PB[l], KBc, KCc[l], n,
           {Grp{ref(y3, 2LL * Kq * KBc, 2 * Kq, OP_T), ref(Tc[l], 2LL * Kq * KCc[l], 2 * Kq, OP_C), 2 * Kq, nullptr,
                nullptr, nullptr}});
    } else {
      formatted_bases(l);
      copy_dev(Tr[l], A.Tr[l]);
      copy_dev(Tc[l], B.Tc[l]);
      identity(PA[l], n, KAr, A.rr_d[l]);
      identity(PB[l], n, KBc, B.rc_d[l]);
    }
    retire(std::move(PA[l + 1]));
    retire(std::move(PB[l + 1]));
    Bp[l + 1].release();
    const int Kr = KCr[l], Kc = KCc[l];

    mark("L" + std::to_string(l) + ".collect");
    // collects of subdivided blocks (mmp.cpp:544-552)
    LA[l].alloc(sz(nb, Kr, KBr), s);
    RB[l].alloc(sz(nb, KAc, Kc), s);
    seg(LA[l], (long long)Kr * KBr, 0, Kr, Q.nearb, Kr, KBr, ns, false,
        {Grp{ref(Tr[l], 2LL * Kn * Kr, 2 * Kn, OP_H), ref(X, 2LL * Kn * KBr, 2 * Kn, OP_N), 2 * Kn, nullptr,
             Q.near_row, nullptr}});
    seg(RB[l], (long long)KAc * Kc, 0, KAc, Q.nearb, KAc, Kc, ns, false,
        {Grp{ref(Xc, 2LL * Kq * KAc, 2 * Kq, OP_T), ref(Tc[l], 2LL * Kq * Kc, 2 * Kq, OP_C), 2 * Kq, nullptr,
             nullptr, Q.near_col}});
    X.release();
    Xc.release();
    DBuf SB;
    adm_factors(l, SB);

    mark("L" + std::to_string(l) + ".targets");
    // case 1 over merged children couplings first (mmp.cpp:573-585), then the
    // triple sums of cases 2-4 accumulate onto the same stores
    Chunked CP;
    merged_into_targets(l, Mg, true, &CP);  // pending targets: compact, while only Mg[l] is live
    alloc_tg(l, true);
    merged_into_targets(l, Mg, false, nullptr);
    Mg.release();
    alloc_parent_merged(l);
    scatter_pending(l, CP);
    CP.release();
    targets(l, SB, nullptr, nullptr, true);
    retire(std::move(SB));
  }

  // ---- top-down split of non-leaf couplings (mmp.cpp:617-659) --------------
  void split() {
    join();
    restore(false);  // C's evicted leaf stores receive split contributions
    splitting = true;
    mark("split");
    for (int l = 1; l < D; ++l) {
      const LevelPlan& L = P.lv[l];
      const LevelPlan& Lc = P.lv[l + 1];
      const DevLevel& Q = DP.lv[l];
      const int nnl = static_cast<int>(L.nl_block.size());
      if (nnl == 0) continue;
      const int Kr = KCr[l], Kc = KCc[l], Kn = KCr[l + 1], Kq = KCc[l + 1];
      const long long first = (long long)L.adm.size() * Kr * Kc;  // compacted store: [adm | NL]
      DBuf Qb(sz(nnl, Kr, 2 * Kq), s);  // NL * T^C_col^T
      segd(Qb, Kr, 2 * Kq, nnl,
           {Grp{ref(Tg[l], (long long)Kr * Kc, Kr, OP_N, first), ref(Tc[l], 2LL * Kq * Kc, 2 * Kq, OP_T), Kc, nullptr,
                nullptr, Q.nl_col}});
      for (int q = 0; q < 4; ++q) {
        const int ri = q >> 1, ci = q & 1;
        const Ref TL = ref(Tr[l], 2LL * Kn * Kr, 2 * Kn, OP_N, (long long)ri * Kn);
        const Ref QR = ref(Qb, 2LL * Kr * Kq, Kr, OP_N, (long long)ci * Kq * Kr);
        if (Q.sp_n[q] > 0)
          seg(Tg[l + 1], (long long)Kn * Kq, 0, Kn, Q.sp_omap[q], Kn, Kq, Q.sp_n[q], true,
              {Grp{TL, QR, Kr, nullptr, Q.sp_prow[q], Q.sp_src[q]}});
        if (Q.sf_n[q] > 0) {  // leaf children: C.full += V^C_row contrib V^C_col^T
          const int m = Q.sf_n[q];
          DBuf Dn(sz(m, Kn, Kq), s), E(sz(m, Kn, NL), s);
          segd(Dn, Kn, Kq, m, {Grp{TL, QR, Kr, nullptr, Q.sf_prow[q], Q.sf_src[q]}});
          segd(E, Kn, NL, m,
               {Grp{ref(Dn, (long long)Kn * Kq, Kn, OP_N), ref(Vc, (long long)NL * Kq, NL, OP_T), Kq, nullptr, nullptr,
                    Q.sf_ccol[q]}});
          seg(F, (long long)NL * NL, 0, NL, Q.sf_near[q], NL, NL, m, true,
              {Grp{ref(Vr, (long long)NL * Kn, NL, OP_N), ref(E, (long long)Kn * NL, Kn, OP_N), Kn, nullptr,
                   Q.sf_crow[q], nullptr}});
        }
      }
      (void)Lc;
    }
  }

  void run() {
    defer_targets = !no_defer_env && !profiling;
    try {
      basis_products();
      leaf_phase();
      leaf_done = true;
      for (int l = D - 1; l >= 1; --l) upper_level(l);
      split();
      join();
      // evicted operand blocks are restored by the destructor, after C has been downloaded
    } catch (const CudaError& e) {
      throw CudaError(std::string(e.what()) + " [phase " + phase + "]");
    }
  }

  // ---- exact H^2 matrix-vector product Y = A X (h2_matrix.cpp:213-278) -----
  // X, Y: device [N x nv] column-major in the ORIGINAL ordering.  Forward
  // transform up the column tree, coupling products, backward transform down
  // the row tree, near field - each level one segmented batched launch.
  void mvp(const double* X, int nv, double* Y, const int* perm) {
    const LevelPlan& LL = P.lv[D];
    const int nL = LL.n;
    const int NV = pad8(nv);
    const int N = P.n_points;
    // leaf-blocked copies of x (tree order, padded NL x NV per leaf)
    DBuf XL(sz(nL, NL, NV), s, true), YL(sz(nL, NL, NV), s, true);
    DVec<int32_t> beg, sizes;
    {
      std::vector<int32_t> b(nL), z(nL);
      int at = 0;
      for (int p = 0; p < nL; ++p) {
        b[p] = at;
        z[p] = LL.size[p];
        at += LL.size[p];
      }
      beg.upload(b, s);
      sizes.upload(z, s);
    }
    mvp_gather_kernel<<<nL, 256, 0, s>>>(X, N, nv, perm, beg.p, sizes.p, XL, NL, NV, W);
    CK(cudaGetLastError());
    launches++;
    // forward: xhat_L = V_col^T x ; xhat_l = sum_s T_col[s]^T xhat_{l+1}[child s]
    std::vector<DBuf> xh(D + 1), yh(D + 1);
    xh[D].alloc(sz(nL, A.Kc[D], NV), s);
    segd(xh[D], A.Kc[D], NV, nL,
         {Grp{ref(A.Vc, (long long)NL * A.Kc[D], NL, OP_T), ref(XL, (long long)NL * NV, NL, OP_N), NL, nullptr,
              nullptr, nullptr}});
    for (int l = D - 1; l >= 1; --l) {
      const int n = P.lv[l].n, K = A.Kc[l], K1 = A.Kc[l + 1];
      xh[l].alloc(sz(n, K, NV), s);
      segd(xh[l], K, NV, n,
           {Grp{ref(A.Tc[l], 2LL * K1 * K, 2 * K1, OP_T), ref(xh[l + 1], (long long)K1 * NV, K1, OP_N), K1, nullptr,
                nullptr, DP.even},
            Grp{ref(A.Tc[l], 2LL * K1 * K, 2 * K1, OP_T, K1), ref(xh[l + 1], (long long)K1 * NV, K1, OP_N), K1,
                nullptr, nullptr, DP.odd}});
    }
    // couplings: yhat_l[i] = sum_{(i,j) adm} S_ij xhat_l[j]
    const int l0 = D == 0 ? 0 : 1;
    for (int l = l0; l <= D; ++l) {
      const int n = P.lv[l].n, Kr = A.Kr[l], Kc = A.Kc[l];
      yh[l].alloc(sz(n, Kr, NV), s);
      if (!xh[l].p) xh[l].alloc(sz(n, Kc, NV), s, true);
      segd(yh[l], Kr, NV, n,
           {Grp{ref(A.S[l], (long long)Kr * Kc, Kr, OP_N), ref(xh[l], (long long)Kc * NV, Kc, OP_N), Kc,
                &DP.lv[l].adm_by_row, nullptr, nullptr}});
    }
    // backward: yhat_{l+1}[child s] += T_row[s] yhat_l
    for (int l = l0; l < D; ++l) {
      const int n = P.lv[l].n, K = A.Kr[l], K1 = A.Kr[l + 1];
      for (int c = 0; c < 2; ++c)
        seg(yh[l + 1], (long long)K1 * NV, 0, K1, c ? DP.odd : DP.even, K1, NV, n, true,
            {Grp{ref(A.Tr[l], 2LL * K1 * K, 2 * K1, OP_N, (long long)c * K1), ref(yh[l], (long long)K * NV, K, OP_N),
                 K, nullptr, nullptr, nullptr}});
    }
    // leaves: y = V_row yhat + sum_full F x
    segd(YL, NL, NV, nL,
         {Grp{ref(A.Vr, (long long)NL * A.Kr[D], NL, OP_N), ref(yh[D], (long long)A.Kr[D] * NV, A.Kr[D], OP_N), A.Kr[D],
              nullptr, nullptr, nullptr},
          Grp{ref(A.F, (long long)NL * NL, NL, OP_N), ref(XL, (long long)NL * NV, NL, OP_N), NL,
              &DP.lv[D].near_by_row, nullptr, nullptr}});
    mvp_scatter_kernel<<<nL, 256, 0, s>>>(YL, NL, NV, perm, beg.p, sizes.p, Y, N, nv, W);
    CK(cudaGetLastError());
    launches++;
  }

  // ---- single Gram truncation on the device (truncation.cpp:9-47) ------------
  // The Gram is zero-padded to a multiple of 8 (padding adds exact zero
  // eigenvalues, never kept) and sent through the same path as the product's
  // Grams; g2 = g3 = 0 so the normalised sum is G/||G||_F (same eigenvectors,
  // same relative threshold).
  void truncate_one(const double* gram_host, int n, double* basis_host, int* rank, int* degenerate) {
    const int np = pad8(n);
    std::vector<double> g(size_t(np) * np * W, 0.0);
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r)
        for (int w = 0; w < W; ++w) g[(r + size_t(c) * np) * W + w] = gram_host[(r + size_t(c) * n) * W + w];
    DBuf g1(g.size(), s), g2(g.size(), s, true), g3(g.size(), s, true);
    CK(cudaMemcpyAsync(g1.p, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    DVec<uint8_t> opdeg;
    opdeg.upload(std::vector<uint8_t>{0}, s);
    Trunc t = truncate(g1, g2, g3, 1, np, opdeg);
    std::vector<double> v(size_t(np) * np * W);
    int rk = 0;
    uint8_t dg = 0;
    CK(cudaMemcpyAsync(v.data(), t.vec.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&rk, t.rank.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&dg, t.degen.p, 1, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < rk; ++c)
      for (int r = 0; r < n; ++r)
        for (int w = 0; w < W; ++w) basis_host[(r + size_t(c) * n) * W + w] = v[(r + size_t(c) * np) * W + w];
    *rank = rk;
    *degenerate = dg;
  }

  // per (phase, kernel) totals of the profiled launches
  void collect_profile(std::vector<ProfileEntry>& out) {
    out.clear();
    if (!profiling) return;
    CK(cudaStreamSynchronize(s));
    std::map<std::string, size_t> at;
    for (ProfRec& r : prof) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      const std::string key = r.phase + "/" + r.kernel;
      auto it = at.find(key);
      if (it == at.end()) {
        at[key] = out.size();
        out.push_back({key, 0, 0.0, 0, 0});
        it = at.find(key);
      }
      ProfileEntry& e = out[it->second];
      e.launches++;
      e.ms += ms;
      e.macs += r.macs;
      e.bytes += r.bytes;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    prof.clear();
    // phase wall times (main stream, gaps included)
    if (!marks.empty()) {
      cudaEvent_t end;
      CK(cudaEventCreate(&end));
      CK(cudaEventRecord(end, s));
      CK(cudaEventSynchronize(end));
      for (size_t i = 0; i < marks.size(); ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, marks[i].second, i + 1 < marks.size() ? marks[i + 1].second : end));
        out.push_back({"wall:" + marks[i].first, 1, ms, 0, 0});
      }
      for (size_t i = 0; i + 1 < host_marks.size(); ++i)
        out.push_back({"host:" + host_marks[i].first, 1, host_marks[i + 1].second - host_marks[i].second, 0, 0});
      host_marks.clear();
      for (auto& m : marks) cudaEventDestroy(m.second);
      cudaEventDestroy(end);
      marks.clear();
    }
  }

  // ---- output in the flat layout (row bases, col bases by id, then blocks) ----
  void download(const h2c_blocks& blocks, HostResult& out, std::vector<double*>& pinned_pool) {
    (void)pinned_pool;
    const int nc = static_cast<int>(P.n_clusters);
    out.scalar = cplx ? H2C_COMPLEX : H2C_REAL;
    out.row_rank.assign(nc, 0);
    out.col_rank.assign(nc, 0);
    out.row_dg.assign(nc, 0);
    out.col_dg.assign(nc, 0);
    out.row_off.assign(nc, -1);
    out.col_off.assign(nc, -1);
    out.block_off.assign(blocks.n_blocks, -1);
    std::vector<std::vector<uint8_t>> hr(D + 1), hc(D + 1);
    for (int l = (D == 0 ? 0 : 1); l <= D; ++l) {
      const int n = P.lv[l].n;
      hr[l].resize(n);
      hc[l].resize(n);
      CK(cudaMemcpyAsync(hr[l].data(), dgr[l].p, n, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hc[l].data(), dgc[l].p, n, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    int64_t total = 0;
    CopyList cl;
    struct Job {
      const double* src;
      int64_t dst;
      int rows, cols, sld, dld;
    };
    std::vector<Job> jobs;
    std::vector<int> lev(nc, 0);
    for (int m = 0; m <= D; ++m)
      for (int id : P.lv[m].id) lev[id] = m;
    for (int side = 0; side < 2; ++side)
      for (int id = 0; id < nc; ++id) {
        const int m = lev[id], p = P.pos_of[id];
        if (m == 0 && D > 0) continue;  // the non-leaf root carries no basis
        auto& rk = side == 0 ? rcr : rcc;
        const int r = static_cast<int>(rk[m][p]);
        (side == 0 ? out.row_rank : out.col_rank)[id] = r;
        (side == 0 ? out.row_dg : out.col_dg)[id] = (side == 0 ? hr : hc)[m][p];
        (side == 0 ? out.row_off : out.col_off)[id] = total;
        if (m == D) {
          const int K = side == 0 ? KCr[D] : KCc[D];
          const double* src = (side == 0 ? Vr.p : Vc.p) + size_t(p) * NL * K * W;
          const int rows = P.lv[D].size[p];
          jobs.push_back({src, total, rows, r, NL, rows});
          total += int64_t(rows) * r;
        } else {
          const int K1 = side == 0 ? KCr[m + 1] : KCc[m + 1];
          const int K0 = side == 0 ? KCr[m] : KCc[m];
          const int c0 = static_cast<int>(rk[m + 1][2 * p]), c1 = static_cast<int>(rk[m + 1][2 * p + 1]);
          const double* base = (side == 0 ? Tr[m].p : Tc[m].p) + size_t(p) * 2 * K1 * K0 * W;
          // stacked [T_c1; T_c2] of shape (c0 + c1) x r from the two padded row slots
          jobs.push_back({base, total, c0, r, 2 * K1, c0 + c1});
          jobs.push_back({base + size_t(K1) * W, total + c0, c1, r, 2 * K1, c0 + c1});
          total += int64_t(c0 + c1) * r;
        }
      }
    // blocks in global order
    std::vector<std::pair<int, int>> where(blocks.n_blocks, {-1, -1});
    for (int m = 0; m <= D; ++m)
      for (size_t b = 0; b < P.lv[m].bglobal.size(); ++b) where[P.lv[m].bglobal[b]] = {m, static_cast<int>(b)};
    for (int64_t g = 0; g < blocks.n_blocks; ++g) {
      const auto [m, b] = where[g];
      const LevelPlan& L = P.lv[m];
      if (L.bkind[b] == kAdm) {
        const int a = L.kidx[b];
        const int rr = static_cast<int>(rcr[m][L.brow[b]]), rc = static_cast<int>(rcc[m][L.bcol[b]]);
        out.block_off[g] = total;
        jobs.push_back({Tg[m].p + size_t(a) * KCr[m] * KCc[m] * W, total, rr, rc, KCr[m], rr});
        total += int64_t(rr) * rc;
      } else if (L.bkind[b] == kFull) {
        const int q = L.kidx[b];
        const int nr = L.size[L.brow[b]], ncl = L.size[L.bcol[b]];
        out.block_off[g] = total;
        jobs.push_back({F.p + size_t(q) * NL * NL * W, total, nr, ncl, NL, nr});
        total += int64_t(nr) * ncl;
      }
    }
    (void)cl;
    out.n_values = total;
    out.pool = ctx.pinned;
    out.values = out.pool->take(std::max<size_t>(1, size_t(total) * W * sizeof(double)), &out.values_bytes);
    // pack into the flat layout through a bounded device buffer (jobs are in destination order),
    // so the download never needs one allocation of C's full size next to the run's buffers
    auto dext = [](const Job& j) { return int64_t(j.cols - 1) * j.dld + j.rows; };  // span in the flat array
    int64_t span_max = 0;
    for (const Job& j : jobs) span_max = std::max(span_max, dext(j));
    const int64_t cap = std::max<int64_t>(stage_scalars(), span_max);  // scalars per batch
    // (+ span_max: a job whose span interleaves with the previous one's - the two halves of a
    // stacked transfer - always joins its batch)
    DBuf flat(size_t(std::min<int64_t>(std::max<int64_t>(total, 1), cap + span_max)) * W, s);
    int64_t dl = 0;
    for (size_t i = 0; i < jobs.size();) {
      const int64_t d0 = jobs[i].dst;
      size_t e = i;
      int64_t d1 = d0;
      while (e < jobs.size() && (jobs[e].dst < d1 || std::max(d1, jobs[e].dst + dext(jobs[e])) - d0 <= cap)) {
        d1 = std::max(d1, jobs[e].dst + dext(jobs[e]));
        ++e;
      }
      CopyList bl;
      for (size_t q = i; q < e; ++q)
        bl.add(jobs[q].src, flat.p + (jobs[q].dst - d0) * W, jobs[q].rows, jobs[q].cols, jobs[q].sld, jobs[q].dld);
      bl.run(s, W, &dl);
      CK(cudaMemcpyAsync(out.values + d0 * W, flat.p, size_t(d1 - d0) * W * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));  // `flat` is reused by the next batch
      i = e;
    }
    launches += dl;
    CK(cudaStreamSynchronize(s));
  }
};

HostResult::~HostResult() {
  if (values && pool) pool->give(values, values_bytes);
}

double* PinnedPool::take(size_t bytes, size_t* got) {
  {
    std::lock_guard<std::mutex> g(mu_);
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= 2 * bytes) {
      double* p = it->second;
      *got = it->first;
      free_.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  CK(cudaMallocHost(&p, bytes));
  *got = bytes;
  return static_cast<double*>(p);
}

void PinnedPool::give(double* p, size_t bytes) {
  std::lock_guard<std::mutex> g(mu_);
  free_.emplace(bytes, p);
  while (free_.size() > 4) {  // keep the pool bounded
    auto it = free_.begin();
    cudaFreeHost(it->second);
    free_.erase(it);
  }
}

PinnedPool::~PinnedPool() {
  for (auto& [b, p] : free_) cudaFreeHost(p);
}

// ---------------------------------------------------------------------------
uint64_t structure_hash(const h2c_tree& t, const h2c_blocks& b) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  mix(&t.n_points, sizeof(int32_t));
  mix(&t.depth, sizeof(int32_t));
  mix(&t.n_clusters, sizeof(int32_t));
  mix(t.parent, sizeof(int32_t) * t.n_clusters);
  mix(t.begin, sizeof(int32_t) * t.n_clusters);
  mix(t.end, sizeof(int32_t) * t.n_clusters);
  mix(t.level, sizeof(int32_t) * t.n_clusters);
  if (t.child0) mix(t.child0, sizeof(int32_t) * t.n_clusters);
  if (t.child1) mix(t.child1, sizeof(int32_t) * t.n_clusters);
  if (t.bbox) mix(t.bbox, sizeof(double) * 6 * t.n_clusters);
  if (t.perm) mix(t.perm, sizeof(int32_t) * t.n_points);
  mix(&b.n_blocks, sizeof(int64_t));
  mix(b.row, sizeof(int32_t) * b.n_blocks);
  mix(b.col, sizeof(int32_t) * b.n_blocks);
  mix(b.kind, b.n_blocks);
  mix(b.level_ptr, sizeof(int64_t) * (b.depth + 2));
  return h;
}

Context::Context(int device) : device_(device) {
  CK(cudaSetDevice(device));
  // the main (critical-path) stream gets the highest priority: its Gram /
  // eigensolver / collect kernels take SM slots ahead of the deferred target
  // sums queued on the low-priority auxiliary stream
  int least = 0, greatest = 0;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t st;
  CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, greatest));
  stream_ = st;
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
}

// Auxiliary stream on a green context with H2B_AUX_SMS SMs (0 / unset or >= the
// device's count: no partition, the default — on cfg2 the partition measured no
// better than stream priorities alone, profiles/r01/ab_defer_partition.txt).
// Returns nullptr when not partitioned.
void* Context::make_aux_stream(int priority) {
  int want = 0;
  if (const char* e = std::getenv("H2B_AUX_SMS")) want = std::atoi(e);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
  if (want <= 0 || want >= sms) return nullptr;
  // driver entry points through the runtime (no link-time libcuda dependency:
  // the library must load on hosts without a driver for the CPU test tier)
  auto sym = [](const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError(std::string("driver entry point ") + name + " unavailable");
    return fn;
  };
  auto cu = [](CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + " failed: CUresult " + std::to_string(int(r)));
  };
  const auto getDev = reinterpret_cast<decltype(&cuDeviceGet)>(sym("cuDeviceGet"));
  const auto getRes = reinterpret_cast<decltype(&cuDeviceGetDevResource)>(sym("cuDeviceGetDevResource"));
  const auto split = reinterpret_cast<decltype(&cuDevSmResourceSplitByCount)>(sym("cuDevSmResourceSplitByCount"));
  const auto genDesc = reinterpret_cast<decltype(&cuDevResourceGenerateDesc)>(sym("cuDevResourceGenerateDesc"));
  const auto gcCreate = reinterpret_cast<decltype(&cuGreenCtxCreate)>(sym("cuGreenCtxCreate"));
  const auto gcStream = reinterpret_cast<decltype(&cuGreenCtxStreamCreate)>(sym("cuGreenCtxStreamCreate"));
  green_destroy_ = sym("cuGreenCtxDestroy");
  CUdevice dev;
  cu(getDev(&dev, device_), "cuDeviceGet");
  CUdevResource all, grp, rem;
  cu(getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  unsigned nb = 1;
  cu(split(&grp, &nb, &all, &rem, 0, static_cast<unsigned>(want)), "cuDevSmResourceSplitByCount");
  CUdevResourceDesc desc;
  cu(genDesc(&desc, &grp, 1), "cuDevResourceGenerateDesc");
  CUgreenCtx g;
  cu(gcCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
  green_ctx_ = g;
  aux_sms_ = static_cast<int>(grp.sm.smCount);
  CUstream st;
  cu(gcStream(&st, g, CU_STREAM_NON_BLOCKING, priority), "cuGreenCtxStreamCreate");
  return st;
}

void* Context::side_stream(int i) {
  if (side_streams_.empty()) {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (int k = 0; k < kSideStreams; ++k) {
      cudaStream_t st = k == 0 ? static_cast<cudaStream_t>(make_aux_stream(least)) : nullptr;
      if (!st) CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, k == 0 ? least : greatest));
      side_streams_.push_back(st);
    }
  }
  return side_streams_[i];
}

Context::~Context() {
  if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
  for (void* st : side_streams_) cudaStreamDestroy(static_cast<cudaStream_t>(st));
  if (green_ctx_ && green_destroy_)
    reinterpret_cast<decltype(&cuGreenCtxDestroy)>(green_destroy_)(static_cast<CUgreenCtx>(green_ctx_));
  dplan_.reset();
  if (stream_) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
    cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
  }
}

const Plan& Context::plan_for(const h2c_tree& t, const h2c_blocks& b, double* build_seconds) {
  const uint64_t key = structure_hash(t, b);
  // a hash hit is confirmed against the cached descriptor contents (the permutation is what
  // mvp / to_dense gather with; the plan itself depends on parent/begin/end/level and the blocks)
  auto same_desc = [&] {
    return t.n_points == plan_->n_points && t.n_clusters == static_cast<int>(plan_->n_clusters) &&
           perm_.size() == size_t(t.n_points) && std::memcmp(perm_.data(), t.perm, sizeof(int32_t) * t.n_points) == 0 &&
           key_rows_ == std::vector<int32_t>(b.row, b.row + b.n_blocks) &&
           key_cols_ == std::vector<int32_t>(b.col, b.col + b.n_blocks);
  };
  if (plan_ && key == plan_key_ && same_desc()) {
    if (build_seconds) *build_seconds = 0.0;
    return *plan_;
  }
  CK(cudaSetDevice(device_));
  dplan_.reset();
  plan_ = std::make_unique<Plan>(build_plan(t, b, std::max(1u, std::thread::hardware_concurrency())));
  perm_.assign(t.perm, t.perm + t.n_points);
  key_rows_.assign(b.row, b.row + b.n_blocks);
  key_cols_.assign(b.col, b.col + b.n_blocks);
  dplan_ = upload_plan(*plan_, static_cast<cudaStream_t>(stream_));
  plan_key_ = key;
  if (build_seconds) *build_seconds = plan_->build_seconds;
  return *plan_;
}

// binds the context's arena to this thread for the duration of a call
struct ArenaScope {
  Arena* prev_a;
  cudaStream_t prev_s;
  ArenaScope(Arena* a, cudaStream_t s) : prev_a(t_arena), prev_s(t_arena_stream) {
    t_arena = a;
    t_arena_stream = s;
  }
  ~ArenaScope() {
    t_arena = prev_a;
    t_arena_stream = prev_s;
  }
};

std::shared_ptr<DevOperand> Context::upload(const h2c_matrix& m) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  double bs = 0;
  const Plan& P = plan_for(*m.tree, *m.blocks, &bs);
  // resident operands live in the context's arena too (it holds nearly all free HBM once created)
  ArenaScope scope(arena(), static_cast<cudaStream_t>(stream_));
  auto X = upload_operand(P, m, static_cast<cudaStream_t>(stream_), &launches_);
  X->key = plan_key_;
  return X;
}

static void fill_report(const Plan& P, const DevOperand& A, const DevOperand& B, EngineRun& R, bool adaptive,
                        double eps, HostResult& out) {
  RankSet rs;
  rs.ar = A.rr;
  rs.ac = A.rc;
  rs.br = B.rr;
  rs.bc = B.rc;
  rs.cr = R.rcr;
  rs.cc = R.rcc;
  for (int l = 0; l <= P.depth; ++l) {
    const size_t n = P.lv[l].n;
    if (rs.cr[l].size() != n) rs.cr[l].assign(n, 0);
    if (rs.cc[l].size() != n) rs.cc[l].assign(n, 0);
  }
  CountOut co;
  count_report(P, rs, adaptive, co);
  out.eps_trunc = adaptive ? eps : 0.0;
  out.adaptive = adaptive ? 1 : 0;
  out.flops = co.flops;
  out.case_flops = co.case_flops;
  out.flops_exec = R.exec_macs;
  out.max_row.clear();
  out.max_col.clear();
  out.case_products.clear();
  out.t1.clear();
  out.t2.clear();
  out.t3.clear();
  for (const LevelCount& c : co.levels) {
    out.max_row.push_back(c.max_row_rank);
    out.max_col.push_back(c.max_col_rank);
    for (int k = 0; k < 4; ++k) out.case_products.push_back(c.case_products[k]);
    out.t1.push_back(c.max_case1_terms);
    out.t2.push_back(c.max_case2_terms);
    out.t3.push_back(c.max_case3_terms);
  }
}


Arena* Context::arena() {
  DeviceShared& D = device_shared(device_);
  std::lock_guard<std::mutex> g(D.init_mu);
  if (!D.tried) {
    D.tried = true;
    // return what the stream-ordered pool keeps cached (release threshold is
    // unlimited) so the arena can claim it
    CK(cudaDeviceSynchronize());
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device_));
    CK(cudaMemPoolTrimTo(pool, 0));
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    // outside the arena: cuSOLVER workspaces (A/B runs), index vectors, small buffers
    const size_t reserve = size_t(4) << 30;
    if (fr > reserve + (size_t(4) << 30)) {
      auto* a = new Arena;
      size_t want = fr - reserve;
      // H2B_ARENA_GB caps the arena (ncu's kernel replay saves and restores device memory and
      // needs room for its copy; the product then runs with the eviction path if it must)
      if (const char* e = std::getenv("H2B_ARENA_GB")) want = std::min(want, size_t(std::atof(e) * double(size_t(1) << 30)));
      if (a->init(want)) D.arena = a;
      else delete a;
    }
  }
  return D.arena;
}

std::recursive_mutex& Context::call_mutex() { return device_shared(device_).call_mu; }

double Context::run_resident(const std::shared_ptr<DevOperand>& a, const std::shared_ptr<DevOperand>& b,
                             double eps, int adaptive, HostResult* out) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  ArenaScope scope(arena(), static_cast<cudaStream_t>(stream_));
  if (!plan_ || a->key != plan_key_ || b->key != plan_key_)
    throw ConfigErr("mmp: operands were uploaded for another structure");
  if (a->scalar != b->scalar) throw ConfigErr("mmp: operands must share the scalar type");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  CK(cudaSetDevice(device_));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaEventRecord(e0, s));
  EngineRun R(*this, *plan_, *dplan_, *a, *b, eps, adaptive != 0, s);
  R.profiling = profile;
  R.run();
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  launches_ = R.launches;
  R.collect_profile(last_profile);
  if (out) {
    h2c_blocks dummy{};
    (void)dummy;
    fill_report(*plan_, *a, *b, R, adaptive != 0, eps, *out);
    out->device_seconds = ms * 1e-3;
    out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return ms * 1e-3;
}

void Context::mvp(const std::shared_ptr<DevOperand>& a, const double* x_host, int nv, double* y_host) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  if (!plan_ || a->key != plan_key_) throw ConfigErr("mvp: operand was uploaded for another structure");
  if (nv < 1) throw ConfigErr("mvp: need at least one vector");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  CK(cudaSetDevice(device_));
  ArenaScope scope(arena(), s);
  const int W = a->scalar == H2C_COMPLEX ? 2 : 1;
  const size_t bytes = size_t(plan_->n_points) * nv * W * sizeof(double);
  DBuf X(bytes / 8, s), Y(bytes / 8, s);
  CK(cudaMemcpyAsync(X.p, x_host, bytes, cudaMemcpyHostToDevice, s));
  DVec<int32_t> perm;
  perm.upload(perm_, s);
  EngineRun R(*this, *plan_, *dplan_, *a, *a, 0.5, true, s);
  R.mvp(X.p, nv, Y.p, perm.p);
  CK(cudaMemcpyAsync(y_host, Y.p, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  launches_ = R.launches;
}

void Context::to_dense(const std::shared_ptr<DevOperand>& a, double* out) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  if (!plan_ || a->key != plan_key_) throw ConfigErr("to_dense: operand was uploaded for another structure");
  const int N = plan_->n_points;
  if (N > 32768) throw ConfigErr("to_dense: N > 32768 (use the MVP)");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  CK(cudaSetDevice(device_));
  ArenaScope scope(arena(), s);
  const int W = a->scalar == H2C_COMPLEX ? 2 : 1;
  const int panel = std::min(N, 2048);
  DBuf X(size_t(N) * panel * W, s), Y(size_t(N) * panel * W, s);
  DVec<int32_t> perm;
  perm.upload(perm_, s);
  EngineRun R(*this, *plan_, *dplan_, *a, *a, 0.5, true, s);
  for (int c0 = 0; c0 < N; c0 += panel) {
    const int cw = std::min(panel, N - c0);
    CK(cudaMemsetAsync(X.p, 0, size_t(N) * cw * W * sizeof(double), s));
    unit_columns_kernel<<<(cw + 255) / 256, 256, 0, s>>>(X.p, N, c0, cw, W);
    CK(cudaGetLastError());
    R.launches++;
    R.mvp(X.p, cw, Y.p, perm.p);
    CK(cudaMemcpyAsync(out + size_t(c0) * N * W, Y.p, size_t(N) * cw * W * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  launches_ = R.launches;
}

void Context::truncate_gram(int scalar, const double* gram, int n, double eps, double* basis, int* rank,
                            int* degenerate) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  if (n < 1) throw ConfigErr("svd_truncate_gram: gram matrix must be square and non-empty");
  if (!(eps > 0.0 && eps < 1.0)) throw ConfigErr("svd_truncate_gram: eps must be in (0,1)");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  CK(cudaSetDevice(device_));
  // a one-cluster dummy run context: only the truncation path is used
  static Plan empty_plan;
  static DevPlan empty_dplan;
  DevOperand dummy;
  dummy.scalar = scalar;
  EngineRun R(*this, empty_plan, empty_dplan, dummy, dummy, eps, true, s);
  R.truncate_one(gram, n, basis, rank, degenerate);
  launches_ = R.launches;
}

void Context::mmp(const h2c_matrix& a, const h2c_matrix& b, double eps, int adaptive, HostResult& out) {
  std::lock_guard<std::recursive_mutex> call_lock(call_mutex());
  const auto t0 = std::chrono::steady_clock::now();
  ArenaScope scope(arena(), static_cast<cudaStream_t>(stream_));
  if (a.tree != b.tree || a.blocks != b.blocks)  // mmp.cpp:58-63
    throw ConfigErr("mmp: operands must share cluster trees and block structure");
  if (a.scalar != b.scalar) throw ConfigErr("mmp: operands must share the scalar type");
  if (adaptive && !(eps > 0.0 && eps < 1.0)) throw ConfigErr("mmp: eps_trunc must be in (0,1)");
  CK(cudaSetDevice(device_));
  double plan_s = 0;
  const Plan& P = plan_for(*a.tree, *a.blocks, &plan_s);
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  int64_t up_launches = 0;
  const bool trace = std::getenv("H2B_E2E_TRACE") != nullptr;  // host-side phase times on stderr
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a0, auto a1) { return std::chrono::duration<double>(a1 - a0).count(); };
  const auto tu0 = now();
  auto A = upload_operand(P, a, s, &up_launches);
  // B shares A's upload only when it is the very same operand (same descriptor or identical
  // descriptor contents); two operands that merely share a value buffer are uploaded apart
  const bool same_operand =
      &a == &b || (a.values == b.values && a.n_values == b.n_values && a.scalar == b.scalar &&
                   a.row_rank == b.row_rank && a.col_rank == b.col_rank && a.row_offset == b.row_offset &&
                   a.col_offset == b.col_offset && a.block_offset == b.block_offset &&
                   a.row_degenerate == b.row_degenerate && a.col_degenerate == b.col_degenerate);
  std::shared_ptr<DevOperand> B = same_operand ? A : upload_operand(P, b, s, &up_launches);
  const auto tu1 = now();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  EngineRun R(*this, P, *dplan_, *A, *B, eps, adaptive != 0, s);
  R.profiling = profile;
  R.restore_operands = false;
  R.run();
  CK(cudaEventRecord(e1, s));
  if (trace) CK(cudaStreamSynchronize(s));
  const auto tr1 = now();
  std::vector<double*> pool;
  R.download(*a.blocks, out, pool);
  if (trace)
    std::fprintf(stderr, "[e2e] plan %.3f s  upload %.3f s  run %.3f s  download %.3f s\n", plan_s, secs(tu0, tu1),
                 secs(tu1, tr1), secs(tr1, now()));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  launches_ = R.launches + up_launches;
  R.collect_profile(last_profile);
  out.h2d_bytes = int64_t(a.n_values) * R.W * 8 + (B.get() == A.get() ? 0 : int64_t(b.n_values) * R.W * 8);
  out.d2h_bytes = out.n_values * R.W * 8;
  fill_report(P, *A, *B, R, adaptive != 0, eps, out);
  out.device_seconds = ms * 1e-3;
  out.plan_seconds = plan_s;
  out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace h2b
