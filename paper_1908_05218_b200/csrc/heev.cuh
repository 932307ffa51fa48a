// Batched Hermitian eigensolver of the truncation (svd_truncate_gram,
// reference truncation.cpp:9-47), hand-written for sm_100a.
//
// One thread-block cluster of CS CTAs per Gram (CS = 1 for the leaf-level
// 32/64-dimensional Grams, up to 16 for the ~600-dimensional Grams of the upper
// levels), so every Gram of a level is solved by one launch:
//
//  1. Householder tridiagonalisation Q^H G Q = T (LAPACK zhetd2 lower form:
//     H_k = I - tau_k v_k v_k^H, real off-diagonal beta_k).  The Gram is
//     distributed over the cluster by columns (column j in CTA j mod CS, in
//     shared memory); per step the column owner forms v_k, every CTA computes
//     y = B v for its own columns (column dot products: B is Hermitian), the
//     partial y and v^H y are exchanged through distributed shared memory, and
//     every CTA applies the rank-2 update B -= v w^H + w v^H to its columns.
//     Two cluster barriers per step.  The v_k go to a global scratch.
//  2. Implicit-shift QL on the real tridiagonal (Wilkinson shift, EISPACK
//     tql2 / NR tqli form) with the eigenvector matrix Z distributed by rows:
//     every CTA runs the (deterministic) rotation chain of a sweep on its own
//     copy of (d, e) in thread 0 and all threads apply the chain to their own
//     rows of Z, so the QL phase needs no inter-CTA traffic at all.
//  3. Rank rule of truncation.cpp:30-45: clamp at 0, sort descending, keep
//     lambda_i > eps * lambda_max (strict, >= 1); an exactly zero Gram (or no
//     positive eigenvalue) gives e_1 and the degenerate flag.
//  4. Back-transformation of the kept columns only: V = H_0 ... H_{n-2} Z_kept,
//     columns spread over the cluster's CTAs and their warps.
//
// Output matches eig_finalize_kernel's contract: vec_out[b] holds the kept
// eigenvectors (descending) in its first rank columns (column-major n x n),
// val_out[b] the sorted clamped eigenvalues, rank_out[b], degen_io[b] |= unit.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

namespace h2b {

namespace cg = cooperative_groups;

struct HeevParams {
  const double* G;   // [batch][n*n] scalars (column-major, full Hermitian)
  double* V;         // [batch][n*n] scalars: Householder vector k in column k, rows k+1..n-1
  double* Zs;        // [batch][n*n] doubles: kept columns of Z (row-major by kept column)
  double* slab;      // global slabs when the Gram does not fit the cluster's shared memory
  double* vec_out;   // [batch][n*n] scalars
  double* val_out;   // [batch][n]
  int* rank_out;
  uint8_t* degen_io;
  int* fail;         // set when a QL iteration does not converge
  long long* prof;   // optional: clock64() phase stamps of block 0 (tools/heev_bench.cu)
  int dbg;           // tools/heev_bench.cu only: bit 0 skips the Z updates (times the QL chain alone)
  int n;
  double eps;
};

template <bool CPLX>
struct HNum;
template <>
struct HNum<false> {
  using T = double;
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ T one() { return 1.0; }
  static __device__ __forceinline__ T conj(T a) { return a; }
  static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
  static __device__ __forceinline__ T cmul(T a, T b) { return a * b; }  // conj(a) * b
  static __device__ __forceinline__ T fma_(T a, T b, T c) { return fma(a, b, c); }
  static __device__ __forceinline__ T cfma(T a, T b, T c) { return fma(a, b, c); }  // conj(a) b + c
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
  static __device__ __forceinline__ T scale(T a, double s) { return a * s; }
  static __device__ __forceinline__ double abs2(T a) { return a * a; }
  static __device__ __forceinline__ double re(T a) { return a; }
  static __device__ __forceinline__ double im(T) { return 0.0; }
  static __device__ __forceinline__ T make(double r, double) { return r; }
  static __device__ __forceinline__ bool nonzero(T a) { return a != 0.0; }
  static __device__ __forceinline__ T shfl_xor(T a, int o) { return __shfl_xor_sync(0xffffffffu, a, o); }
};
template <>
struct HNum<true> {
  using T = double2;
  static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ T one() { return make_double2(1.0, 0.0); }
  static __device__ __forceinline__ T conj(T a) { return make_double2(a.x, -a.y); }
  static __device__ __forceinline__ T mul(T a, T b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
  }
  static __device__ __forceinline__ T cmul(T a, T b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
  }
  static __device__ __forceinline__ T fma_(T a, T b, T c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
  }
  static __device__ __forceinline__ T cfma(T a, T b, T c) {
    return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
  }
  static __device__ __forceinline__ T add(T a, T b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ T sub(T a, T b) { return make_double2(a.x - b.x, a.y - b.y); }
  static __device__ __forceinline__ T scale(T a, double s) { return make_double2(a.x * s, a.y * s); }
  static __device__ __forceinline__ double abs2(T a) { return fma(a.x, a.x, a.y * a.y); }
  static __device__ __forceinline__ double re(T a) { return a.x; }
  static __device__ __forceinline__ double im(T a) { return a.y; }
  static __device__ __forceinline__ T make(double r, double i) { return make_double2(r, i); }
  static __device__ __forceinline__ bool nonzero(T a) { return a.x != 0.0 || a.y != 0.0; }
  static __device__ __forceinline__ T shfl_xor(T a, int o) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, o), __shfl_xor_sync(0xffffffffu, a.y, o));
  }
};

// shared-memory layout (in doubles) of heev_kernel for n, cluster size CS
struct HeevLayout {
  int n, CS, W, ncl, nrl, ld;
  long long slab, vown, yown, vloc, yall, dd, ee, misc, total;
  __host__ __device__ HeevLayout(int n_, int cs, bool cplx, bool slab_in_smem) {
    n = n_;
    CS = cs;
    W = cplx ? 2 : 1;
    ncl = (n + CS - 1) / CS;
    nrl = ncl;
    ld = slab_in_smem ? n + 1 : n;  // odd column stride in shared memory: conflict-free column teams
    long long at = 0;
    auto take = [&](long long cnt) {
      const long long r = at;
      at += (cnt + 1) & ~1LL;  // 16-byte aligned regions
      return r;
    };
    slab = slab_in_smem ? take((long long)ncl * ld * W) : -1;
    vown = take((long long)n * W);  // also: QL rotation buffers, back-transform staging
    yown = take((long long)n * W);
    vloc = take((long long)n * W);
    yall = take((long long)n * W);
    dd = take(n);
    ee = take(n);  // also: sort order (ints) after the QL phase
    misc = take(64);
    total = at;
  }
};

template <bool CPLX, bool SMEM>
__global__ void __launch_bounds__(512) heev_kernel(const HeevParams p) {
  using N = HNum<CPLX>;
  using T = typename N::T;
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CS = static_cast<int>(cl.num_blocks());
  const int r = static_cast<int>(cl.block_rank());
  const int b = blockIdx.x / CS;
  const int n = p.n;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const HeevLayout L(n, CS, CPLX, SMEM);
  const int ncl = L.ncl, nrl = L.nrl, ld = L.ld;
  // cluster barrier (a plain block barrier for single-CTA clusters: no L1 flush)
  auto csync = [&] {
    if (CS > 1) cl.sync();
    else __syncthreads();
  };

  T* slab = SMEM ? reinterpret_cast<T*>(sm + L.slab)
                 : reinterpret_cast<T*>(p.slab) + ((size_t)b * CS + r) * (size_t)ncl * ld;
  T* vown = reinterpret_cast<T*>(sm + L.vown);  // owner's Householder vector of the step
  T* yown = reinterpret_cast<T*>(sm + L.yown);  // y of this CTA's columns
  T* vloc = reinterpret_cast<T*>(sm + L.vloc);  // local copy of v
  T* yall = reinterpret_cast<T*>(sm + L.yall);  // gathered y
  double* d = sm + L.dd;
  double* e = sm + L.ee;
  double* misc = sm + L.misc;
  double* pub = misc + 40;  // published: [0,1] tau, [2] beta, [3] d_k, [4] gamma part, [6] nonzero flag

  const T* G = reinterpret_cast<const T*>(p.G) + (size_t)b * n * n;
  T* Vg = reinterpret_cast<T*>(p.V) + (size_t)b * n * n;
  const bool stamp = p.prof && blockIdx.x == 0 && threadIdx.x == 0;
  if (stamp) p.prof[0] = clock64();

  // ---- load own columns, detect an exactly zero Gram ----------------------
  int nzf = 0;
  for (long long x = tid; x < (long long)ncl * n; x += nt) {
    const int jl = static_cast<int>(x / n), i = static_cast<int>(x % n);
    const int j = jl * CS + r;
    T v = N::zero();
    if (j < n) v = G[i + (size_t)j * n];
    slab[(size_t)jl * ld + i] = v;
    nzf |= N::nonzero(v) ? 1 : 0;
  }
  nzf = __syncthreads_or(nzf);
  if (tid == 0) pub[6] = nzf ? 1.0 : 0.0;
  csync();
  if (warp == 0) {
    const int nz = __any_sync(0xffffffffu, lane < CS && (*cl.map_shared_rank(pub + 6, lane)) != 0.0);
    if (lane == 0) misc[38] = nz;
  }
  __syncthreads();
  const bool nonzero = misc[38] != 0.0;

  // ---- 1. tridiagonalisation ------------------------------------------------
  long long tprev = stamp ? clock64() : 0;
  auto lap = [&](int slot) {
    if (stamp) {
      const long long t = clock64();
      p.prof[slot] += t - tprev;
      tprev = t;
    }
  };
  for (int k = 0; k + 1 < n; ++k) {
    const int o = k % CS;
    if (r == o) {
      T* col = slab + (size_t)(k / CS) * ld;
      if (warp == 0) {  // zlarfg on x = B(k+1:n, k)
        double s2 = 0.0;
        for (int i = k + 2 + lane; i < n; i += 32) s2 += N::abs2(col[i]);
        for (int of = 16; of > 0; of >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, of);
        if (lane == 0) {
          const T alpha = col[k + 1];
          const double ar = N::re(alpha), ai = N::im(alpha);
          double tr = 0.0, ti = 0.0, beta = ar, sr = 1.0, si = 0.0;
          if (!(s2 == 0.0 && ai == 0.0)) {
            beta = -copysign(sqrt(fma(ar, ar, fma(ai, ai, s2))), ar);
            tr = (beta - ar) / beta;
            ti = -ai / beta;
            const double xr = ar - beta, xi = ai;  // scal = 1 / (alpha - beta)
            const double den = fma(xr, xr, xi * xi);
            sr = xr / den;
            si = -xi / den;
          }
          pub[0] = tr;
          pub[1] = ti;
          pub[2] = beta;
          pub[3] = N::re(col[k]);
          misc[34] = sr;
          misc[35] = si;
        }
      }
      __syncthreads();
      const T scal = N::make(misc[34], misc[35]);
      const bool h_id = pub[0] == 0.0 && pub[1] == 0.0;
      for (int i = k + 1 + tid; i < n; i += nt) {
        const T vi = (i == k + 1) ? N::one() : (h_id ? N::zero() : N::mul(col[i], scal));
        vown[i] = vi;
        Vg[i + (size_t)k * n] = vi;
      }
      if (tid == 0) Vg[k + (size_t)k * n] = N::make(pub[0], pub[1]);  // tau_k on the diagonal slot
    }
    lap(8);
    csync();  // (1) v, tau published by the owner
    const double* po = cl.map_shared_rank(pub, o);
    const T tau = N::make(po[0], po[1]);
    const T* vo = r == o ? vown : cl.map_shared_rank(vown, o);
    for (int i = k + 1 + tid; i < n; i += nt) vloc[i] = vo[i];
    if (tid == 0) {
      e[k] = po[2];
      d[k] = po[3];
    }
    __syncthreads();
    lap(9);
    // y_j = sum_{i>k} conj(B_ij) v_i for own columns j > k: a team of ts lanes per column
    const int jl0 = (k + 1 - r + CS - 1) / CS;  // first local column with j > k
    {
      const int act = ncl - jl0;
      int ts = SMEM ? 1 : 32;  // global slabs: a full warp per column (coalesced rows)
      while (ts < 32 && act * ts < nt) ts <<= 1;
      const int teams = nt / ts, team = tid / ts, tl = tid % ts;
      for (int base = jl0; base < ncl; base += teams) {
        const int jl = base + team;
        const int j = jl * CS + r;
        const bool ok = jl < ncl && j < n;
        T acc = N::zero();
        if (ok) {
          const T* __restrict__ cj = slab + (size_t)jl * ld;
          if (SMEM) {
            for (int i = k + 1 + tl; i < n; i += ts) acc = N::cfma(cj[i], vloc[i], acc);
          } else {  // L2-resident slab: 8 loads in flight per lane
            T a1 = N::zero(), a2 = N::zero(), a3 = N::zero();
            int i = k + 1 + tl;
            for (; i + 7 * ts < n; i += 8 * ts) {
              const T b0 = cj[i], b1 = cj[i + ts], b2 = cj[i + 2 * ts], b3 = cj[i + 3 * ts];
              const T b4 = cj[i + 4 * ts], b5 = cj[i + 5 * ts], b6 = cj[i + 6 * ts], b7 = cj[i + 7 * ts];
              acc = N::cfma(b0, vloc[i], acc);
              a1 = N::cfma(b1, vloc[i + ts], a1);
              a2 = N::cfma(b2, vloc[i + 2 * ts], a2);
              a3 = N::cfma(b3, vloc[i + 3 * ts], a3);
              acc = N::cfma(b4, vloc[i + 4 * ts], acc);
              a1 = N::cfma(b5, vloc[i + 5 * ts], a1);
              a2 = N::cfma(b6, vloc[i + 6 * ts], a2);
              a3 = N::cfma(b7, vloc[i + 7 * ts], a3);
            }
            for (; i + 3 * ts < n; i += 4 * ts) {
              const T b0 = cj[i], b1 = cj[i + ts], b2 = cj[i + 2 * ts], b3 = cj[i + 3 * ts];
              acc = N::cfma(b0, vloc[i], acc);
              a1 = N::cfma(b1, vloc[i + ts], a1);
              a2 = N::cfma(b2, vloc[i + 2 * ts], a2);
              a3 = N::cfma(b3, vloc[i + 3 * ts], a3);
            }
            for (; i < n; i += ts) acc = N::cfma(cj[i], vloc[i], acc);
            acc = N::add(N::add(acc, a1), N::add(a2, a3));
          }
        }
        for (int of = ts >> 1; of > 0; of >>= 1) acc = N::add(acc, N::shfl_xor(acc, of));
        if (ok && tl == 0) yown[j] = acc;
      }
    }
    __syncthreads();
    lap(10);
    if (warp == 0) {  // gamma part = sum_{own j > k} conj(v_j) y_j, fixed order
      double gp = 0.0;
      for (int jl = jl0 + lane; jl < ncl; jl += 32) {
        const int j = jl * CS + r;
        if (j < n) gp += N::re(N::cmul(vloc[j], yown[j]));
      }
      for (int of = 16; of > 0; of >>= 1) gp += __shfl_xor_sync(0xffffffffu, gp, of);
      if (lane == 0) pub[4] = gp;
    }
    csync();  // (2) y parts and gamma parts published
    for (int i = k + 1 + tid; i < n; i += nt) {
      const int q = i % CS;
      yall[i] = q == r ? yown[i] : *cl.map_shared_rank(yown + i, q);
    }
    if (warp == 0) {  // the CS gamma parts loaded in parallel, summed in rank order (same in every CTA)
      const double part = lane < CS ? *cl.map_shared_rank(pub + 4, lane) : 0.0;
      double g = 0.0;
      for (int q = 0; q < CS; ++q) g += __shfl_sync(0xffffffffu, part, q);
      if (lane == 0) misc[36] = g;
    }
    __syncthreads();
    lap(11);
    // rank-2 update of own columns j > k, rows i > k with w = tau y - (|tau|^2 gamma / 2) v:
    // B_ij -= v_i conj(w_j) + w_i conj(v_j)
    {
      const double c = 0.5 * N::abs2(tau) * misc[36];
      const int m = n - k - 1;
      const int ncol = ncl - jl0;
      // w = tau y - c v for every row i > k, once (in place of the gathered y)
      for (int i = k + 1 + tid; i < n; i += nt) yall[i] = N::sub(N::mul(tau, yall[i]), N::scale(vloc[i], c));
      __syncthreads();
      const T* w = yall;
      if (SMEM || CPLX || n <= 256) {
        // a thread owns a row i (v_i, w_i in registers) and a strided subset of the own columns;
        // v_j, w_j are warp-uniform broadcasts
        const int rp = m < nt ? m : nt;  // rows per pass
        const int groups = nt / rp;
        const int g = tid / rp;
        if (g < groups)
          for (int i = k + 1 + tid % rp; i < n; i += rp) {
            const T vi = vloc[i], wi = w[i];
            for (int jl = jl0 + g; jl < ncl; jl += groups) {
              const int j = jl * CS + r;
              if (j >= n) break;
              T* a = slab + (size_t)jl * ld + i;
              *a = N::sub(N::sub(*a, N::mul(vi, N::conj(w[j]))), N::mul(wi, N::conj(vloc[j])));
            }
          }
      } else {  // large real Grams in an L2-resident slab: 8 loads in flight before the stores
        const int tot = ncol * m;  // <= n^2: fits an int
        constexpr int U = 8;
        for (int x0 = tid; x0 < tot; x0 += U * nt) {
          int ii[U], jj[U];
          T av[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int x = x0 + u * nt;
            jj[u] = -1;
            if (x < tot) {
              const int q = x / m;
              const int jl = jl0 + q;
              ii[u] = k + 1 + (x - q * m);
              if (jl * CS + r < n) jj[u] = jl;
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (jj[u] >= 0) av[u] = slab[(size_t)jj[u] * ld + ii[u]];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (jj[u] >= 0) {
              const int i = ii[u], j = jj[u] * CS + r;
              slab[(size_t)jj[u] * ld + i] =
                  N::sub(N::sub(av[u], N::mul(vloc[i], N::conj(w[j]))), N::mul(w[i], N::conj(vloc[j])));
            }
        }
      }
    }
    __syncthreads();
    lap(12);
  }
  {  // last diagonal entry (owner of column n-1)
    const int o = (n - 1) % CS;
    if (r == o && tid == 0) pub[3] = N::re(slab[(size_t)((n - 1) / CS) * ld + (n - 1)]);
    csync();
    if (tid == 0) {
      d[n - 1] = *cl.map_shared_rank(pub + 3, o);
      e[n - 1] = 0.0;
    }
    csync();  // every CTA has read pub before anyone reuses it
  }
  if (stamp) p.prof[1] = clock64();

  // ---- 2. QL on (d, e), Z distributed by rows (row i in CTA i mod CS) ------
  // Thread 0 produces the rotation chain of sweep s+1 while warps 1.. apply the chain of
  // sweep s to their rows of Z (double-buffered, one barrier per sweep).
  double* Z = SMEM ? sm + L.slab : reinterpret_cast<double*>(slab);  // Z[c * nrl + il]
  double* rcb[2] = {reinterpret_cast<double*>(vown), reinterpret_cast<double*>(yown)};
  double* rsb[2] = {reinterpret_cast<double*>(vloc), reinterpret_cast<double*>(yall)};
  int* meta = reinterpret_cast<int*>(misc + 48);  // [2 * buf + 0] mm, [+1] cnt; [4] done; [5] fail
  for (long long x = tid; x < (long long)n * nrl; x += nt) {
    const int c = static_cast<int>(x / nrl), il = static_cast<int>(x % nrl);
    Z[x] = (il * CS + r == c) ? 1.0 : 0.0;
  }
  int l = 0, iter = 0, sweeps = 0, rots = 0;
  double tol = 0.0;
  // one QL sweep (Wilkinson shift) on the unreduced block [l, mm] into buffer q; returns false
  // when every eigenvalue has converged.  Deflation is absolute, |e_m| <= eps_mach ||T||
  // (the Householder reduction already perturbs every eigenvalue by O(eps_mach ||G||); the
  // rank rule compares against eps * lambda_max), so the null-space half of a Gram's spectrum
  // costs no extra sweeps.
  // Called by all of warp 0 (uniform control flow): the scan for the next negligible
  // off-diagonal runs 32 positions per step (ballot); the chain itself runs on lane 0.
  auto produce = [&](int q) -> void {
    double* rc = rcb[q];
    double* rs = rsb[q];
    int cnt = 0, mm = l;
    if (lane == 0) meta[2 * q + 1] = 0;  // no chain unless one is produced below
    for (;;) {
      if (l >= n) {
        if (lane == 0) meta[4] = 1;
        return;
      }
      mm = n - 1;
      for (int b0 = l; b0 < n - 1; b0 += 32) {
        const int i = b0 + lane;
        const unsigned hit = __ballot_sync(0xffffffffu, i < n - 1 && fabs(e[i]) <= tol);
        if (hit) {
          mm = b0 + __ffs(hit) - 1;
          break;
        }
      }
      if (mm == l) {
        ++l;
        iter = 0;
        continue;
      }
      if (++iter > 60) {
        if (lane == 0) {
          meta[5] = 1;
          meta[4] = 1;
        }
        return;
      }
      break;
    }
    if (lane != 0) return;
    double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
    double rr = hypot(g, 1.0);
    g = d[mm] - d[l] + e[l] / (g + copysign(rr, g));
    double s = 1.0, c = 1.0, pp = 0.0;
    bool early = false;
    double ei = e[mm - 1], di = d[mm - 1], di1 = d[mm];
    for (int i = mm - 1; i >= l; --i) {
      const double ein = i > l ? e[i - 1] : 0.0, din = i > l ? d[i - 1] : 0.0;  // prefetch
      const double f = s * ei, bb = c * ei;
      const double t2 = fma(f, f, g * g);
      if (t2 == 0.0) {
        e[i + 1] = 0.0;
        d[i + 1] = di1 - pp;
        e[mm] = 0.0;
        early = true;
        break;
      }
#ifdef HEEV_DIV_ROTATION
      const double rt = sqrt(t2);
      const double inv = 1.0 / rt;
      e[i + 1] = rt;
#else
      const double inv = rsqrt(t2);
      e[i + 1] = t2 * inv;
#endif
      s = f * inv;
      c = g * inv;
      g = di1 - pp;
      rr = fma(di - g, s, 2.0 * c * bb);
      pp = s * rr;
      d[i + 1] = g + pp;
      g = fma(c, rr, -bb);
      rc[cnt] = c;
      rs[cnt] = s;
      ++cnt;
      ei = ein;
      di1 = di;
      di = din;
    }
    if (!early) {
      d[l] -= pp;
      e[l] = g;
      e[mm] = 0.0;
    }
    meta[2 * q] = mm;
    meta[2 * q + 1] = cnt;
    ++sweeps;
    rots += cnt;
  };
  if (warp == 0) {
    double an = 0.0;
    for (int i = lane; i < n; i += 32) an = fmax(an, fabs(d[i]) + fabs(e[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0));
    for (int of = 16; of > 0; of >>= 1) an = fmax(an, __shfl_xor_sync(0xffffffffu, an, of));
    tol = 2.2204460492503131e-16 * an;
    if (lane == 0) {
      meta[4] = 0;
      meta[5] = 0;
      meta[0] = 0;
      meta[1] = 0;
    }
    __syncwarp();
    produce(0);
  }
  __syncthreads();
  for (int sw = 0;; ++sw) {
    const int q = sw & 1;
    const int mm = meta[2 * q], cnt = meta[2 * q + 1];
    const bool done = meta[4] != 0;
    __syncthreads();  // everyone has read this sweep's meta before the producer overwrites buffer q^1
    if (done && cnt == 0) break;
    if (warp == 0) {
      if (!meta[4]) produce(q ^ 1);
      else if (lane == 0) meta[2 * (q ^ 1) + 1] = 0;
      __syncwarp();
    } else if (!(p.dbg & 1)) {
      const double* rc = rcb[q];
      const double* rs = rsb[q];
      for (int il = tid - 32; il < nrl; il += nt - 32) {
        double* __restrict__ zc0 = Z + il;
        double carry = zc0[(size_t)mm * nrl];
        if (SMEM) {
          for (int t = 0; t < cnt; ++t) {
            const int i = mm - 1 - t;
            const double zi = zc0[(size_t)i * nrl];
            const double c = rc[t], s = rs[t];
            zc0[(size_t)(i + 1) * nrl] = fma(s, zi, c * carry);
            carry = fma(c, zi, -s * carry);
          }
        } else {
          // global slab: the next z values are loaded ahead of the stores (no store-to-load
          // serialisation through L2)
          double nxt[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) nxt[u] = (u < cnt) ? zc0[(size_t)(mm - 1 - u) * nrl] : 0.0;
          for (int t = 0; t < cnt; t += 4) {
            double cur[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
#pragma unroll
            for (int u = 0; u < 4; ++u) nxt[u] = (t + 4 + u < cnt) ? zc0[(size_t)(mm - 5 - t - u) * nrl] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (t + u < cnt) {
                const int i = mm - 1 - t - u;
                const double c = rc[t + u], s = rs[t + u];
                zc0[(size_t)(i + 1) * nrl] = fma(s, cur[u], c * carry);
                carry = fma(c, cur[u], -s * carry);
              }
          }
        }
        if (cnt > 0) zc0[(size_t)(mm - cnt) * nrl] = carry;
      }
    }
    __syncthreads();
    if (done) break;
  }
  if (stamp) {
    p.prof[5] = sweeps;
    p.prof[6] = rots;
  }
  if (tid == 0 && meta[5] && r == 0) atomicExch(p.fail, 1);
  if (stamp) p.prof[2] = clock64();

  // ---- 3. rank rule (truncation.cpp:30-45) ----------------------------------
  int* idx = reinterpret_cast<int*>(e);  // e is dead after the QL phase
  __syncthreads();
  double top = 0.0;
  for (int i = 0; i < n; ++i) top = fmax(top, fmax(d[i], 0.0));  // every thread, same order
  const bool unit = !nonzero || !(top > 0.0);
  for (int i = tid; i < n; i += nt) {
    const double li = fmax(d[i], 0.0);
    int pos = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = fmax(d[j], 0.0);
      pos += (lj > li || (lj == li && j > i)) ? 1 : 0;
    }
    idx[pos] = i;
  }
  __syncthreads();
  int rank = 1;
  if (!unit) {
    rank = 0;
    while (rank < n && fmax(d[idx[rank]], 0.0) > p.eps * top) ++rank;
    rank = rank < 1 ? 1 : rank;
  }
  if (r == 0) {
    for (int i = tid; i < n; i += nt) p.val_out[(size_t)b * n + i] = fmax(d[idx[i]], 0.0);
    if (tid == 0) {
      p.rank_out[b] = rank;
      p.degen_io[b] = (unit ? 1 : 0) | p.degen_io[b];
    }
  }
  T* out = reinterpret_cast<T*>(p.vec_out) + (size_t)b * n * n;
  if (unit) {
    if (r == 0)
      for (int i = tid; i < n; i += nt) out[i] = i == 0 ? N::one() : N::zero();
    csync();
    return;
  }
  if (stamp) p.prof[3] = clock64();

  // ---- 4. back-transformation of the kept columns -----------------------------
  double* Zs = p.Zs + (size_t)b * n * n;
  for (long long x = tid; x < (long long)rank * nrl; x += nt) {
    const int c = static_cast<int>(x / nrl), il = static_cast<int>(x % nrl);
    const int i = il * CS + r;
    if (i < n) Zs[(size_t)c * n + i] = Z[(size_t)idx[c] * nrl + il];
  }
  __threadfence();
  csync();
  T* zc = SMEM ? reinterpret_cast<T*>(sm + L.slab) : slab;  // own kept columns c = r, r + CS, ...
  const int nown = (rank - r + CS - 1) / CS;
  for (long long x = tid; x < (long long)nown * n; x += nt) {
    const int q = static_cast<int>(x / n), i = static_cast<int>(x % n);
    zc[x] = N::make(Zs[(size_t)(q * CS + r) * n + i], 0.0);
  }
  // reflectors k = n-2 .. 0, staged 4 at a time in shared memory (the phase-1 vector buffers);
  // each warp applies them to up to 4 of the CTA's columns at a time
  T* stg[4] = {vown, yown, vloc, yall};
  for (int k0 = n - 2; k0 >= 0; k0 -= 4) {
    const int nk = min(4, k0 + 1);
    __syncthreads();
    for (int q = 0; q < nk; ++q) {
      const int k = k0 - q;
      const T* vk = Vg + (size_t)k * n;
      for (int i = k + tid; i < n; i += nt) stg[q][i] = vk[i];  // [k] = tau_k, [k+1..] = v_k
    }
    __syncthreads();
    for (int q0 = warp * 4; q0 < nown; q0 += nw * 4) {
      const int nq = min(4, nown - q0);
      for (int q = 0; q < nk; ++q) {
        const int k = k0 - q;
        const T* vk = stg[q];
        T dot[4] = {N::zero(), N::zero(), N::zero(), N::zero()};
        for (int i = k + 1 + lane; i < n; i += 32) {
          const T vi = vk[i];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < nq) dot[c] = N::cfma(vi, zc[(size_t)(q0 + c) * n + i], dot[c]);
        }
        const T tauk = vk[k];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          for (int of = 16; of > 0; of >>= 1) dot[c] = N::add(dot[c], N::shfl_xor(dot[c], of));
          dot[c] = N::mul(tauk, dot[c]);
        }
        for (int i = k + 1 + lane; i < n; i += 32) {
          const T vi = vk[i];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < nq) {
              T* z = zc + (size_t)(q0 + c) * n + i;
              *z = N::sub(*z, N::mul(vi, dot[c]));
            }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (long long x = tid; x < (long long)nown * n; x += nt) {
    const int q = static_cast<int>(x / n), i = static_cast<int>(x % n);
    out[(size_t)(q * CS + r) * n + i] = zc[x];
  }
  if (stamp) p.prof[4] = clock64();
  csync();
}

}  // namespace h2b
