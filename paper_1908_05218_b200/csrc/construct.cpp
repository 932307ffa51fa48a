// Synthetic H^2 inputs for the BASELINE.json configurations (input side; the
// reference only builds H^2 matrices from a dense N x N matrix,
// h2_matrix.cpp:141-181, which is infeasible at these sizes).
//
//  - build_chebyshev: nested tensor Chebyshev interpolation on the clusters'
//    bounding boxes (leaf V = Lagrange polynomials at the points, transfer
//    E = parent polynomials at the child's nodes, coupling S = kernel at node
//    pairs), orthonormalised bottom-up with Householder QR (V = Q R, stacked
//    [R_c1 E_c1; R_c2 E_c2] = Q R, couplings R_t S R_s^T) so the operand meets
//    the MMP precondition of orthonormal nested bases (mmp.hpp:54-56).
//  - build_fd_laplacian: the 7-point stencil in H^2 form (exact full blocks,
//    zero admissible blocks with the degenerate e_1 bases build_h2 produces for
//    a zero far field, truncation.cpp:16-23).
#include <atomic>
#include <memory>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <thread>
#include <type_traits>
#include <algorithm>

#include "construct_dev.hpp"
#include "structure.hpp"

namespace h2b {

namespace {

// f(k) for k in [0, n) on `threads` threads, dynamically scheduled in chunks (fixed_chunk > 0:
// that many per grab - 1 for loops whose iterations differ widely in cost)
template <class F>
void pfor(int64_t n, int threads, F&& f, int64_t fixed_chunk = 0) {
  threads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n)));
  std::atomic<int64_t> next{0};
  const int64_t chunk =
      fixed_chunk > 0 ? fixed_chunk : std::max<int64_t>(1, std::min<int64_t>(64, n / (8 * int64_t(threads))));
  auto work = [&] {
    for (;;) {
      const int64_t i = next.fetch_add(chunk);
      if (i >= n) break;
      for (int64_t k = i; k < std::min(n, i + chunk); ++k) f(k);
    }
  };
  if (threads == 1) {
    work();
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work);
  for (auto& th : pool) th.join();
}

// column-major dense helpers (real)
struct Dm {
  int r = 0, c = 0;
  std::vector<double> d;
  Dm() = default;
  Dm(int rows, int cols) : r(rows), c(cols), d(size_t(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return d[i + size_t(j) * r]; }
  double operator()(int i, int j) const { return d[i + size_t(j) * r]; }
};

Dm matmul(const Dm& a, const Dm& b) {
  Dm c(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k) {
      const double bk = b(k, j);
      if (bk == 0.0) continue;
      const double* ac = &a.d[size_t(k) * a.r];
      double* cc = &c.d[size_t(j) * c.r];
      for (int i = 0; i < a.r; ++i) cc[i] += ac[i] * bk;
    }
  return c;
}

// Householder QR: a (m x n) = Q (m x r) R (r x n), r = min(m, n)
void house_qr(const Dm& a, Dm& Q, Dm& R) {
  const int m = a.r, n = a.c, r = std::min(m, n);
  Dm w = a;
  std::vector<std::vector<double>> vs;
  std::vector<double> betas;
  for (int k = 0; k < r; ++k) {
    double nrm = 0.0;
    for (int i = k; i < m; ++i) nrm += w(i, k) * w(i, k);
    nrm = std::sqrt(nrm);
    std::vector<double> v(m - k, 0.0);
    double beta = 0.0;
    if (nrm > 0.0) {
      const double alpha = w(k, k) >= 0 ? -nrm : nrm;
      for (int i = k; i < m; ++i) v[i - k] = w(i, k);
      v[0] -= alpha;
      double vn = 0.0;
      for (double x : v) vn += x * x;
      if (vn > 0.0) {
        beta = 2.0 / vn;
        for (int j = k; j < n; ++j) {
          double s = 0.0;
          for (int i = k; i < m; ++i) s += v[i - k] * w(i, j);
          s *= beta;
          for (int i = k; i < m; ++i) w(i, j) -= s * v[i - k];
        }
      }
    }
    vs.push_back(std::move(v));
    betas.push_back(beta);
  }
  R = Dm(r, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= std::min(j, r - 1); ++i) R(i, j) = w(i, j);
  Q = Dm(m, r);
  for (int j = 0; j < r; ++j) Q(j, j) = 1.0;
  for (int k = r - 1; k >= 0; --k) {
    const auto& v = vs[k];
    if (betas[k] == 0.0) continue;
    for (int j = 0; j < r; ++j) {
      double s = 0.0;
      for (int i = k; i < m; ++i) s += v[i - k] * Q(i, j);
      s *= betas[k];
      for (int i = k; i < m; ++i) Q(i, j) -= s * v[i - k];
    }
  }
}

struct Box {
  double c[3], h[3];
};

double cheb_node(const Box& b, int d, int i, int m) {
  return b.c[d] + b.h[d] * std::cos((2.0 * i + 1.0) * M_PI / (2.0 * m));
}

// Lagrange basis polynomial i (of m) of the box in dimension d at x
double lagrange(const Box& b, int d, int i, int m, double x) {
  const double xi = cheb_node(b, d, i, m);
  double v = 1.0;
  for (int j = 0; j < m; ++j) {
    if (j == i) continue;
    const double xj = cheb_node(b, d, j, m);
    v *= (x - xj) / (xi - xj);
  }
  return v;
}

}  // namespace

void HostH2::desc(h2c_matrix* d) const {
  d->scalar = scalar;
  d->row_rank = row_rank.data();
  d->col_rank = col_rank.data();
  d->row_degenerate = row_dg.data();
  d->col_degenerate = col_dg.data();
  d->row_offset = row_off.data();
  d->col_offset = col_off.data();
  d->block_offset = block_off.data();
  d->values = values.data();
  d->n_values = static_cast<int64_t>(values.size()) / (scalar == H2C_COMPLEX ? 2 : 1);
}

namespace {

using cd = std::complex<double>;

// host BLAS/LAPACK for the input constructor (the scipy wheel's OpenBLAS, symbols prefixed
// `scipy_`); never used by the product path
extern "C" {
void scipy_cblas_dgemm(int order, int ta, int tb, int m, int n, int k, double alpha, const double* a, int lda,
                       const double* b, int ldb, double beta, double* c, int ldc);
void scipy_cblas_zgemm(int order, int ta, int tb, int m, int n, int k, const void* alpha, const void* a, int lda,
                       const void* b, int ldb, const void* beta, void* c, int ldc);
void scipy_dsyevd_(const char* jobz, const char* uplo, const int* n, double* a, const int* lda, double* w,
                   double* work, const int* lwork, int* iwork, const int* liwork, int* info, size_t, size_t);
void scipy_zheevd_(const char* jobz, const char* uplo, const int* n, void* a, const int* lda, double* w, void* work,
                   const int* lwork, double* rwork, const int* lrwork, int* iwork, const int* liwork, int* info,
                   size_t, size_t);
void scipy_openblas_set_num_threads(int);
}

// column-major dense matrix of scalar S
template <class S>
struct M {
  int r = 0, c = 0;
  std::vector<S> d;
  M() = default;
  M(int rows, int cols) : r(rows), c(cols), d(size_t(rows) * cols, S(0)) {}
  S& operator()(int i, int j) { return d[i + size_t(j) * r]; }
  const S& operator()(int i, int j) const { return d[i + size_t(j) * r]; }
};

enum Op { kN = 111, kT = 112, kC = 113 };

// C = op(A) op(B) (+ C if acc)
template <class S>
void gemm(Op oa, Op ob, const M<S>& a, const M<S>& b, M<S>& c, bool acc = false) {
  const int m = oa == kN ? a.r : a.c, k = oa == kN ? a.c : a.r, n = ob == kN ? b.c : b.r;
  if (!acc) c = M<S>(m, n);
  if (m == 0 || n == 0 || k == 0) return;
  if constexpr (std::is_same_v<S, double>) {
    scipy_cblas_dgemm(102, oa == kC ? kT : oa, ob == kC ? kT : ob, m, n, k, 1.0, a.d.data(), a.r, b.d.data(), b.r,
                      acc ? 1.0 : 0.0, c.d.data(), c.r);
  } else {
    const cd one(1.0), beta(acc ? 1.0 : 0.0);
    scipy_cblas_zgemm(102, oa, ob, m, n, k, &one, a.d.data(), a.r, b.d.data(), b.r, &beta, c.d.data(), c.r);
  }
}

template <class S>
M<S> lift(const Dm& a) {
  M<S> o(a.r, a.c);
  for (size_t i = 0; i < a.d.size(); ++i) o.d[i] = S(a.d[i]);
  return o;
}

// svd_truncate_gram (truncation.cpp:9-47) on the host: keep lambda_i > eps * lambda_max (>= 1);
// zero Gram -> e_1, degenerate.  Returns the basis (n x rank), eigenvectors descending.
template <class S>
M<S> truncate_gram(const M<S>& g, double eps, bool& degenerate) {
  const int n = g.r;
  degenerate = false;
  bool zero = true;
  for (const S& x : g.d)
    if (x != S(0)) {
      zero = false;
      break;
    }
  auto unit = [&] {
    M<S> e(n, 1);
    e(0, 0) = S(1);
    degenerate = true;
    return e;
  };
  if (zero) return unit();
  M<S> a = g;
  std::vector<double> w(n);
  int info = 0, lwork = -1, liwork = -1, lrwork = -1, iwq = 0;
  const int lda = n;
  if constexpr (std::is_same_v<S, double>) {
    double wq = 0;
    scipy_dsyevd_("V", "L", &n, a.d.data(), &lda, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
    lwork = static_cast<int>(wq);
    liwork = iwq;
    std::vector<double> work(std::max(1, lwork));
    std::vector<int> iwork(std::max(1, liwork));
    scipy_dsyevd_("V", "L", &n, a.d.data(), &lda, w.data(), work.data(), &lwork, iwork.data(), &liwork, &info, 1,
                  1);
  } else {
    cd wq = 0;
    double rq = 0;
    scipy_zheevd_("V", "L", &n, a.d.data(), &lda, w.data(), &wq, &lwork, &rq, &lrwork, &iwq, &liwork, &info, 1, 1);
    lwork = static_cast<int>(wq.real());
    lrwork = static_cast<int>(rq);
    liwork = iwq;
    std::vector<cd> work(std::max(1, lwork));
    std::vector<double> rwork(std::max(1, lrwork));
    std::vector<int> iwork(std::max(1, liwork));
    scipy_zheevd_("V", "L", &n, a.d.data(), &lda, w.data(), work.data(), &lwork, rwork.data(), &lrwork, iwork.data(),
                  &liwork, &info, 1, 1);
  }
  if (info != 0) throw std::runtime_error("construct: eigensolver failed");
  for (double& x : w) x = std::max(x, 0.0);
  const double top = w[n - 1];
  if (top <= 0.0) return unit();
  int rank = 0;
  while (rank < n && w[n - 1 - rank] > eps * top) ++rank;
  rank = std::max(rank, 1);
  M<S> out(n, rank);
  for (int j = 0; j < rank; ++j)
    for (int i = 0; i < n; ++i) out(i, j) = a(i, n - 1 - j);
  return out;
}

struct Cheb {
  int m = 0;  // order per dimension
  Box box;
  double node(int d, int i) const { return cheb_node(box, d, i, m); }
  double lag(int d, int i, double x) const { return lagrange(box, d, i, m, x); }
  int k() const { return m * m * m; }
};

template <class S>
std::unique_ptr<HostH2> chebyshev_impl(const h2c_tree& t, const h2c_blocks& b, const double* xyz, int kernel,
                                       double kappa, double diagonal, const int* orders, double eps_rc,
                                       int threads) {
  constexpr bool cplx = !std::is_same_v<S, double>;
  constexpr int W = cplx ? 2 : 1;
  const int nc = t.n_clusters, D = t.depth;
  auto out = std::make_unique<HostH2>();
  out->scalar = cplx ? H2C_COMPLEX : H2C_REAL;
  const int* perm = t.perm;
  const bool trace = std::getenv("H2B_CONSTRUCT_TRACE") != nullptr;  // phase wall times on stderr
  auto t_last = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[construct] %-22s %8.3f s\n", what, std::chrono::duration<double>(now - t_last).count());
    t_last = now;
  };

  // interpolation boxes: bounding boxes of the points the matrix is evaluated on (the
  // tree's own points, or e.g. jittered copies over the same tree), degenerate extents widened
  std::vector<Cheb> cb(nc);
  for (int c = 0; c < nc; ++c) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int p = t.begin[c]; p < t.end[c]; ++p)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], xyz[3 * perm[p] + d]);
        hi[d] = std::max(hi[d], xyz[3 * perm[p] + d]);
      }
    double ext = 0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
    for (int d = 0; d < 3; ++d) {
      cb[c].box.c[d] = 0.5 * (lo[d] + hi[d]);
      cb[c].box.h[d] = std::max(0.5 * (hi[d] - lo[d]), 1e-6 * std::max(ext, 1e-300));
    }
    cb[c].m = orders[t.level[c]];
    if (cb[c].m < 1 || cb[c].m > 64) throw std::invalid_argument("chebyshev order must be in [1, 64]");
  }
  std::vector<std::vector<int>> levels(D + 1);
  for (int c = 0; c < nc; ++c) levels[t.level[c]].push_back(c);
  const int lmin = D == 0 ? 0 : 1;

  // 1. nested interpolation bases, orthonormalised bottom-up: V_c = Q_c R_c (leaf),
  //    [R_c1 E_c1; R_c2 E_c2] = Q_c R_c (non-leaf; E = parent Lagrange polynomials at the child's nodes)
  std::vector<Dm> Qb(nc), Rb(nc);
  for (int l = D; l >= lmin; --l) {
    const auto& ids = levels[l];
    pfor(static_cast<int64_t>(ids.size()), threads, [&](int64_t q) {
      const int c = ids[q];
      const Cheb& C = cb[c];
      const int m = C.m, k = C.k();
      if (t.child0[c] < 0) {
        const int n = t.end[c] - t.begin[c];
        Dm V(n, k);
        for (int p = 0; p < n; ++p) {
          const double* x = &xyz[3 * perm[t.begin[c] + p]];
          double lx[64], ly[64], lz[64];
          for (int i = 0; i < m; ++i) {
            lx[i] = C.lag(0, i, x[0]);
            ly[i] = C.lag(1, i, x[1]);
            lz[i] = C.lag(2, i, x[2]);
          }
          for (int iz = 0; iz < m; ++iz)
            for (int iy = 0; iy < m; ++iy)
              for (int ix = 0; ix < m; ++ix) V(p, ix + m * (iy + m * iz)) = lx[ix] * ly[iy] * lz[iz];
        }
        house_qr(V, Qb[c], Rb[c]);
      } else {
        const int c1 = t.child0[c], c2 = t.child1[c];
        const int r1 = Rb[c1].r, r2 = Rb[c2].r;
        Dm Z(r1 + r2, k);
        for (int s = 0; s < 2; ++s) {
          const int ch = s ? c2 : c1;
          const Cheb& H = cb[ch];
          const int mh = H.m;
          Dm E(H.k(), k);  // E[nu', nu] = L^parent_nu(xi^child_nu')
          for (int jz = 0; jz < mh; ++jz)
            for (int jy = 0; jy < mh; ++jy)
              for (int jx = 0; jx < mh; ++jx) {
                const double px = H.node(0, jx), py = H.node(1, jy), pz = H.node(2, jz);
                double lx[64], ly[64], lz[64];
                for (int i = 0; i < m; ++i) {
                  lx[i] = C.lag(0, i, px);
                  ly[i] = C.lag(1, i, py);
                  lz[i] = C.lag(2, i, pz);
                }
                for (int iz = 0; iz < m; ++iz)
                  for (int iy = 0; iy < m; ++iy)
                    for (int ix = 0; ix < m; ++ix)
                      E(jx + mh * (jy + mh * jz), ix + m * (iy + m * iz)) = lx[ix] * ly[iy] * lz[iz];
              }
          const Dm RE = matmul(Rb[ch], E);
          for (int j = 0; j < k; ++j)
            for (int i = 0; i < RE.r; ++i) Z(i + (s ? r1 : 0), j) = RE(i, j);
        }
        house_qr(Z, Qb[c], Rb[c]);
      }
    });
  }
  tick("nested bases");
  // kernel value at distance r
  auto G = [&](double r) -> S {
    const double f = 1.0 / (4.0 * M_PI * r);
    if constexpr (cplx) {
      double sn, cs;
      ::sincos(kappa * r, &sn, &cs);
      return S(f * cs, -f * sn);
    } else {
      return S(f);
    }
  };
  (void)kernel;
  // 2. couplings in the orthonormal coordinates: S_ts = R_t K(xi_t, xi_s) R_s^T (recomputed
  //    when needed instead of stored: at 1M points the un-recompressed set would not fit in RAM)
  std::vector<int64_t> adm;
  for (int64_t q = 0; q < b.n_blocks; ++q)
    if (b.kind[q] == H2C_ADMISSIBLE) adm.push_back(q);
  auto nodes = [&](const Cheb& X) {
    Dm xr(3, X.k());
    for (int iz = 0; iz < X.m; ++iz)
      for (int iy = 0; iy < X.m; ++iy)
        for (int ix = 0; ix < X.m; ++ix) {
          const int i = ix + X.m * (iy + X.m * iz);
          xr(0, i) = X.node(0, ix), xr(1, i) = X.node(1, iy), xr(2, i) = X.node(2, iz);
        }
    return xr;
  };
  auto coupling_raw = [&](int64_t q) {
    const int r = b.row[q], s = b.col[q];
    const Dm xr = nodes(cb[r]), ys = nodes(cb[s]);
    const int kr = xr.c, ks = ys.c;
    const M<double> Rr = lift<double>(Rb[r]), Rs = lift<double>(Rb[s]);
    // K stacked [Re K; Im K] (W k_r x k_s), X = K R_s^T, S = R_r X (per part)
    M<double> K(W * kr, ks), X;
    for (int j = 0; j < ks; ++j)
      for (int i = 0; i < kr; ++i) {
        const double dx = xr(0, i) - ys(0, j), dy = xr(1, i) - ys(1, j), dz = xr(2, i) - ys(2, j);
        const S g = G(std::sqrt(dx * dx + dy * dy + dz * dz));
        if constexpr (cplx) {
          K(i, j) = g.real();
          K(kr + i, j) = g.imag();
        } else {
          K(i, j) = g;
        }
      }
    gemm(kN, kT, K, Rs, X);
    M<S> out_s(Rr.r, Rs.r);
    for (int part = 0; part < W; ++part) {
      M<double> Xp(kr, Rs.r), Sp;
      for (int j = 0; j < Rs.r; ++j)
        std::copy(&X.d[size_t(j) * X.r + part * kr], &X.d[size_t(j) * X.r + part * kr + kr], &Xp.d[size_t(j) * kr]);
      gemm(kN, kN, Rr, Xp, Sp);
      for (size_t i = 0; i < Sp.d.size(); ++i) {
        if constexpr (cplx)
          out_s.d[i] += part ? S(0.0, Sp.d[i]) : S(Sp.d[i], 0.0);
        else
          out_s.d[i] = Sp.d[i];
      }
    }
    return out_s;
  };
  scipy_openblas_set_num_threads(1);  // parallel over clusters / blocks instead

  // Device path for the two coupling passes (construct_dev.cu): kernel evaluation + batched
  // GEMMs on the GPU when one is present (H2B_CONSTRUCT_HOST=1 keeps everything on the host).
  const bool use_dev = cdev_available() && std::getenv("H2B_CONSTRUCT_HOST") == nullptr;
  std::unique_ptr<CouplingDev, void (*)(CouplingDev*)> dev(use_dev ? cdev_create(cplx, kappa) : nullptr, cdev_destroy);
  std::vector<int> pos_in_level(nc, -1);
  for (int l = 0; l <= D; ++l)
    for (size_t i = 0; i < levels[l].size(); ++i) pos_in_level[levels[l][i]] = static_cast<int>(i);
  std::vector<std::vector<int64_t>> adm_level(D + 1);  // per level, sorted by row position (stable)
  for (int64_t q : adm) adm_level[t.level[b.row[q]]].push_back(q);
  for (auto& v : adm_level)
    std::stable_sort(v.begin(), v.end(), [&](int64_t x, int64_t y) {
      return pos_in_level[b.row[x]] < pos_in_level[b.row[y]];
    });
  auto dev_level = [&](int l) {
    const auto& ids = levels[l];
    std::vector<double> boxes(6 * ids.size());
    std::vector<const double*> R(ids.size());
    std::vector<int> r(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) {
      const Cheb& X = cb[ids[i]];
      for (int d2 = 0; d2 < 3; ++d2) {
        boxes[6 * i + d2] = X.box.c[d2];
        boxes[6 * i + 3 + d2] = X.box.h[d2];
      }
      R[i] = Rb[ids[i]].d.data();
      r[i] = Rb[ids[i]].r;
    }
    cdev_level(dev.get(), static_cast<int>(ids.size()), boxes.data(), ids.empty() ? 1 : cb[ids[0]].m, R.data(),
               r.data());
  };
  auto level_blocks = [&](int l, std::vector<int>& br, std::vector<int>& bc) {
    br.clear();
    bc.clear();
    for (int64_t q : adm_level[l]) {
      br.push_back(pos_in_level[b.row[q]]);
      bc.push_back(pos_in_level[b.col[q]]);
    }
  };

  // 3. optional recompression (the reference's build_h2 rule, h2_matrix.cpp:83-121, applied to the
  //    interpolation operand): the row Gram of cluster t over its far field (own admissible
  //    partners plus those inherited from its ancestors, far_partners h2_matrix.cpp:22-46) is
  //    V_t Z_t V_t^H with Z_t = sum_s S_ts S_ts^H + T_t Z_parent T_t^H (orthonormal V_t), so the
  //    leaf basis is V_t * trunc(Z_t) and a parent's transfer is trunc(X Z_p X^H) with
  //    X = [P_c1 T_c1; P_c2 T_c2], P_c = (new basis)^H (old basis).  The kernel and point sets are
  //    symmetric, so the column basis equals the row basis and S'_ts = P_t S_ts P_s^T.
  std::vector<M<S>> basis(nc), P(nc);  // final basis blocks (leaf n x k', transfer (k1'+k2') x k')
  std::vector<uint8_t> dg(nc, 0);
  const bool rc = eps_rc > 0;
  if (rc) {
    std::vector<std::vector<int64_t>> by_row(nc);
    for (int64_t q : adm) by_row[b.row[q]].push_back(q);
    std::vector<M<S>> Z(nc);
    for (int l = lmin; l <= D; ++l) {
      const auto& ids = levels[l];
      std::vector<M<S>> zown;
      if (dev) {  // sum_s S_ts S_ts^H of the level on the device
        zown.resize(ids.size());
        std::vector<double*> zp(ids.size());
        for (size_t i = 0; i < ids.size(); ++i) {
          zown[i] = M<S>(Qb[ids[i]].c, Qb[ids[i]].c);
          zp[i] = reinterpret_cast<double*>(zown[i].d.data());
        }
        std::vector<int> br, bc;
        level_blocks(l, br, bc);
        if (!br.empty()) {
          try {
            dev_level(l);
            cdev_grams(dev.get(), static_cast<int>(br.size()), br.data(), bc.data(), zp.data());
          } catch (const std::exception& e) {  // e.g. the HBM is held by a product context: host path
            if (trace) std::fprintf(stderr, "[construct] device pass failed (%s); host path\n", e.what());
            dev.reset();
            zown.clear();
          }
        }
      }
      if (zown.empty() && static_cast<int64_t>(ids.size()) < 8 * int64_t(threads)) {
        // Host path on a level with few clusters (the upper levels, whose blocks are the expensive
        // ones): parallel over the level's blocks instead of its clusters, in bounded batches;
        // each cluster's sum still runs in its block order.
        zown.resize(ids.size());
        std::vector<std::pair<int, int64_t>> items;
        for (size_t qi = 0; qi < ids.size(); ++qi) {
          zown[qi] = M<S>(Qb[ids[qi]].c, Qb[ids[qi]].c);
          for (int64_t q : by_row[ids[qi]]) items.emplace_back(static_cast<int>(qi), q);
        }
        const size_t budget = size_t(2) << 30;  // bytes of per-block Grams alive at once
        for (size_t pos = 0; pos < items.size();) {
          size_t end = pos, bytes = 0;
          while (end < items.size() && (end == pos || bytes < budget)) {
            const size_t rk = Qb[ids[items[end].first]].c;
            bytes += rk * rk * sizeof(S);
            ++end;
          }
          std::vector<M<S>> gs(end - pos);
          pfor(static_cast<int64_t>(end - pos), threads, [&](int64_t i) {
            const M<S> Sq = coupling_raw(items[pos + i].second);
            gemm(kN, kC, Sq, Sq, gs[i]);
          }, 1);
          for (size_t i = pos; i < end; ++i) {
            M<S>& z = zown[items[i].first];
            const M<S>& g = gs[i - pos];
            for (size_t x = 0; x < z.d.size(); ++x) z.d[x] += g.d[x];
          }
          pos = end;
        }
      }
      pfor(static_cast<int64_t>(ids.size()), threads, [&](int64_t qi) {
        const int c = ids[qi];
        const int rk = Qb[c].c;
        M<S> z(rk, rk);
        if (!zown.empty()) {
          z = std::move(zown[qi]);
        } else {
          for (int64_t q : by_row[c]) {
            const M<S> Sq = coupling_raw(q);
            gemm(kN, kC, Sq, Sq, z, true);
          }
        }
        const int p = t.parent[c];
        if (p >= 0 && t.level[p] >= lmin && Z[p].r > 0) {
          // T_c = rows of Q_p belonging to child c
          const int off = (t.child0[p] == c) ? 0 : Qb[t.child0[p]].c;
          M<S> T(rk, Qb[p].c);
          for (int j = 0; j < T.c; ++j)
            for (int i = 0; i < rk; ++i) T(i, j) = S(Qb[p](off + i, j));
          M<S> TZ;
          gemm(kN, kN, T, Z[p], TZ);
          gemm(kN, kC, TZ, T, z, true);
        }
        Z[c] = std::move(z);
      });
    }
    tick("far-field Grams");
    for (int l = D; l >= lmin; --l) {
      const auto& ids = levels[l];
      pfor(static_cast<int64_t>(ids.size()), threads, [&](int64_t qi) {
        const int c = ids[qi];
        bool deg = false;
        if (t.child0[c] < 0) {
          const M<S> U = truncate_gram(Z[c], eps_rc, deg);
          gemm(kN, kN, lift<S>(Qb[c]), U, basis[c]);
          M<S> Ph(U.c, U.r);
          for (int i = 0; i < U.r; ++i)
            for (int j = 0; j < U.c; ++j) {
              if constexpr (cplx)
                Ph(j, i) = std::conj(U(i, j));
              else
                Ph(j, i) = U(i, j);
            }
          P[c] = std::move(Ph);
        } else {
          const int c1 = t.child0[c], c2 = t.child1[c];
          const int r1 = Qb[c1].c;
          const int k1 = P[c1].r, k2 = P[c2].r;
          M<S> X(k1 + k2, Qb[c].c);
          for (int sd = 0; sd < 2; ++sd) {
            const int ch = sd ? c2 : c1;
            M<S> T(Qb[ch].c, Qb[c].c);
            for (int j = 0; j < T.c; ++j)
              for (int i = 0; i < T.r; ++i) T(i, j) = S(Qb[c]((sd ? r1 : 0) + i, j));
            M<S> PT;
            gemm(kN, kN, P[ch], T, PT);
            for (int j = 0; j < X.c; ++j)
              for (int i = 0; i < PT.r; ++i) X(i + (sd ? k1 : 0), j) = PT(i, j);
          }
          M<S> XZ, Gm;
          gemm(kN, kN, X, Z[c], XZ);
          gemm(kN, kC, XZ, X, Gm);
          const M<S> U = truncate_gram(Gm, eps_rc, deg);
          basis[c] = U;
          gemm(kC, kN, U, X, P[c]);
        }
        dg[c] = deg ? 1 : 0;
        Z[c] = M<S>();  // released once used
      });
    }
    tick("truncation");
  } else {
    for (int c = 0; c < nc; ++c)
      if (!(t.parent[c] < 0 && D > 0)) basis[c] = lift<S>(Qb[c]);
  }

  // layout: bases (row == col, shared offsets), then blocks in global order
  int64_t total = 0;
  out->row_rank.assign(nc, 0);
  out->row_dg.assign(nc, 0);
  out->row_off.assign(nc, -1);
  for (int c = 0; c < nc; ++c) {
    if (t.parent[c] < 0 && D > 0) continue;
    out->row_rank[c] = basis[c].c;
    out->row_dg[c] = dg[c];
    out->row_off[c] = total;
    total += int64_t(basis[c].r) * basis[c].c;
  }
  out->block_off.assign(b.n_blocks, -1);
  for (int64_t q = 0; q < b.n_blocks; ++q) {
    const int r = b.row[q], s = b.col[q];
    if (b.kind[q] == H2C_ADMISSIBLE) {
      out->block_off[q] = total;
      total += int64_t(out->row_rank[r]) * out->row_rank[s];
    } else if (b.kind[q] == H2C_INADMISSIBLE_LEAF) {
      out->block_off[q] = total;
      total += int64_t(t.end[r] - t.begin[r]) * (t.end[s] - t.begin[s]);
    }
  }
  out->values.assign(size_t(total) * W, 0.0);
  S* V = reinterpret_cast<S*>(out->values.data());
  for (int c = 0; c < nc; ++c) {
    if (out->row_off[c] < 0) continue;
    std::copy(basis[c].d.begin(), basis[c].d.end(), V + out->row_off[c]);
  }
  bool dev_done = false;
  if (dev) {
    try {
    for (int l = lmin; l <= D; ++l) {
      std::vector<int> br, bc;
      level_blocks(l, br, bc);
      if (br.empty()) continue;
      dev_level(l);
      const auto& ids = levels[l];
      std::vector<const double*> pp(ids.size());
      std::vector<int> kp(ids.size());
      for (size_t i = 0; i < ids.size(); ++i) {
        pp[i] = rc ? reinterpret_cast<const double*>(P[ids[i]].d.data()) : nullptr;
        kp[i] = rc ? P[ids[i]].r : Qb[ids[i]].c;
      }
      std::vector<double*> dst(br.size());
      for (size_t i = 0; i < br.size(); ++i) dst[i] = reinterpret_cast<double*>(V + out->block_off[adm_level[l][i]]);
      cdev_project(dev.get(), rc ? pp.data() : nullptr, kp.data(), static_cast<int>(br.size()), br.data(), bc.data(),
                   dst.data());
    }
    dev_done = true;
    } catch (const std::exception& e) {  // host path below recomputes every coupling
      if (trace) std::fprintf(stderr, "[construct] device pass failed (%s); host path\n", e.what());
      dev.reset();
    }
  }
  if (!dev_done) {
    // the few upper-level blocks (k up to 729) cost ~10^4 leaf-level blocks each: heaviest first,
    // one block per grab
    std::vector<int64_t> order(adm);
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
      return int64_t(cb[b.row[x]].k()) * cb[b.col[x]].k() > int64_t(cb[b.row[y]].k()) * cb[b.col[y]].k();
    });
    pfor(static_cast<int64_t>(order.size()), threads, [&](int64_t a) {
      const int64_t q = order[a];
      M<S> Sq = coupling_raw(q);
      if (rc) {
        M<S> PS;
        gemm(kN, kN, P[b.row[q]], Sq, PS);
        gemm(kN, kT, PS, P[b.col[q]], Sq);
      }
      std::copy(Sq.d.begin(), Sq.d.end(), V + out->block_off[q]);
    }, 1);
  }
  tick("couplings");
  pfor(b.n_blocks, threads, [&](int64_t q) {
    if (b.kind[q] != H2C_INADMISSIBLE_LEAF) return;
    const int r = b.row[q], s = b.col[q];
    const int nr = t.end[r] - t.begin[r], ns = t.end[s] - t.begin[s];
    for (int j = 0; j < ns; ++j) {
      const int pj = perm[t.begin[s] + j];
      for (int i = 0; i < nr; ++i) {
        const int pi = perm[t.begin[r] + i];
        S v = S(diagonal);
        if (pi != pj) {
          const double* x = &xyz[3 * pi];
          const double* y = &xyz[3 * pj];
          const double d = std::sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) +
                                     (x[2] - y[2]) * (x[2] - y[2]));
          if (d == 0.0) throw std::runtime_error("duplicate points");
          v = G(d);
        }
        V[out->block_off[q] + i + int64_t(j) * nr] = v;
      }
    }
  });
  out->col_rank = out->row_rank;
  out->col_dg = out->row_dg;
  out->col_off = out->row_off;
  return out;
}

}  // namespace

std::unique_ptr<HostH2> build_chebyshev(const h2c_tree& t, const h2c_blocks& b, const double* xyz, int kernel,
                                        double kappa, double diagonal, const int* orders, double eps_recompress,
                                        int threads) {
  if (!(eps_recompress >= 0.0 && eps_recompress < 1.0)) throw std::invalid_argument("eps_recompress must be in [0,1)");
  if (kernel == 1) return chebyshev_impl<std::complex<double>>(t, b, xyz, kernel, kappa, diagonal, orders,
                                                               eps_recompress, threads);
  return chebyshev_impl<double>(t, b, xyz, kernel, kappa, diagonal, orders, eps_recompress, threads);
}

std::unique_ptr<HostH2> build_fd_laplacian(const h2c_tree& t, const h2c_blocks& b, const double* xyz, double h) {
  const int nc = t.n_clusters, D = t.depth;
  auto out = std::make_unique<HostH2>();
  out->scalar = H2C_REAL;
  out->row_rank.assign(nc, 0);
  out->row_dg.assign(nc, 0);
  out->row_off.assign(nc, -1);
  int64_t total = 0;
  for (int c = 0; c < nc; ++c) {
    if (t.parent[c] < 0 && D > 0) continue;
    out->row_rank[c] = 1;
    out->row_dg[c] = 1;
    out->row_off[c] = total;
    total += t.child0[c] < 0 ? (t.end[c] - t.begin[c]) : 2;
  }
  out->block_off.assign(b.n_blocks, -1);
  for (int64_t q = 0; q < b.n_blocks; ++q) {
    if (b.kind[q] == H2C_ADMISSIBLE) {
      out->block_off[q] = total;
      total += 1;
    } else if (b.kind[q] == H2C_INADMISSIBLE_LEAF) {
      out->block_off[q] = total;
      total += int64_t(t.end[b.row[q]] - t.begin[b.row[q]]) * (t.end[b.col[q]] - t.begin[b.col[q]]);
    }
  }
  out->values.assign(total, 0.0);
  for (int c = 0; c < nc; ++c)
    if (out->row_off[c] >= 0) out->values[out->row_off[c]] = 1.0;  // e_1
  for (int64_t q = 0; q < b.n_blocks; ++q) {
    if (b.kind[q] != H2C_INADMISSIBLE_LEAF) continue;
    const int r = b.row[q], s = b.col[q];
    const int nr = t.end[r] - t.begin[r], ns = t.end[s] - t.begin[s];
    for (int j = 0; j < ns; ++j)
      for (int i = 0; i < nr; ++i) {
        const int pi = t.perm[t.begin[r] + i], pj = t.perm[t.begin[s] + j];
        double v = 0.0;
        if (pi == pj) v = 6.0;
        else {
          const double* x = &xyz[3 * pi];
          const double* y = &xyz[3 * pj];
          const double d = std::sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) +
                                     (x[2] - y[2]) * (x[2] - y[2]));
          if (std::abs(d - h) <= 1e-9 * h) v = -1.0;
        }
        out->values[out->block_off[q] + i + int64_t(j) * nr] = v;
      }
  }
  out->col_rank = out->row_rank;
  out->col_dg = out->row_dg;
  out->col_off = out->row_off;
  return out;
}

}  // namespace h2b
