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
#include <cmath>
#include <complex>
#include <stdexcept>
#include <thread>

#include "structure.hpp"

namespace h2b {

namespace {

template <class F>
void pfor(int64_t n, int threads, F&& f) {
  threads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n)));
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (;;) {
      const int64_t i = next.fetch_add(64);
      if (i >= n) break;
      for (int64_t k = i; k < std::min(n, i + 64); ++k) f(k);
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

std::unique_ptr<HostH2> build_chebyshev(const h2c_tree& t, const h2c_blocks& b, const double* xyz, int kernel,
                                        double kappa, double diagonal, int order, double eps_recompress,
                                        int threads) {
  if (order < 1) throw std::invalid_argument("chebyshev order must be >= 1");
  if (eps_recompress > 0) throw std::invalid_argument("recompression is not available in this build");
  const bool cplx = kernel == 1;
  const int W = cplx ? 2 : 1;
  const int m = order, k = m * m * m;
  const int nc = t.n_clusters, D = t.depth;
  auto out = std::make_unique<HostH2>();
  out->scalar = cplx ? H2C_COMPLEX : H2C_REAL;

  // interpolation boxes: cluster bounding boxes (degenerate extents widened)
  std::vector<Box> box(nc);
  for (int c = 0; c < nc; ++c) {
    const double* bb = &t.bbox[6 * c];
    double ext = 0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, bb[d + 3] - bb[d]);
    for (int d = 0; d < 3; ++d) {
      box[c].c[d] = 0.5 * (bb[d] + bb[d + 3]);
      box[c].h[d] = std::max(0.5 * (bb[d + 3] - bb[d]), 1e-6 * std::max(ext, 1e-300));
    }
  }
  // nested bases bottom-up: Q (stored basis) and R factors
  std::vector<Dm> Qb(nc), Rb(nc);
  std::vector<int> lvl_ids_start;
  std::vector<std::vector<int>> levels(D + 1);
  for (int c = 0; c < nc; ++c) levels[t.level[c]].push_back(c);
  const int* perm = t.perm;
  for (int l = D; l >= (D == 0 ? 0 : 1); --l) {
    const auto& ids = levels[l];
    pfor(static_cast<int64_t>(ids.size()), threads, [&](int64_t q) {
      const int c = ids[q];
      if (t.child0[c] < 0) {
        const int n = t.end[c] - t.begin[c];
        Dm V(n, k);
        for (int p = 0; p < n; ++p) {
          const double* x = &xyz[3 * perm[t.begin[c] + p]];
          double lx[64], ly[64], lz[64];
          for (int i = 0; i < m; ++i) {
            lx[i] = lagrange(box[c], 0, i, m, x[0]);
            ly[i] = lagrange(box[c], 1, i, m, x[1]);
            lz[i] = lagrange(box[c], 2, i, m, x[2]);
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
          Dm E(k, k);  // E[nu', nu] = L^parent_nu(xi^child_nu')
          for (int jz = 0; jz < m; ++jz)
            for (int jy = 0; jy < m; ++jy)
              for (int jx = 0; jx < m; ++jx) {
                const double px = cheb_node(box[ch], 0, jx, m), py = cheb_node(box[ch], 1, jy, m),
                             pz = cheb_node(box[ch], 2, jz, m);
                for (int iz = 0; iz < m; ++iz)
                  for (int iy = 0; iy < m; ++iy)
                    for (int ix = 0; ix < m; ++ix)
                      E(jx + m * (jy + m * jz), ix + m * (iy + m * iz)) =
                          lagrange(box[c], 0, ix, m, px) * lagrange(box[c], 1, iy, m, py) *
                          lagrange(box[c], 2, iz, m, pz);
              }
          const Dm RE = matmul(Rb[ch], E);
          for (int j = 0; j < k; ++j)
            for (int i = 0; i < RE.r; ++i) Z(i + (s ? r1 : 0), j) = RE(i, j);
        }
        house_qr(Z, Qb[c], Rb[c]);
      }
    });
  }
  // kernel value at distance r
  auto G = [&](double r, double& re, double& im) {
    const double f = 1.0 / (4.0 * M_PI * r);
    if (!cplx) {
      re = f;
      im = 0.0;
    } else {
      re = f * std::cos(kappa * r);
      im = -f * std::sin(kappa * r);
    }
  };
  // layout: bases (row == col, shared offsets), then blocks in global order
  int64_t total = 0;
  out->row_rank.assign(nc, 0);
  out->row_dg.assign(nc, 0);
  out->row_off.assign(nc, -1);
  for (int c = 0; c < nc; ++c) {
    if (t.parent[c] < 0 && D > 0) continue;
    out->row_rank[c] = Qb[c].c;
    out->row_off[c] = total;
    total += int64_t(Qb[c].r) * Qb[c].c;
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
  double* V = out->values.data();
  for (int c = 0; c < nc; ++c) {
    if (out->row_off[c] < 0) continue;
    const Dm& Q = Qb[c];
    for (int j = 0; j < Q.c; ++j)
      for (int i = 0; i < Q.r; ++i) V[(out->row_off[c] + i + int64_t(j) * Q.r) * W] = Q(i, j);
  }
  pfor(b.n_blocks, threads, [&](int64_t q) {
    const int r = b.row[q], s = b.col[q];
    if (b.kind[q] == H2C_ADMISSIBLE) {
      // S = kernel at node pairs, then R_r S R_s^T
      Dm Sre(k, k), Sim(k, k);
      for (int jz = 0; jz < m; ++jz)
        for (int jy = 0; jy < m; ++jy)
          for (int jx = 0; jx < m; ++jx) {
            const double y[3] = {cheb_node(box[s], 0, jx, m), cheb_node(box[s], 1, jy, m),
                                 cheb_node(box[s], 2, jz, m)};
            const int jj = jx + m * (jy + m * jz);
            for (int iz = 0; iz < m; ++iz)
              for (int iy = 0; iy < m; ++iy)
                for (int ix = 0; ix < m; ++ix) {
                  const double x[3] = {cheb_node(box[r], 0, ix, m), cheb_node(box[r], 1, iy, m),
                                       cheb_node(box[r], 2, iz, m)};
                  const double d = std::sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) +
                                             (x[2] - y[2]) * (x[2] - y[2]));
                  double re, im;
                  G(d, re, im);
                  Sre(ix + m * (iy + m * iz), jj) = re;
                  Sim(ix + m * (iy + m * iz), jj) = im;
                }
          }
      const Dm& Rr = Rb[r];
      const Dm& Rs = Rb[s];
      Dm RsT(Rs.c, Rs.r);
      for (int i = 0; i < Rs.r; ++i)
        for (int j = 0; j < Rs.c; ++j) RsT(j, i) = Rs(i, j);
      for (int part = 0; part < W; ++part) {
        const Dm C = matmul(matmul(Rr, part ? Sim : Sre), RsT);
        for (int j = 0; j < C.c; ++j)
          for (int i = 0; i < C.r; ++i) V[(out->block_off[q] + i + int64_t(j) * C.r) * W + part] = C(i, j);
      }
    } else if (b.kind[q] == H2C_INADMISSIBLE_LEAF) {
      const int nr = t.end[r] - t.begin[r], ns = t.end[s] - t.begin[s];
      for (int j = 0; j < ns; ++j) {
        const int pj = perm[t.begin[s] + j];
        for (int i = 0; i < nr; ++i) {
          const int pi = perm[t.begin[r] + i];
          double re = diagonal, im = 0.0;
          if (pi != pj) {
            const double* x = &xyz[3 * pi];
            const double* y = &xyz[3 * pj];
            const double d = std::sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) +
                                       (x[2] - y[2]) * (x[2] - y[2]));
            if (d == 0.0) throw std::runtime_error("duplicate points");
            G(d, re, im);
          }
          V[(out->block_off[q] + i + int64_t(j) * nr) * W] = re;
          if (cplx) V[(out->block_off[q] + i + int64_t(j) * nr) * W + 1] = im;
        }
      }
    }
  });
  out->col_rank = out->row_rank;
  out->col_dg = out->row_dg;
  out->col_off = out->row_off;
  return out;
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
