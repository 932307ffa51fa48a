// Device evaluation of the interpolation couplings of the Chebyshev constructor
// (see construct_dev.hpp).  Per chunk of admissible blocks of one level:
//   1. cheb_kernel_eval: K_b = K(xi_t, xi_s) at the tensor Chebyshev node pairs,
//      stored as the stacked real matrix [Re K; Im K] (W k x k);
//   2. X_b = K_b R_s^T                       (W k x r, real)
//   3. S_b = R_t X_b  per real/imaginary part (r x r), interleaved;
//   4. grams: Z_t += sum_{b in row t} S_b S_b^H, the segmented sum over the row's blocks in
//      block order (deterministic); project: P_t S_b P_s^T (two products).
// Every product runs on the engine's own segmented batched DMMA kernel (seg_gemm3,
// kernels.cuh) - no library GEMM.  All per-cluster matrices are zero-padded to the level's
// largest rank / node count rounded up to 8 (the kernel's k-chunk), which is exact for
// every product above.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "construct_dev.hpp"
#include "kernels.cuh"

namespace h2b {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("construct (device): ") + what + ": " + cudaGetErrorString(e));
}
int up8(int x) { return (x + 7) / 8 * 8; }

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev() = default;
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() { release(); }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    ck(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)), "cudaMalloc");
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// node coordinate d of node index i (i = ix + m (iy + m iz)) of a box (c[3], h[3])
__device__ __forceinline__ void node_xyz(const double* box, int m, int i, double x[3]) {
  const int id[3] = {i % m, (i / m) % m, i / (m * m)};
#pragma unroll
  for (int d = 0; d < 3; ++d) x[d] = box[d] + box[3 + d] * cos((2.0 * id[d] + 1.0) * M_PI / (2.0 * m));
}

// K_b for the blocks of a chunk: out[b] is (W kp) x kp column-major (kp = k rounded up to 8, zero
// padding), rows [0,kp) real part, [kp, 2kp) imaginary part (complex); kernel 1/(4 pi r) or
// exp(-i kappa r)/(4 pi r)
__global__ void cheb_kernel_eval(const double* boxes, int m, int k, int kp, const int* brow, const int* bcol, int W,
                                 double kappa, double* out) {
  const int b = blockIdx.x;
  const double* bt = boxes + 6 * brow[b];
  const double* bs = boxes + 6 * bcol[b];
  double* K = out + (size_t)b * W * kp * kp;
  for (int x = blockIdx.y * blockDim.x + threadIdx.x; x < kp * kp; x += gridDim.y * blockDim.x) {
    const int i = x % kp, j = x / kp;
    double re = 0.0, im = 0.0;
    if (i < k && j < k) {
      double xi[3], yj[3];
      node_xyz(bt, m, i, xi);
      node_xyz(bs, m, j, yj);
      const double dx = xi[0] - yj[0], dy = xi[1] - yj[1], dz = xi[2] - yj[2];
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double f = 1.0 / (4.0 * M_PI * r);
      if (W == 1) {
        re = f;
      } else {
        double sn, cs;
        sincos(kappa * r, &sn, &cs);
        re = f * cs;
        im = -f * sn;
      }
    }
    K[i + (size_t)j * W * kp] = re;
    if (W == 2) K[kp + i + (size_t)j * 2 * kp] = im;
  }
}

// Sc[b] = S0[b] + i S1[b]  (r x r planes -> interleaved complex)
__global__ void interleave_kernel(const double* planes, int rr, double* out) {
  const int b = blockIdx.x;
  const double* re = planes + (size_t)(2 * b) * rr;
  const double* im = planes + (size_t)(2 * b + 1) * rr;
  double* o = out + (size_t)b * 2 * rr;
  for (int x = threadIdx.x; x < rr; x += blockDim.x) {
    o[2 * x] = re[x];
    o[2 * x + 1] = im[x];
  }
}

__global__ void iota_kernel(int* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}

// ---- the engine's segmented batched DMMA kernel (kernels.cuh) as the constructor's GEMM --------
template <int TM, int TN, bool CX>
void seg_launch_cfg(const SegParams& sp, cudaStream_t s) {
  constexpr int sm = Seg2Cfg<TM, TN, CX, 8, 4>::SMEM;
  auto kern = seg_gemm3_kernel<TM, TN, CX, 8, 4, 2, 2, CX>;  // complex: 3-multiplication form
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm), "smem attribute");
  const int tiles = ((sp.M + TM - 1) / TM) * ((sp.N + TN - 1) / TN);
  // grid.x carries the outputs (<= 2^31 - 1), grid.y the tiles of one output
  kern<<<dim3(sp.n_out, tiles), 128, sm, s>>>(sp);
  ck(cudaGetLastError(), "seg_gemm launch");
}

template <bool CX>
void seg_launch_tiles(const SegParams& sp, cudaStream_t s) {
  const bool m64 = sp.M > 32, n64 = sp.N > 32;
  if (m64 && n64) seg_launch_cfg<64, 64, CX>(sp, s);
  else if (m64) seg_launch_cfg<64, 32, CX>(sp, s);
  else if (n64) seg_launch_cfg<32, 64, CX>(sp, s);
  else seg_launch_cfg<32, 32, CX>(sp, s);
}

struct Mat {  // batch of column-major matrices: base, element stride, element offset, ld, op, index list
  const double* p;
  long long stride, off;
  int ld, op;
  const int* idx;  // matrix index per output (nullptr: the output's own index)
};

// out[t] (M x N, stride Os, ld Old; storage index omap[t] if given) (+)= sum over the outputs'
// entries of op(L) op(R) with inner dimension K; ptr == nullptr: one entry per output
void seg_product(bool cplx, cudaStream_t s, double* out, long long Os, long long Ooff, int Old, const int* omap, int M,
                 int N, int n_out, bool acc, const Mat& L, const Mat& R, int K, const int* ptr = nullptr) {
  if (n_out <= 0) return;
  if (K % 8 != 0) throw std::logic_error("construct (device): inner dimension not a multiple of 8");
  SegParams sp{};
  sp.out = out;
  sp.Os = Os;
  sp.Ooff = Ooff;
  sp.Old = Old;
  sp.omap = omap;
  sp.M = M;
  sp.N = N;
  sp.n_out = n_out;
  sp.accumulate = acc ? 1 : 0;
  sp.ngroups = 1;
  SegGroup& G = sp.g[0];
  G.L = L.p;
  G.Ls = L.stride;
  G.Loff = L.off;
  G.Lld = L.ld;
  G.opL = L.op;
  G.R = R.p;
  G.Rs = R.stride;
  G.Roff = R.off;
  G.Rld = R.ld;
  G.opR = R.op;
  G.K = K;
  G.ptr = ptr;
  G.li = L.idx;
  G.ri = R.idx;
  if (cplx) seg_launch_tiles<true>(sp, s);
  else seg_launch_tiles<false>(sp, s);
}

}  // namespace

struct CouplingDev {
  bool cplx = false;
  int W = 1;
  double kappa = 0.0;
  cudaStream_t s = nullptr;
  // level: n clusters of order m (k = m^3 nodes, kp = k rounded up to 8), ranks r[i] <= rmax,
  // rp = rmax rounded up to 8
  int n = 0, m = 0, k = 0, kp = 0, rmax = 0, rp = 0;
  std::vector<int> r;
  Dev<double> box, R, P, K, X, Sp, Sc, T1, Z, out;
  Dev<int> brow, bcol, segp, segr, iota;
  std::vector<double> host_out;
};

bool cdev_available() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

CouplingDev* cdev_create(bool cplx, double kappa) {
  auto* d = new CouplingDev;
  d->cplx = cplx;
  d->W = cplx ? 2 : 1;
  d->kappa = kappa;
  ck(cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking), "stream");
  return d;
}

void cdev_destroy(CouplingDev* d) {
  if (!d) return;
  if (d->s) cudaStreamSynchronize(d->s);
  if (d->s) cudaStreamDestroy(d->s);
  delete d;
}

void cdev_level(CouplingDev* d, int n, const double* boxes, int m, const double* const* R, const int* r) {
  d->n = n;
  d->m = m;
  d->k = m * m * m;
  d->kp = up8(d->k);
  d->r.assign(r, r + n);
  d->rmax = 1;
  for (int i = 0; i < n; ++i) d->rmax = std::max(d->rmax, r[i]);
  d->rp = up8(d->rmax);
  d->box.alloc(size_t(6) * n);
  ck(cudaMemcpy(d->box.p, boxes, sizeof(double) * 6 * n, cudaMemcpyHostToDevice), "boxes");
  // R_i as rp x kp, zero padded
  const size_t rk = size_t(d->rp) * d->kp;
  std::vector<double> hr(rk * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < d->k; ++c)
      for (int a = 0; a < r[i]; ++a) hr[i * rk + a + size_t(c) * d->rp] = R[i][a + size_t(c) * r[i]];
  d->R.alloc(rk * n);
  ck(cudaMemcpy(d->R.p, hr.data(), sizeof(double) * rk * n, cudaMemcpyHostToDevice), "R");
}

namespace {

// S (interleaved when complex, rp x rp per block) for blocks [b0, b0 + nbc) of the uploaded lists
void chunk_couplings(CouplingDev* d, int b0, int nbc) {
  const int W = d->W, k = d->k, kp = d->kp, rp = d->rp;
  const size_t wkk = size_t(W) * kp * kp, wkr = size_t(W) * kp * rp, rr = size_t(rp) * rp;
  d->K.alloc(wkk * nbc);
  d->X.alloc(wkr * nbc);
  d->Sp.alloc(rr * W * nbc);
  {
    dim3 grid(nbc, std::max(1, std::min(64, (kp * kp + 255) / 256)));
    cheb_kernel_eval<<<grid, 256, 0, d->s>>>(d->box.p, d->m, k, kp, d->brow.p + b0, d->bcol.p + b0, W, d->kappa,
                                             d->K.p);
    ck(cudaGetLastError(), "kernel eval");
  }
  const size_t rk = size_t(rp) * kp;
  // X_b = K_b R_s^T  (W kp x rp; real product on the stacked [Re; Im] rows, R is real)
  seg_product(false, d->s, d->X.p, (long long)wkr, 0, W * kp, nullptr, W * kp, rp, nbc, false,
              Mat{d->K.p, (long long)wkk, 0, W * kp, OP_N, nullptr},
              Mat{d->R.p, (long long)rk, 0, rp, OP_T, d->bcol.p + b0}, kp);
  // S_b,part = R_t X_b,part  (rp x rp), planes [Re S_b; Im S_b] of rr doubles each
  for (int p = 0; p < W; ++p)
    seg_product(false, d->s, d->Sp.p, (long long)(rr * W), (long long)(p * rr), rp, nullptr, rp, rp, nbc, false,
                Mat{d->R.p, (long long)rk, 0, rp, OP_N, d->brow.p + b0},
                Mat{d->X.p, (long long)wkr, (long long)p * kp, W * kp, OP_N, nullptr}, kp);
  if (W == 2) {
    d->Sc.alloc(rr * 2 * nbc);
    interleave_kernel<<<nbc, 256, 0, d->s>>>(d->Sp.p, static_cast<int>(rr), d->Sc.p);
    ck(cudaGetLastError(), "interleave");
  }
}

const double* chunk_S(CouplingDev* d) { return d->W == 2 ? d->Sc.p : d->Sp.p; }

int chunk_size(CouplingDev* d, size_t extra_per_block) {
  const size_t W = d->W, k = d->kp, r = d->rp;
  const size_t per = W * k * k + W * k * r + 2 * W * r * r + extra_per_block;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const size_t budget = std::min<size_t>(fr / 2, size_t(8) << 30) / 8;
  return static_cast<int>(std::max<size_t>(16, std::min<size_t>(budget / per, 1 << 16)));
}

void upload_blocks(CouplingDev* d, int nb, const int* brow, const int* bcol) {
  d->brow.alloc(nb);
  d->bcol.alloc(nb);
  ck(cudaMemcpy(d->brow.p, brow, sizeof(int) * nb, cudaMemcpyHostToDevice), "brow");
  ck(cudaMemcpy(d->bcol.p, bcol, sizeof(int) * nb, cudaMemcpyHostToDevice), "bcol");
}

}  // namespace

void cdev_grams(CouplingDev* d, int nb, const int* brow, const int* bcol, double* const* zout) {
  if (nb <= 0) return;
  const int W = d->W, rp = d->rp;
  const size_t rr = size_t(rp) * rp;  // elements per Gram
  upload_blocks(d, nb, brow, bcol);
  d->Z.alloc(rr * W * d->n);
  ck(cudaMemsetAsync(d->Z.p, 0, sizeof(double) * rr * W * d->n, d->s), "Z");
  const int chunk = chunk_size(d, 0);
  d->iota.alloc(std::min(chunk, nb));
  {
    const int ni = std::min(chunk, nb);
    iota_kernel<<<(ni + 255) / 256, 256, 0, d->s>>>(d->iota.p, ni);
    ck(cudaGetLastError(), "iota");
  }
  for (int b0 = 0; b0 < nb; b0 += chunk) {
    const int nbc = std::min(chunk, nb - b0);
    chunk_couplings(d, b0, nbc);
    // segments of equal row within the chunk (blocks are sorted by row): Z_row += sum_b S_b S_b^H,
    // one output per segment, its blocks in ascending order (a row cut by a chunk boundary
    // continues in the next chunk: accumulate)
    std::vector<int> sp{0}, sr;
    for (int b = 0; b < nbc; ++b) {
      if (b > 0 && brow[b0 + b] != brow[b0 + b - 1]) sp.push_back(b);
      if (sr.size() < sp.size()) sr.push_back(brow[b0 + b]);
    }
    sp.push_back(nbc);
    d->segp.alloc(sp.size());
    d->segr.alloc(sr.size());
    ck(cudaMemcpyAsync(d->segp.p, sp.data(), sizeof(int) * sp.size(), cudaMemcpyHostToDevice, d->s), "seg");
    ck(cudaMemcpyAsync(d->segr.p, sr.data(), sizeof(int) * sr.size(), cudaMemcpyHostToDevice, d->s), "seg");
    const double* S = chunk_S(d);
    seg_product(W == 2, d->s, d->Z.p, (long long)rr, 0, rp, d->segr.p, rp, rp, static_cast<int>(sr.size()), true,
                Mat{S, (long long)rr, 0, rp, OP_N, d->iota.p}, Mat{S, (long long)rr, 0, rp, W == 2 ? OP_H : OP_T, d->iota.p},
                rp, d->segp.p);
    ck(cudaStreamSynchronize(d->s), "sync");  // sp / sr go out of scope; K, X, S are reused
  }
  std::vector<double> hz(rr * W * d->n);
  ck(cudaMemcpy(hz.data(), d->Z.p, sizeof(double) * hz.size(), cudaMemcpyDeviceToHost), "Z down");
  std::vector<char> seen(d->n, 0);
  for (int b = 0; b < nb; ++b) seen[brow[b]] = 1;
  for (int i = 0; i < d->n; ++i) {
    if (!seen[i] || !zout[i]) continue;
    const int ri = d->r[i];
    for (int c = 0; c < ri; ++c)
      for (int a = 0; a < ri; ++a)
        for (int w = 0; w < W; ++w)
          zout[i][(a + size_t(c) * ri) * W + w] += hz[(i * rr + a + size_t(c) * rp) * W + w];
  }
}

void cdev_project(CouplingDev* d, const double* const* P, const int* kp, int nb, const int* brow, const int* bcol,
                  double* const* dst) {
  if (nb <= 0) return;
  const int W = d->W, rp = d->rp;
  const size_t rr = size_t(rp) * rp;  // elements
  upload_blocks(d, nb, brow, bcol);
  int kq = 8;  // padded new rank
  if (P) {
    int kpmax = 1;
    for (int i = 0; i < d->n; ++i) kpmax = std::max(kpmax, kp[i]);
    kq = up8(kpmax);
    const size_t pr = size_t(kq) * rp;  // elements per P_i (kq x rp, zero padded)
    std::vector<double> hp(pr * W * d->n, 0.0);
    for (int i = 0; i < d->n; ++i)
      for (int c = 0; c < d->r[i]; ++c)
        for (int a = 0; a < kp[i]; ++a)
          for (int w = 0; w < W; ++w)
            hp[(i * pr + a + size_t(c) * kq) * W + w] = P[i][(a + size_t(c) * kp[i]) * W + w];
    d->P.alloc(hp.size());
    ck(cudaMemcpy(d->P.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice), "P");
  }
  const size_t oo = P ? size_t(kq) * kq : rr;  // elements per result
  const int chunk = chunk_size(d, P ? (size_t(kq) * rp + oo) * W : 0);
  for (int b0 = 0; b0 < nb; b0 += chunk) {
    const int nbc = std::min(chunk, nb - b0);
    chunk_couplings(d, b0, nbc);
    const double* S = chunk_S(d);
    const double* res = S;
    if (P) {
      const size_t pr = size_t(kq) * rp, t1 = size_t(kq) * rp;
      d->T1.alloc(t1 * W * nbc);
      d->out.alloc(oo * W * nbc);
      // T1_b = P_t S_b  (kq x rp), out_b = T1_b P_s^T  (kq x kq)
      seg_product(W == 2, d->s, d->T1.p, (long long)t1, 0, kq, nullptr, kq, rp, nbc, false,
                  Mat{d->P.p, (long long)pr, 0, kq, OP_N, d->brow.p + b0}, Mat{S, (long long)rr, 0, rp, OP_N, nullptr}, rp);
      seg_product(W == 2, d->s, d->out.p, (long long)oo, 0, kq, nullptr, kq, kq, nbc, false,
                  Mat{d->T1.p, (long long)t1, 0, kq, OP_N, nullptr},
                  Mat{d->P.p, (long long)pr, 0, kq, OP_T, d->bcol.p + b0}, rp);
      res = d->out.p;
    }
    d->host_out.resize(oo * W * nbc);
    ck(cudaMemcpyAsync(d->host_out.data(), res, sizeof(double) * oo * W * nbc, cudaMemcpyDeviceToHost, d->s), "out down");
    ck(cudaStreamSynchronize(d->s), "sync");
    const int ld = P ? kq : rp;
    for (int b = 0; b < nbc; ++b) {
      const int t = brow[b0 + b], u = bcol[b0 + b];
      const int mr = P ? kp[t] : d->r[t], mc = P ? kp[u] : d->r[u];
      double* o = dst[b0 + b];
      const double* src = d->host_out.data() + b * oo * W;
      for (int c = 0; c < mc; ++c)
        std::memcpy(o + size_t(c) * mr * W, src + size_t(c) * ld * W, sizeof(double) * mr * W);
    }
  }
}

}  // namespace h2b
