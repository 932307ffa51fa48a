// Device evaluation of the interpolation couplings of the Chebyshev constructor
// (see construct_dev.hpp).  Per chunk of admissible blocks of one level:
//   1. cheb_kernel_eval: K_b = K(xi_t, xi_s) at the tensor Chebyshev node pairs,
//      stored as the stacked real matrix [Re K; Im K] (W k x k);
//   2. X_b = K_b R_s^T                       (batched DGEMM, W k x r)
//   3. S_b = R_t X_b  per real/imaginary part (batched DGEMM, r x r), interleaved;
//   4. grams: G_b = S_b S_b^H (batched ZGEMM/DGEMM), summed per row cluster in block
//      order (deterministic); project: P_t S_b P_s^T (two batched GEMMs).
// All per-cluster matrices are zero-padded to the level's largest rank, which is
// exact for every product above.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "construct_dev.hpp"

namespace h2b {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("construct (device): ") + what + ": " + cudaGetErrorString(e));
}
void cb(cublasStatus_t e, const char* what) {
  if (e != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string("construct (device): cuBLAS ") + what);
}

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

// K_b for the blocks of a chunk: out[b] is (W k) x k column-major, rows [0,k) real part,
// [k, 2k) imaginary part (complex); kernel 1/(4 pi r) or exp(-i kappa r)/(4 pi r)
__global__ void cheb_kernel_eval(const double* boxes, int m, int k, const int* brow, const int* bcol, int W,
                                 double kappa, double* out) {
  const int b = blockIdx.x;
  const double* bt = boxes + 6 * brow[b];
  const double* bs = boxes + 6 * bcol[b];
  double* K = out + (size_t)b * W * k * k;
  for (int x = blockIdx.y * blockDim.x + threadIdx.x; x < k * k; x += gridDim.y * blockDim.x) {
    const int i = x % k, j = x / k;
    double xi[3], yj[3];
    node_xyz(bt, m, i, xi);
    node_xyz(bs, m, j, yj);
    const double dx = xi[0] - yj[0], dy = xi[1] - yj[1], dz = xi[2] - yj[2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double f = 1.0 / (4.0 * M_PI * r);
    if (W == 1) {
      K[i + (size_t)j * k] = f;
    } else {
      double sn, cs;
      sincos(kappa * r, &sn, &cs);
      K[i + (size_t)j * 2 * k] = f * cs;
      K[k + i + (size_t)j * 2 * k] = -f * sn;
    }
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

// Z[row] += sum of G over the row's consecutive blocks (fixed order)
__global__ void row_sum_kernel(const double* G, const int* seg_ptr, const int* seg_row, int elems, double* Z) {
  const int s = blockIdx.x;
  const int b0 = seg_ptr[s], b1 = seg_ptr[s + 1];
  double* z = Z + (size_t)seg_row[s] * elems;
  for (int x = blockIdx.y * blockDim.x + threadIdx.x; x < elems; x += gridDim.y * blockDim.x) {
    double v = z[x];
    for (int b = b0; b < b1; ++b) v += G[(size_t)b * elems + x];
    z[x] = v;
  }
}

}  // namespace

struct CouplingDev {
  bool cplx = false;
  int W = 1;
  double kappa = 0.0;
  cublasHandle_t h = nullptr;
  cudaStream_t s = nullptr;
  // level
  int n = 0, m = 0, k = 0, rmax = 0;
  std::vector<int> r;
  Dev<double> box, R, P, K, X, Sp, Sc, G, T1, Z, out;
  Dev<int> brow, bcol, segp, segr;
  Dev<const double*> pa, pb;
  Dev<double*> pc;
  std::vector<double> host_out;
  int kpmax = 0;
  std::vector<int> kp;
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
  cb(cublasCreate(&d->h), "create");
  cb(cublasSetStream(d->h, d->s), "set stream");
  return d;
}

void cdev_destroy(CouplingDev* d) {
  if (!d) return;
  if (d->s) cudaStreamSynchronize(d->s);
  if (d->h) cublasDestroy(d->h);
  if (d->s) cudaStreamDestroy(d->s);
  delete d;
}

void cdev_level(CouplingDev* d, int n, const double* boxes, int m, const double* const* R, const int* r) {
  d->n = n;
  d->m = m;
  d->k = m * m * m;
  d->r.assign(r, r + n);
  d->rmax = 1;
  for (int i = 0; i < n; ++i) d->rmax = std::max(d->rmax, r[i]);
  d->box.alloc(size_t(6) * n);
  ck(cudaMemcpy(d->box.p, boxes, sizeof(double) * 6 * n, cudaMemcpyHostToDevice), "boxes");
  const size_t rk = size_t(d->rmax) * d->k;
  std::vector<double> hr(rk * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < d->k; ++c)
      for (int a = 0; a < r[i]; ++a) hr[i * rk + a + size_t(c) * d->rmax] = R[i][a + size_t(c) * r[i]];
  d->R.alloc(rk * n);
  ck(cudaMemcpy(d->R.p, hr.data(), sizeof(double) * rk * n, cudaMemcpyHostToDevice), "R");
}

namespace {

// S (interleaved when complex, rmax x rmax per block) for blocks [b0, b1) of the lists
void chunk_couplings(CouplingDev* d, int b0, int nbc) {
  const int W = d->W, k = d->k, r = d->rmax;
  const size_t wkk = size_t(W) * k * k, wkr = size_t(W) * k * r, rr = size_t(r) * r;
  d->K.alloc(wkk * nbc);
  d->X.alloc(wkr * nbc);
  d->Sp.alloc(rr * W * nbc);
  {
    dim3 grid(nbc, std::max(1, std::min(64, (k * k + 255) / 256)));
    cheb_kernel_eval<<<grid, 256, 0, d->s>>>(d->box.p, d->m, k, d->brow.p + b0, d->bcol.p + b0, W, d->kappa, d->K.p);
    ck(cudaGetLastError(), "kernel eval");
  }
  std::vector<int> hrow(nbc), hcol(nbc);
  ck(cudaMemcpy(hrow.data(), d->brow.p + b0, sizeof(int) * nbc, cudaMemcpyDeviceToHost), "rows");
  ck(cudaMemcpy(hcol.data(), d->bcol.p + b0, sizeof(int) * nbc, cudaMemcpyDeviceToHost), "cols");
  const double one = 1.0, zero = 0.0;
  const size_t rk = size_t(r) * k;
  std::vector<const double*> A(size_t(nbc) * W), B(size_t(nbc) * W);
  std::vector<double*> C(size_t(nbc) * W);
  // X_b = K_b R_s^T  (W k x r)
  for (int b = 0; b < nbc; ++b) {
    A[b] = d->K.p + b * wkk;
    B[b] = d->R.p + hcol[b] * rk;
    C[b] = d->X.p + b * wkr;
  }
  d->pa.alloc(A.size());
  d->pb.alloc(B.size());
  d->pc.alloc(C.size());
  ck(cudaMemcpyAsync(d->pa.p, A.data(), sizeof(void*) * nbc, cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pb.p, B.data(), sizeof(void*) * nbc, cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pc.p, C.data(), sizeof(void*) * nbc, cudaMemcpyHostToDevice, d->s), "ptrs");
  cb(cublasDgemmBatched(d->h, CUBLAS_OP_N, CUBLAS_OP_T, W * k, r, k, &one, d->pa.p, W * k, d->pb.p, r, &zero, d->pc.p,
                        W * k, nbc),
     "X = K R^T");
  // S_b,part = R_t X_b,part  (r x r)
  for (int b = 0; b < nbc; ++b)
    for (int p = 0; p < W; ++p) {
      A[size_t(b) * W + p] = d->R.p + hrow[b] * rk;
      B[size_t(b) * W + p] = d->X.p + b * wkr + size_t(p) * k;
      C[size_t(b) * W + p] = d->Sp.p + (size_t(b) * W + p) * rr;
    }
  ck(cudaStreamSynchronize(d->s), "sync");  // the pointer arrays are rewritten
  ck(cudaMemcpyAsync(d->pa.p, A.data(), sizeof(void*) * A.size(), cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pb.p, B.data(), sizeof(void*) * B.size(), cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pc.p, C.data(), sizeof(void*) * C.size(), cudaMemcpyHostToDevice, d->s), "ptrs");
  cb(cublasDgemmBatched(d->h, CUBLAS_OP_N, CUBLAS_OP_N, r, r, k, &one, d->pa.p, r, d->pb.p, W * k, &zero, d->pc.p, r,
                        nbc * W),
     "S = R X");
  if (W == 2) {
    d->Sc.alloc(rr * 2 * nbc);
    interleave_kernel<<<nbc, 256, 0, d->s>>>(d->Sp.p, static_cast<int>(rr), d->Sc.p);
    ck(cudaGetLastError(), "interleave");
  }
  ck(cudaStreamSynchronize(d->s), "sync");
}

const double* chunk_S(CouplingDev* d) { return d->W == 2 ? d->Sc.p : d->Sp.p; }

// batched C_b = op(A_b) op(B_b) for interleaved-complex (W = 2) or real matrices
void gemm_batched(CouplingDev* d, cublasOperation_t oa, cublasOperation_t ob, int m, int n, int kk,
                  const std::vector<const double*>& A, int lda, const std::vector<const double*>& B, int ldb,
                  const std::vector<double*>& C, int ldc) {
  const int nb = static_cast<int>(A.size());
  d->pa.alloc(nb);
  d->pb.alloc(nb);
  d->pc.alloc(nb);
  ck(cudaMemcpyAsync(d->pa.p, A.data(), sizeof(void*) * nb, cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pb.p, B.data(), sizeof(void*) * nb, cudaMemcpyHostToDevice, d->s), "ptrs");
  ck(cudaMemcpyAsync(d->pc.p, C.data(), sizeof(void*) * nb, cudaMemcpyHostToDevice, d->s), "ptrs");
  if (d->W == 1) {
    const double one = 1.0, zero = 0.0;
    cb(cublasDgemmBatched(d->h, oa, ob, m, n, kk, &one, d->pa.p, lda, d->pb.p, ldb, &zero, d->pc.p, ldc, nb), "dgemm");
  } else {
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
    cb(cublasZgemmBatched(d->h, oa, ob, m, n, kk, &one, reinterpret_cast<const cuDoubleComplex* const*>(d->pa.p), lda,
                          reinterpret_cast<const cuDoubleComplex* const*>(d->pb.p), ldb, &zero,
                          reinterpret_cast<cuDoubleComplex* const*>(d->pc.p), ldc, nb),
       "zgemm");
  }
  ck(cudaStreamSynchronize(d->s), "sync");
}

int chunk_size(CouplingDev* d, int extra_per_block) {
  const size_t W = d->W, k = d->k, r = d->rmax;
  const size_t per = W * k * k + W * k * r + 2 * W * r * r + size_t(extra_per_block);
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
  const int W = d->W, r = d->rmax;
  const size_t rr = size_t(r) * r * W;
  upload_blocks(d, nb, brow, bcol);
  d->Z.alloc(rr * d->n);
  ck(cudaMemset(d->Z.p, 0, sizeof(double) * rr * d->n), "Z");
  const int chunk = chunk_size(d, static_cast<int>(rr));
  for (int b0 = 0; b0 < nb; b0 += chunk) {
    const int nbc = std::min(chunk, nb - b0);
    chunk_couplings(d, b0, nbc);
    const double* S = chunk_S(d);
    d->G.alloc(rr * nbc);
    std::vector<const double*> A(nbc), B(nbc);
    std::vector<double*> C(nbc);
    for (int b = 0; b < nbc; ++b) {
      A[b] = B[b] = S + b * rr;
      C[b] = d->G.p + b * rr;
    }
    gemm_batched(d, CUBLAS_OP_N, W == 2 ? CUBLAS_OP_C : CUBLAS_OP_T, r, r, r, A, r, B, r, C, r);
    // segments of equal row within the chunk (blocks are sorted by row)
    std::vector<int> sp{0}, sr;
    for (int b = 0; b < nbc; ++b) {
      if (b > 0 && brow[b0 + b] != brow[b0 + b - 1]) sp.push_back(b);
      if (sr.size() < sp.size()) sr.push_back(brow[b0 + b]);
    }
    sp.push_back(nbc);
    d->segp.alloc(sp.size());
    d->segr.alloc(sr.size());
    ck(cudaMemcpy(d->segp.p, sp.data(), sizeof(int) * sp.size(), cudaMemcpyHostToDevice), "seg");
    ck(cudaMemcpy(d->segr.p, sr.data(), sizeof(int) * sr.size(), cudaMemcpyHostToDevice), "seg");
    dim3 grid(static_cast<unsigned>(sr.size()), static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(16, rr / 1024))));
    row_sum_kernel<<<grid, 256, 0, d->s>>>(d->G.p, d->segp.p, d->segr.p, static_cast<int>(rr), d->Z.p);
    ck(cudaGetLastError(), "row sum");
    ck(cudaStreamSynchronize(d->s), "sync");
  }
  std::vector<double> hz(rr * d->n);
  ck(cudaMemcpy(hz.data(), d->Z.p, sizeof(double) * hz.size(), cudaMemcpyDeviceToHost), "Z down");
  std::vector<char> seen(d->n, 0);
  for (int b = 0; b < nb; ++b) seen[brow[b]] = 1;
  for (int i = 0; i < d->n; ++i) {
    if (!seen[i] || !zout[i]) continue;
    const int ri = d->r[i];
    for (int c = 0; c < ri; ++c)
      for (int a = 0; a < ri; ++a)
        for (int w = 0; w < W; ++w) zout[i][(a + size_t(c) * ri) * W + w] += hz[i * rr + (a + size_t(c) * r) * W + w];
  }
}

void cdev_project(CouplingDev* d, const double* const* P, const int* kp, int nb, const int* brow, const int* bcol,
                  double* const* dst) {
  if (nb <= 0) return;
  const int W = d->W, r = d->rmax;
  const size_t rr = size_t(r) * r * W;
  upload_blocks(d, nb, brow, bcol);
  int kpmax = 1;
  if (P) {
    for (int i = 0; i < d->n; ++i) kpmax = std::max(kpmax, kp[i]);
    const size_t pr = size_t(kpmax) * r * W;
    std::vector<double> hp(pr * d->n, 0.0);
    for (int i = 0; i < d->n; ++i)
      for (int c = 0; c < d->r[i]; ++c)
        for (int a = 0; a < kp[i]; ++a)
          for (int w = 0; w < W; ++w) hp[i * pr + (a + size_t(c) * kpmax) * W + w] = P[i][(a + size_t(c) * kp[i]) * W + w];
    d->P.alloc(pr * d->n);
    ck(cudaMemcpy(d->P.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice), "P");
  }
  const size_t oo = P ? size_t(kpmax) * kpmax * W : rr;
  const int chunk = chunk_size(d, static_cast<int>(P ? size_t(kpmax) * r * W + oo : 0));
  for (int b0 = 0; b0 < nb; b0 += chunk) {
    const int nbc = std::min(chunk, nb - b0);
    chunk_couplings(d, b0, nbc);
    const double* S = chunk_S(d);
    const double* res = S;
    if (P) {
      const size_t pr = size_t(kpmax) * r * W;
      d->T1.alloc(size_t(kpmax) * r * W * nbc);
      d->out.alloc(oo * nbc);
      std::vector<const double*> A(nbc), B(nbc);
      std::vector<double*> C(nbc);
      for (int b = 0; b < nbc; ++b) {  // T1 = P_t S
        A[b] = d->P.p + brow[b0 + b] * pr;
        B[b] = S + b * rr;
        C[b] = d->T1.p + b * size_t(kpmax) * r * W;
      }
      gemm_batched(d, CUBLAS_OP_N, CUBLAS_OP_N, kpmax, r, r, A, kpmax, B, r, C, kpmax);
      for (int b = 0; b < nbc; ++b) {  // out = T1 P_s^T
        A[b] = d->T1.p + b * size_t(kpmax) * r * W;
        B[b] = d->P.p + bcol[b0 + b] * pr;
        C[b] = d->out.p + b * oo;
      }
      gemm_batched(d, CUBLAS_OP_N, CUBLAS_OP_T, kpmax, kpmax, r, A, kpmax, B, kpmax, C, kpmax);
      res = d->out.p;
    }
    d->host_out.resize(oo * nbc);
    ck(cudaMemcpy(d->host_out.data(), res, sizeof(double) * oo * nbc, cudaMemcpyDeviceToHost), "out down");
    const int ld = P ? kpmax : r;
    for (int b = 0; b < nbc; ++b) {
      const int t = brow[b0 + b], u = bcol[b0 + b];
      const int mr = P ? kp[t] : d->r[t], mc = P ? kp[u] : d->r[u];
      double* o = dst[b0 + b];
      const double* src = d->host_out.data() + b * oo;
      for (int c = 0; c < mc; ++c)
        std::memcpy(o + size_t(c) * mr * W, src + size_t(c) * ld * W, sizeof(double) * mr * W);
    }
  }
}

}  // namespace h2b
