// Eigensolver options for the upper-level Gram matrices (dimension 2 x child
// rank, few matrices per level): cuSOLVER batched syev vs per-matrix syevd /
// syevdx / syevj, on PSD test matrices with the Grams' decaying spectrum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/eig_bench.cu -lcusolver -lcublas -o /tmp/eig_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <thread>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)
#define CS(x) do { cusolverStatus_t s_ = (x); if (s_ != CUSOLVER_STATUS_SUCCESS) { printf("cusolver %d line %d\n", int(s_), __LINE__); exit(1); } } while (0)

// G = Q diag(lam) Q^T with lam_i = 10^(-20 i / n) (half the spectrum below 1e-10)
static void make_psd(std::vector<double>& G, int n, int seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd;
  std::vector<double> Q(size_t(n) * n);
  for (auto& x : Q) x = nd(rng);
  // Gram-Schmidt (twice) for an orthonormal Q
  for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j < n; ++j) {
      double* qj = &Q[size_t(j) * n];
      for (int i = 0; i < j; ++i) {
        const double* qi = &Q[size_t(i) * n];
        double d = 0;
        for (int k = 0; k < n; ++k) d += qi[k] * qj[k];
        for (int k = 0; k < n; ++k) qj[k] -= d * qi[k];
      }
      double nr = 0;
      for (int k = 0; k < n; ++k) nr += qj[k] * qj[k];
      nr = std::sqrt(nr);
      for (int k = 0; k < n; ++k) qj[k] /= nr;
    }
  G.assign(size_t(n) * n, 0.0);
  for (int l = 0; l < n; ++l) {
    const double lam = std::pow(10.0, -20.0 * l / n);
    const double* q = &Q[size_t(l) * n];
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r) G[r + size_t(c) * n] += lam * q[r] * q[c];
  }
}

int main(int argc, char** argv) {
  struct Lv { int n, count; };
  std::vector<Lv> lv = {{390, 2}, {450, 4}, {556, 8}, {610, 16}, {566, 32}, {504, 64}, {406, 128}, {256, 256}, {128, 512}};
  if (argc > 1) lv = {{atoi(argv[1]), atoi(argv[2])}};
  cusolverDnHandle_t h;
  CS(cusolverDnCreate(&h));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CS(cusolverDnSetStream(h, st));
  cusolverDnParams_t prm;
  CS(cusolverDnCreateParams(&prm));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (const Lv& L : lv) {
    const int n = L.n, count = L.count;
    std::vector<double> one, all(size_t(n) * n * count);
    for (int b = 0; b < std::min(count, 4); ++b) {
      make_psd(one, n, 7 + b);
      std::copy(one.begin(), one.end(), all.begin() + size_t(b) * n * n);
    }
    for (int b = 4; b < count; ++b) std::copy(all.begin() + size_t(b % 4) * n * n, all.begin() + size_t(b % 4 + 1) * n * n, all.begin() + size_t(b) * n * n);
    double *G, *A, *w;
    int* info;
    CK(cudaMalloc(&G, all.size() * 8));
    CK(cudaMalloc(&A, all.size() * 8));
    CK(cudaMalloc(&w, size_t(n) * count * 8));
    CK(cudaMalloc(&info, count * 4));
    CK(cudaMemcpy(G, all.data(), all.size() * 8, cudaMemcpyHostToDevice));
    auto timeit = [&](const char* name, auto&& fn) {
      CK(cudaMemcpyAsync(A, G, all.size() * 8, cudaMemcpyDeviceToDevice, st));
      fn();  // warm
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpyAsync(A, G, all.size() * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      fn();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      // check: largest eigenvalue ~ 1
      std::vector<double> hw(size_t(n) * count);
      CK(cudaMemcpy(hw.data(), w, hw.size() * 8, cudaMemcpyDeviceToHost));
      double mx = 0;
      for (int i = 0; i < n; ++i) mx = std::max(mx, hw[i]);
      printf("n=%4d count=%4d  %-22s %9.3f ms  (%.3f ms/matrix)  lam_max %.6f\n", n, count, name, ms, ms / count, mx);
    };
    {  // batched syev
      size_t db = 0, hb = 0;
      CS(cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                           CUDA_R_64F, w, CUDA_R_64F, &db, &hb, count));
      void* dw;
      CK(cudaMalloc(&dw, db + 16));
      std::vector<char> hw(hb + 1);
      timeit("XsyevBatched", [&] {
        CS(cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                  CUDA_R_64F, w, CUDA_R_64F, dw, db, hw.data(), hb, info, count));
      });
      CK(cudaFree(dw));
    }
    {  // per-matrix syevd
      size_t db = 0, hb = 0;
      CS(cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                     CUDA_R_64F, w, CUDA_R_64F, &db, &hb));
      void* dw;
      CK(cudaMalloc(&dw, db + 16));
      std::vector<char> hw(hb + 1);
      timeit("Xsyevd loop", [&] {
        for (int b = 0; b < count; ++b)
          CS(cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A + size_t(b) * n * n,
                              n, CUDA_R_64F, w + size_t(b) * n, CUDA_R_64F, dw, db, hw.data(), hb, info + b));
      });
      CK(cudaFree(dw));
    }
    {  // per-matrix syevdx: eigenpairs with lambda > 1e-12 (superset of the kept ones)
      size_t db = 0, hb = 0;
      int64_t found = 0;
      double vl = 1e-12, vu = 1e300;
      CS(cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_V, CUBLAS_FILL_MODE_LOWER, n,
                                      CUDA_R_64F, A, n, &vl, &vu, 0, 0, &found, CUDA_R_64F, w, CUDA_R_64F, &db, &hb));
      void* dw;
      CK(cudaMalloc(&dw, db + 16));
      std::vector<char> hw(hb + 1);
      timeit("Xsyevdx loop (>1e-12)", [&] {
        for (int b = 0; b < count; ++b)
          CS(cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_V, CUBLAS_FILL_MODE_LOWER, n,
                               CUDA_R_64F, A + size_t(b) * n * n, n, &vl, &vu, 0, 0, &found, CUDA_R_64F,
                               w + size_t(b) * n, CUDA_R_64F, dw, db, hw.data(), hb, info + b));
      });
      printf("    syevdx found %lld\n", (long long)found);
      CK(cudaFree(dw));
    }
    if (n <= 640) {  // per-matrix syevj (Jacobi)
      syevjInfo_t sj;
      CS(cusolverDnCreateSyevjInfo(&sj));
      CS(cusolverDnXsyevjSetTolerance(sj, 1e-14));
      CS(cusolverDnXsyevjSetMaxSweeps(sj, 30));
      int lw = 0;
      CS(cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, w, &lw, sj));
      double* dw;
      CK(cudaMalloc(&dw, size_t(lw) * 8 + 16));
      timeit("Dsyevj loop", [&] {
        for (int b = 0; b < count; ++b)
          CS(cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A + size_t(b) * n * n, n,
                              w + size_t(b) * n, dw, lw, info + b, sj));
      });
      CK(cudaFree(dw));
      CS(cusolverDnDestroySyevjInfo(sj));
    }
    {  // syevd on 4 host threads, each with its own handle + stream
      const int T = std::min(count, 4);
      std::vector<cusolverDnHandle_t> hs(T);
      std::vector<cudaStream_t> ss(T);
      std::vector<void*> dws(T);
      size_t db = 0, hb = 0;
      CS(cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                     CUDA_R_64F, w, CUDA_R_64F, &db, &hb));
      for (int i = 0; i < T; ++i) {
        CS(cusolverDnCreate(&hs[i]));
        CK(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
        CS(cusolverDnSetStream(hs[i], ss[i]));
        CK(cudaMalloc(&dws[i], db + 16));
      }
      CK(cudaMemcpy(A, G, all.size() * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int i = 0; i < T; ++i)
        th.emplace_back([&, i] {
          std::vector<char> hw(hb + 1);
          cusolverDnParams_t p2;
          cusolverDnCreateParams(&p2);
          for (int b = i; b < count; b += T)
            CS(cusolverDnXsyevd(hs[i], p2, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F,
                                A + size_t(b) * n * n, n, CUDA_R_64F, w + size_t(b) * n, CUDA_R_64F, dws[i], db,
                                hw.data(), hb, info + b));
          cudaStreamSynchronize(ss[i]);
          cusolverDnDestroyParams(p2);
        });
      for (auto& x : th) x.join();
      auto t1 = std::chrono::steady_clock::now();
      const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      printf("n=%4d count=%4d  %-22s %9.3f ms  (%.3f ms/matrix)  [wall]\n", n, count, "Xsyevd 4 threads", ms, ms / count);
      for (int i = 0; i < T; ++i) {
        cusolverDnDestroy(hs[i]);
        cudaStreamDestroy(ss[i]);
        cudaFree(dws[i]);
      }
    }
    CK(cudaFree(G));
    CK(cudaFree(A));
    CK(cudaFree(w));
    CK(cudaFree(info));
  }
  return 0;
}
