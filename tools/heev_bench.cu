// Standalone timing / accuracy check of heev_kernel (csrc/heev.cuh) on batches of
// synthetic Grams shaped like the MMP's (a PSD low-rank part with a graded spectrum
// plus an exact null space, normalised), against cuSOLVER's XsyevBatched.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1908_05218_b200/csrc \
//        tools/heev_bench.cu -o /tmp/heev_bench -lcusolver -lcublas
//   /tmp/heev_bench n count cplx [lib]
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "heev.cuh"

using namespace h2b;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 64;
  const int count = argc > 2 ? std::atoi(argv[2]) : 1024;
  const bool cplx = argc > 3 && std::atoi(argv[3]) != 0;
  const int W = cplx ? 2 : 1;
  const double eps = 1e-8;
  // Grams: G = M M^H with M = Q diag(s) (n x k), k = n/2, s graded 1 .. 1e-12, random Q
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  const int k = n / 2;
  std::vector<double> G(size_t(count) * n * n * W, 0.0);
  const int distinct = std::min(count, 8);
  for (int b = 0; b < distinct; ++b) {
    std::vector<std::complex<double>> M(size_t(n) * k);
    for (int j = 0; j < k; ++j) {
      const double s = std::pow(10.0, -12.0 * j / std::max(1, k - 1));
      for (int i = 0; i < n; ++i) M[i + size_t(j) * n] = s * std::complex<double>(nd(rng), cplx ? nd(rng) : 0.0);
    }
    double nrm = 0;
    std::vector<std::complex<double>> g(size_t(n) * n);
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r) {
        std::complex<double> acc = 0;
        for (int j = 0; j < k; ++j) acc += M[r + size_t(j) * n] * std::conj(M[c + size_t(j) * n]);
        g[r + size_t(c) * n] = acc;
        nrm += std::norm(acc);
      }
    nrm = std::sqrt(nrm);
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r) {
        const std::complex<double> v = g[r + size_t(c) * n] / nrm;
        G[(size_t(b) * n * n + r + size_t(c) * n) * W] = v.real();
        if (cplx) G[(size_t(b) * n * n + r + size_t(c) * n) * W + 1] = v.imag();
      }
  }
  for (int b = distinct; b < count; ++b)
    std::copy(G.begin() + size_t(b % distinct) * n * n * W, G.begin() + size_t(b % distinct + 1) * n * n * W,
              G.begin() + size_t(b) * n * n * W);

  double *dG, *dV, *dZ, *dSlab = nullptr, *dVec, *dVal;
  int *dRank, *dFail;
  uint8_t* dDeg;
  const size_t nn = size_t(count) * n * n;
  CK(cudaMalloc(&dG, nn * W * 8));
  CK(cudaMalloc(&dV, nn * W * 8));
  CK(cudaMalloc(&dZ, nn * 8));
  CK(cudaMalloc(&dVec, nn * W * 8));
  CK(cudaMalloc(&dVal, size_t(count) * n * 8));
  CK(cudaMalloc(&dRank, count * 4));
  CK(cudaMalloc(&dFail, 4));
  CK(cudaMalloc(&dDeg, count));
  CK(cudaMemcpy(dG, G.data(), nn * W * 8, cudaMemcpyHostToDevice));
  constexpr int kMaxSmem = 232448;
  int CS = 0;
  bool smem = true;
  for (int cs : {1, 2, 4, 8, 16})
    if (HeevLayout(n, cs, cplx, true).total * 8 <= kMaxSmem) {
      CS = cs;
      break;
    }
  if (!CS) {
    CS = 16;
    smem = false;
  }
  if (argc > 6) CS = std::atoi(argv[6]);       // forced cluster size
  if (argc > 7) smem = std::atoi(argv[7]) != 0;  // forced slab placement
  const HeevLayout L(n, CS, cplx, smem);
  if (!smem) CK(cudaMalloc(&dSlab, size_t(count) * CS * L.ncl * L.ld * W * 8));
  const int nt = argc > 5 ? std::atoi(argv[5]) : (n <= 64 ? 128 : (n <= 192 ? 256 : 512));
  long long* dProf;
  CK(cudaMalloc(&dProf, 16 * sizeof(long long)));
  CK(cudaMemset(dProf, 0, 16 * sizeof(long long)));
  HeevParams hp{dG, dV, dZ, dSlab, dVec, dVal, dRank, dDeg, dFail, dProf, argc > 8 ? std::atoi(argv[8]) : 0, n, eps};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(count) * CS);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = size_t(L.total) * 8;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  auto launch = [&] {
    CK(cudaMemset(dDeg, 0, count));
    CK(cudaMemset(dFail, 0, 4));
    auto go = [&](auto kern) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cfg.dynamicSmemBytes)));
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CK(cudaLaunchKernelEx(&cfg, kern, hp));
    };
    if (cplx) smem ? go(heev_kernel<true, true>) : go(heev_kernel<true, false>);
    else smem ? go(heev_kernel<false, true>) : go(heev_kernel<false, false>);
  };
  launch();
  CK(cudaDeviceSynchronize());
  {
    long long pr[16];
    CK(cudaMemcpy(pr, dProf, sizeof(pr), cudaMemcpyDeviceToHost));
    std::printf("  block0 cycles: load+tridiag %lld  QL %lld  rank %lld  back %lld  sweeps %lld rotations %lld\n",
                pr[1] - pr[0], pr[2] - pr[1], pr[3] - pr[2], pr[4] - pr[3], pr[5], pr[6]);
    std::printf("  tridiag steps: householder %lld  sync1+v %lld  y %lld  gamma+sync2+gather %lld  rank2 %lld\n",
                pr[8], pr[9], pr[10], pr[11], pr[12]);
  }
  hp.prof = nullptr;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  // accuracy of Gram 0: residual ||G v - lambda v|| and orthogonality of the kept vectors
  std::vector<double> vec(size_t(n) * n * W), val(n);
  int rank = 0, fail = 0;
  CK(cudaMemcpy(vec.data(), dVec, size_t(n) * n * W * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(val.data(), dVal, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&rank, dRank, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&fail, dFail, 4, cudaMemcpyDeviceToHost));
  auto at_ = [&](const std::vector<double>& a, int r, int c) {
    return std::complex<double>(a[(r + size_t(c) * n) * W], cplx ? a[(r + size_t(c) * n) * W + 1] : 0.0);
  };
  double res = 0, orth = 0;
  for (int c = 0; c < rank; ++c) {
    for (int r = 0; r < n; ++r) {
      std::complex<double> acc = 0;
      for (int q = 0; q < n; ++q) acc += at_(G, r, q) * at_(vec, q, c);
      res = std::max(res, std::abs(acc - val[c] * at_(vec, r, c)));
    }
    for (int c2 = 0; c2 <= c; ++c2) {
      std::complex<double> d = 0;
      for (int r = 0; r < n; ++r) d += std::conj(at_(vec, r, c2)) * at_(vec, r, c);
      orth = std::max(orth, std::abs(d - (c == c2 ? 1.0 : 0.0)));
    }
  }
  std::printf("heev n=%d count=%d cplx=%d CS=%d smem=%d threads=%d: %.3f ms (%.1f us/Gram)  rank=%d fail=%d "
              "resid=%.2e orth=%.2e lmax=%.3e\n",
              n, count, int(cplx), CS, int(smem), nt, ms, 1e3 * ms / count, rank, fail, res, orth, val[0]);
  if (argc > 4 && std::atoi(argv[4])) {  // cuSOLVER batched for comparison
    cusolverDnHandle_t h;
    cusolverDnCreate(&h);
    double *dA, *dW, *dWork;
    int* dInfo;
    CK(cudaMalloc(&dA, nn * W * 8));
    CK(cudaMalloc(&dW, size_t(count) * n * 8));
    CK(cudaMalloc(&dInfo, count * 4));
    size_t db = 0, hb = 0;
    const cudaDataType dt = cplx ? CUDA_C_64F : CUDA_R_64F;
    cusolverDnXsyevBatched_bufferSize(h, nullptr, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dt, dA, n,
                                      CUDA_R_64F, dW, dt, &db, &hb, count);
    CK(cudaMalloc(&dWork, db + 16));
    std::vector<char> hw(hb + 1);
    auto lib = [&] {
      CK(cudaMemcpy(dA, dG, nn * W * 8, cudaMemcpyDeviceToDevice));
      cusolverDnXsyevBatched(h, nullptr, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dt, dA, n, CUDA_R_64F,
                             dW, dt, dWork, db, hw.data(), hb, dInfo, count);
    };
    lib();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) lib();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("cusolver XsyevBatched n=%d count=%d cplx=%d: %.3f ms (incl. copy)\n", n, count, int(cplx), ms / reps);
  }
  return 0;
}
