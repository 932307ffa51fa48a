// Do DMMA (tensor pipe) and DFMA (fp64 pipe) share throughput on sm_100a?
// Runs DMMA-only, DFMA-only and mixed loops (same warp and split warps).
#include <cstdio>
#include <cuda_runtime.h>

template <int NMMA, int NFMA>
__global__ void mix_loop(double* out, int iters, int split) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  double f[16];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int i = 0; i < 16; ++i) f[i] = i;
  const int warp = threadIdx.x >> 5;
  const bool do_mma = !split || (warp & 1) == 0;
  const bool do_fma = !split || (warp & 1) == 1;
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < NMMA; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i % 8][0]), "+d"(c[i % 8][1]) : "d"(a), "d"(b));
    }
    if (do_fma) {
#pragma unroll
      for (int r = 0; r < NFMA; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(a, f[i], b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NMMA, int NFMA>
void run(const char* name, double* out, int sms, int threads, int split) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 2;
  mix_loop<NMMA, NFMA><<<blocks, threads>>>(out, 10, split);
  cudaEventRecord(e0);
  mix_loop<NMMA, NFMA><<<blocks, threads>>>(out, iters, split);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * threads / 32 / (split ? 2 : 1);
  const double fm = 2.0 * 256 * NMMA * iters * warps, ff = 2.0 * 32 * 16 * NFMA * iters * warps;
  printf("%-28s threads=%4d  dmma %.2f + dfma %.2f = %.2f TFLOP/s (%.3f ms)\n", name, threads, fm / ms / 1e9,
         ff / ms / 1e9, (fm + ff) / ms / 1e9, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 2 * 1024);
  for (int threads : {256, 512}) {
    run<8, 0>("dmma only", out, sms, threads, 0);
    run<0, 1>("dfma only", out, sms, threads, 0);
    run<8, 1>("same warp 8 mma : 16 fma", out, sms, threads, 0);
    run<8, 2>("same warp 8 mma : 32 fma", out, sms, threads, 0);
    run<8, 4>("same warp 8 mma : 64 fma", out, sms, threads, 0);
    run<8, 8>("split warps", out, sms, threads, 1);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
