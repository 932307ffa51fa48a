// Probe: a green context with a subset of SMs, its stream driven from the
// runtime API (<<<>>>, cudaMallocAsync, events) — which SMs do its blocks run on?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a tools/green_ctx_probe.cu -lcuda -o /tmp/gprobe
#include <cstdio>
#include <set>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* m; cuGetErrorString(r_, &m); printf("CU %s line %d\n", m, __LINE__); return 1; } } while (0)
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void where(int* out, long long spin) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sm;
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  for (unsigned want : {16u, 100u, 120u, 132u}) {
    CUdevResource grp, rem;
    unsigned nb = 1;
    CU(cuDevSmResourceSplitByCount(&grp, &nb, &all, &rem, 0, want));
    CUdevResourceDesc desc;
    CU(cuDevResourceGenerateDesc(&desc, &grp, 1));
    CUgreenCtx g;
    CU(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream cs;
    CU(cuGreenCtxStreamCreate(&cs, g, CU_STREAM_NON_BLOCKING, 0));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cs);
    const int blocks = 4 * 148;
    int* d;
    CK(cudaMallocAsync(&d, blocks * sizeof(int), st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    where<<<blocks, 128, 0, st>>>(d, 200000);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    std::vector<int> h(blocks);
    CK(cudaMemcpyAsync(h.data(), d, blocks * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::set<int> sms(h.begin(), h.end());
    printf("want %u -> group %u SMs (remaining %u): blocks ran on %zu distinct SMs, %.3f ms\n", want, grp.sm.smCount,
           rem.sm.smCount, sms.size(), ms);
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
    CU(cuStreamDestroy(cs));
    CU(cuGreenCtxDestroy(g));
  }
  // reference: the same kernel on a normal stream
  int* d;
  CK(cudaMalloc(&d, 4 * 148 * sizeof(int)));
  where<<<4 * 148, 128>>>(d, 200000);
  std::vector<int> h(4 * 148);
  CK(cudaMemcpy(h.data(), d, h.size() * sizeof(int), cudaMemcpyDeviceToHost));
  printf("primary context: %zu distinct SMs\n", std::set<int>(h.begin(), h.end()).size());
  return 0;
}
