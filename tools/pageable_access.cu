// Probe: can the GPU read pageable host memory directly (HMM / ATS), and how fast?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pma tools/pageable_access.cu && /tmp/pma
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <chrono>
#include <cstring>
__global__ void rd(const float *p, float *o, size_t n) { float s = 0; for (size_t i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += gridDim.x * blockDim.x) s += p[i]; if (s == 123.f) o[0] = s; }
int main() {
  int v = 0, u = 0, h = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0);
  cudaDeviceGetAttribute(&u, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  cudaDeviceGetAttribute(&h, cudaDevAttrHostRegisterSupported, 0);
  printf("pageableMemoryAccess %d usesHostPageTables %d hostRegister %d\n", v, u, h);
  {  // cost of pinning a pageable buffer per call (the alternative to staging through pinned slots)
    size_t bytes = 256u << 20;
    char *p = (char *)malloc(bytes);
    memset(p, 1, bytes);
    auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
    auto t1 = std::chrono::steady_clock::now();
    cudaHostUnregister(p);
    auto t2 = std::chrono::steady_clock::now();
    printf("cudaHostRegister 256 MB: %.2f ms, unregister %.2f ms (%s)\n",
           std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t2 - t1).count(), cudaGetErrorString(e));
    free(p);
  }
  if (v) {
    size_t n = 64 << 20; float *p = (float *)malloc(n * 4); for (size_t i = 0; i < n; ++i) p[i] = 1.f;
    float *o; cudaMalloc(&o, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    rd<<<148 * 4, 256>>>(p, o, n); cudaDeviceSynchronize();
    cudaEventRecord(a); rd<<<148 * 4, 256>>>(p, o, n); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("device read of pageable 256 MB: %.2f ms = %.1f GB/s (%s)\n", ms, n * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
