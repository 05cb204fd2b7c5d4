// Microbenchmark: does a warp issuing tcgen05.mma get starved of issue slots
// by busy ALU/MUFU warps on the same SM sub-partition (SMSP = warp % 4)?
// Warp 0 lane 0 issues TS M128 N128 MMAs; background warps run FFMA2 + MUFU
// loops.  mode 0: no background; 1: background on SMSPs 1..3 only (warps 1,2,3,5,6,7);
// 2: background on all SMSPs incl. SMSP 0 (warps 4, 8 share with the MMA warp).
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

__global__ void __launch_bounds__(384, 1) k(long long *out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  uint32_t sb = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); done = 0; }
  if (warp == 0) tmem_alloc<1>(smem_u32(&slot), 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  const bool bg = warp != 0 && ((mode == 1 && (warp % 4) != 0) || mode == 2);
  if (bg) {
    float x = threadIdx.x * 1e-3f, y = 0.5f;
    while (!done) {
#pragma unroll 16
      for (int i = 0; i < 64; ++i) {
        x = fmaf(x, 0.999f, 0.001f);
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
        y += e;
      }
    }
    if (y == 1.2345f) out[1000] = 1;
  }
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, 128, 0, 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t b = smem_desc_sw128(sb + (i & 7) * 2048, 16384, 1024);
      mma_f16_ts<1>(tm + 256, tm + (i & 7) * 8, b, id, 1);
    }
    long long t1 = clock64();
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = clock64() - t0;
    done = 1;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tm, 512); }
}

int main() {
  long long *d; cudaMalloc(&d, 148 * 16 + 8192);
  long long h[296];
  const int iters = 4096;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int mode = 0; mode < 3; ++mode) {
    k<<<148, 384, 40000>>>(d, iters, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double is = 0, tot = 0;
    for (int i = 0; i < 148; ++i) { is += h[2 * i]; tot += h[2 * i + 1]; }
    printf("mode %d: issue %.1f cycles/MMA, complete %.1f cycles/MMA %s\n", mode, is / 148 / iters,
           tot / 148 / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
