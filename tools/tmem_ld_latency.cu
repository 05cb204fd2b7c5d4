// Microbenchmark: latency of one softmax-style S load (4 x tcgen05.ld
// 32x32b.x32 + wait, 16 KiB per warp) by a full warpgroup (4 warps, one per
// TMEM lane quarter), with the tensor pipe idle vs running back-to-back TS
// M128 N128 MMAs (FA's O += P.V) or SS MMAs (FA's S = Q.K^T).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tmem_ld_latency.cu -o /tmp/tld -lcuda
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

__global__ void __launch_bounds__(160, 1) k(long long *out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  __shared__ unsigned long long acc_cyc, acc_n;
  const int warp = threadIdx.x / 32;
  uint32_t sb = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); done = 0; acc_cyc = 0; acc_n = 0; }
  if (warp == 0) tmem_alloc<1>(smem_u32(&slot), 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (warp >= 1) {
    const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16);  // S at columns [0,128)
    unsigned long long cyc = 0, n = 0;
    uint32_t x = 0;
    for (int it = 0; it < 400 && (mode == 0 || !done); ++it) {
      uint32_t r[128];
      const long long t0 = clock64();
      tmem_ld_32x32b_x32(base + 0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld_32x32b_x32(base + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld_32x32b_x32(base + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[64]));
      tmem_ld_32x32b_x32(base + 96, *reinterpret_cast<uint32_t(*)[32]>(&r[96]));
      tmem_ld_wait();
      const long long t1 = clock64();
#pragma unroll
      for (int c = 0; c < 128; c += 8) x += r[c];
      cyc += t1 - t0; ++n;
      { long long t = clock64(); while (clock64() - t < 300) {} }
    }
    if ((threadIdx.x & 31) == 0) { atomicAdd(&acc_cyc, cyc); atomicAdd(&acc_n, n); }
    if (x == 12345) out[1000] = x;
  }
  if (threadIdx.x == 0 && mode != 0) {
    const uint32_t id = idesc_bf16(128, 128, 0, 1);
    for (int i = 0; i < iters; ++i) {
      const uint64_t b = smem_desc_sw128(sb + (i & 7) * 2048, 16384, 1024);
      if (mode == 1) mma_f16_ts<1>(tm + 256, tm + 128 + (i & 7) * 8, b, id, 1);  // O[256,384) += P[128,192) V
      else mma_f16_ss<1>(tm + 384, b, b, idesc_bf16(128, 128, 0, 0), 1);          // S' [384,512)
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    done = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = acc_cyc; out[2 * blockIdx.x + 1] = acc_n; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tm, 512); }
}

int main() {
  long long *d; cudaMalloc(&d, 148 * 16 + 8192);
  long long h[296];
  const char *names[3] = {"pipe idle        ", "TS MMAs (P.V)    ", "SS MMAs (Q.K^T)  "};
  for (int mode = 0; mode < 3; ++mode) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k<<<148, 160, 40000>>>(d, 200000, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0, n = 0;
    for (int i = 0; i < 148; ++i) { cyc += h[2 * i]; n += h[2 * i + 1]; }
    printf("%s: %.1f cycles per 4 x ld.32x32b.x32 + wait (warpgroup, 64 KiB) %s\n", names[mode], cyc / n,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
