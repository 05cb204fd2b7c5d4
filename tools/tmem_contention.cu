// Microbenchmark: tcgen05.mma throughput while other warps read TMEM with
// tcgen05.ld at a controlled rate (the FA softmax warps' S loads).
// Thread 0 issues TS M128 N128 MMAs (B MN-major, as FA's P.V) back to back;
// warps 1..NW read 32 columns x 32 lanes per tcgen05.ld, pausing DELAY cycles
// between loads.  Reports cycles per MMA and the achieved LDTM bytes/clk/SM.
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

template <int SHAPE>  // 0: ld 32x32b.x32, 1: ld 4 x 32x32b.x32, 2: st 32x32b.x16 (P stores)
__global__ void __launch_bounds__(256, 1) k(long long *out, int iters, int delay, int nw) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  __shared__ unsigned long long loads;
  const int warp = threadIdx.x / 32;
  uint32_t sb = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); done = 0; loads = 0; }
  if (warp == 0) tmem_alloc<1>(smem_u32(&slot), 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (warp >= 1 && warp <= nw) {
    const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + 128;
    unsigned long long n = 0;
    uint32_t x = 0;
    while (!done) {
      if (SHAPE == 0) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(base + (n & 3) * 32, r);
        tmem_ld_wait();
        x += r[0] + r[31];
        n += 4096;
      } else if (SHAPE == 1) {
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(base + c * 32, r);
        tmem_ld_wait();
        x += r[0] + r[31];
        n += 16384;
      } else {
        uint32_t r[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) r[c] = x + c;
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st_32x32b_x16(base + 64 + c * 16, r);
        tmem_st_wait();
        x += 1;
        n += 8192;
      }
      if (delay) { long long t = clock64(); while (clock64() - t < delay) {} }
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(&loads, n);
    if (x == 12345) out[1000] = x;
  }
  long long cyc = 0;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, 128, 0, 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t b = smem_desc_sw128(sb + (i & 7) * 2048, 16384, 1024);
      mma_f16_ts<1>(tm + 256, tm + (i & 7) * 8, b, id, 1);
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    cyc = clock64() - t0;
    done = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = cyc; out[2 * blockIdx.x + 1] = loads; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tm, 512); }
}

int main() {
  long long *d; cudaMalloc(&d, 148 * 16 + 8192);
  long long h[296];
  const int iters = 8192;
  for (int shape = 0; shape < 3; ++shape)
    for (int nw : {1, 3, 7})
      for (int delay : {0, 200, 800, 2000}) {
        auto kern = shape == 0 ? k<0> : shape == 1 ? k<1> : k<2>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
        kern<<<148, 256, 40000>>>(d, iters, delay, nw);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = 0, ld = 0;
        for (int i = 0; i < 148; ++i) { cyc += h[2 * i]; ld += h[2 * i + 1]; }
        cyc /= 148; ld /= 148;
        printf("%s nw %d delay %4d: %.1f cycles/MMA, TMEM ld/st %.1f B/clk/SM %s\n",
               shape == 0 ? "ld x32 " : shape == 1 ? "ld x128" : "st x16 ", nw,
               delay, cyc / iters, ld / cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
