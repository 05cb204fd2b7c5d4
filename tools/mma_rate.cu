// Microbenchmark: tcgen05.mma issue->completion rate for the FA shapes.
// One CTA per SM, one thread issues `iters` MMAs of a given kind into TMEM and
// waits on the commit barrier; reports cycles per MMA (K=16).
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

// 4: TS M128 N128 with MN-major B (FA's P.V: V [keys, d] row-major, two 64-col panels)
// 5: SS M128 N128 with MN-major B
// 6/7: latency of one 8-MMA group (SS / TS-MN) issued from an idle pipe, commit+wait each time
template <int MODE>  // 0: SS M128 N128, 1: TS M128 N128, 2: SS M128 N256, 3: SS M128 N64
__global__ void __launch_bounds__(128, 1) k(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  uint32_t sb = smem_u32(sm);
  sb = (sb + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<1>(smem_u32(&slot), 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (MODE >= 8 && warp >= 1) {
    // background TMEM readers (like the softmax warps' tcgen05.ld of S):
    // warps 1..3 read columns [128, 256) of their lane quarter until the MMAs finish
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tm + ((uint32_t)(warp * 32) << 16) + 128 + ((acc & 3) * 32), r);
      tmem_ld_wait();
      acc += r[0] & 1;
      if (MODE == 10) tmem_st_32x32b_x16(tm + ((uint32_t)(warp * 32) << 16) + 64, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
    }
    if (acc == 12345) out[1000] = acc;
  }
  if (threadIdx.x == 0) {
    constexpr int N = MODE == 2 ? 256 : ((MODE == 3 || MODE == 11 || MODE == 12) ? 64 : 128);
    constexpr bool BMN = MODE == 4 || MODE == 5 || MODE == 7 || MODE == 8 || MODE == 10;
    const uint32_t id = idesc_bf16(128, N, 0, BMN ? 1 : 0);
    long long t0 = clock64();
    if (MODE >= 6) {
      uint32_t ph = 0;
      for (int g = 0; g < iters / 8; ++g) {
        for (int i = 0; i < 8; ++i) {
          const uint64_t a = smem_desc_sw128(sb + (i & 3) * 32, 16, 1024);
          const uint64_t b = BMN ? smem_desc_sw128(sb + 32768 + i * 2048, 16384, 1024)
                                 : smem_desc_sw128(sb + 32768 + (i & 3) * 32, 16, 1024);
          if (MODE == 7) mma_f16_ts<1>(tm + 256, tm + (i & 7) * 8, b, id, 1);
          else mma_f16_ss<1>(tm, a, b, id, 1);
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), ph);
        ph ^= 1;
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        const uint64_t a = smem_desc_sw128(sb + (i & 3) * 32, 16, 1024);
        const uint64_t b = BMN ? smem_desc_sw128(sb + 32768 + (i & 7) * 2048, 16384, 1024)
                               : smem_desc_sw128(sb + 32768 + (i & 3) * 32, 16, 1024);
        if (MODE == 1 || MODE == 4 || MODE == 8 || MODE == 10) mma_f16_ts<1>(tm + 256, tm + (i & 7) * 8, b, id, 1);
        else if (MODE == 11) mma_f16_ss<1>(tm + (i & 1) * 64, a, b, id, 1);     // two independent N64 chains
        else if (MODE == 12) mma_f16_ss<1>(tm + (i & 3) * 64, a, b, id, 1);     // four independent N64 chains
        else mma_f16_ss<1>(tm, a, b, id, 1);
      }
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
    }
    out[blockIdx.x] = clock64() - t0;
    done = 1;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tm, 512); }
}

int main() {
  long long *d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int iters = 4096;
  auto run = [&](auto kern, const char *name, int n) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
    kern<<<148, 128, 120000>>>(d, iters);
    kern<<<148, 128, 120000>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("%-22s %s cycles/MMA %.1f  (ideal %d)\n", name, cudaGetErrorString(e), avg / iters, n);
  };
  run(k<0>, "SS M128 N128 K16", 64);
  run(k<1>, "TS M128 N128 K16", 64);
  run(k<2>, "SS M128 N256 K16", 128);
  run(k<3>, "SS M128 N64 K16", 32);
  run(k<4>, "TS M128 N128 B-MN", 64);
  run(k<5>, "SS M128 N128 B-MN", 64);
  run(k<6>, "SS group-of-8 from idle", 64);
  run(k<7>, "TS-MN group-of-8 idle", 64);
  run(k<8>, "TS-MN + 3 warps LDTM", 64);
  run(k<9>, "SS + 3 warps LDTM", 64);
  run(k<10>, "TS-MN + LDTM+STTM", 64);
  run(k<11>, "SS N64 x2 chains", 32);
  run(k<12>, "SS N64 x4 chains", 32);
  return 0;
}
