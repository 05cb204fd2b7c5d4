// Probe: where does tcgen05.mma.kind::mxf8f6f4.block_scale read its UE8M0
// scale factors from in TMEM?  A = B = 1.0 (e4m3), K = 32, so
// D[m][n] = 32 * sfa(m) * sfb(n).  Scale bytes are written with tcgen05.st
// at known (lane, column, byte) positions with codes that identify them;
// decoding D tells which slot the hardware used for each row / column.
//
//   exp 0: SFA byte (L, C, Y) = 1 + L            -> which lane feeds row m
//   exp 1: SFA byte (L, C, Y) = 100 + 4 C + Y     -> which column / byte
//   exp 2/3: same for SFB (per output column n), with SFA = 127 (1.0)
// each for sf_id = 0 and 1, N = 128 and 256.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

__global__ void __launch_bounds__(128, 1) probe(float *out, int exp, int sf_id, int N) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t *a_s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  uint8_t *b_s = a_s + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 128 * 128; i += 128) a_s[i] = 0x38;  // e4m3 1.0
  for (int i = threadIdx.x; i < 256 * 128; i += 128) b_s[i] = 0x38;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<1>(smem_u32(&slot), 512);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  // D at cols [0, 256); SFA at cols [256, 264); SFB at cols [264, 272)
  const uint32_t row = warp * 32 + lane;
  uint32_t va[8], vb[8];
  for (int c = 0; c < 8; ++c) {
    uint32_t wa = 0, wb = 0;
    for (int y = 0; y < 4; ++y) {
      uint32_t ca = 127, cb = 127;
      if (exp == 0) ca = 1 + row;
      if (exp == 1) ca = 100 + 4 * c + y;
      if (exp == 2) cb = 1 + row;
      if (exp == 3) cb = 100 + 4 * c + y;
      wa |= ca << (8 * y);
      wb |= cb << (8 * y);
    }
    va[c] = wa;
    vb[c] = wb;
  }
  tmem_st_32x32b_x8(tm + ((uint32_t)(warp * 32) << 16) + 256, va);
  tmem_st_32x32b_x8(tm + ((uint32_t)(warp * 32) << 16) + 264, vb);
  tmem_st_wait();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t ad = smem_desc_sw128(smem_u32(a_s), 16, 1024);
    const uint64_t bd = smem_desc_sw128(smem_u32(b_s), 16, 1024);
    const uint32_t id = idesc_mxf8(128, N, sf_id, sf_id);
    mma_mxf8_ss<1>(tm, ad, bd, id, tm + 256, tm + 264, 0);
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tm + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int e = 0; e < 32; ++e) out[row * 256 + c + e] = __uint_as_float(r[e]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tm, 512); }
}

int main() {
  float *d;
  cudaMalloc(&d, 128 * 256 * 4);
  static float h[128 * 256];
  for (int N : {128, 256})
    for (int sf_id : {0, 1, 2})
      for (int exp = 0; exp < 4; ++exp) {
        cudaMemset(d, 0, 128 * 256 * 4);
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
        probe<<<1, 128, 60000>>>(d, exp, sf_id, N);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("N=%d sf_id=%d exp=%d: %s\n", N, sf_id, exp, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        // code = log2(D / 32) + 127
        printf("N=%d sf_id=%d exp=%d ", N, sf_id, exp);
        if (exp < 2) {
          printf("rows:");
          for (int m : {0, 1, 31, 32, 33, 63, 64, 96, 127}) {
            float v = h[m * 256 + 0];
            printf(" m%d->%d", m, (int)lrintf(log2f(v / 32.f)) + 127);
          }
        } else {
          printf("cols:");
          for (int n : {0, 1, 31, 32, 64, 127, 128, 129, 160, 255}) {
            if (n >= N) continue;
            float v = h[0 * 256 + n];
            printf(" n%d->%d", n, (int)lrintf(log2f(v / 32.f)) + 127);
          }
        }
        printf("\n");
      }
  return 0;
}
