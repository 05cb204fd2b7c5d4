// Microbenchmark: cycles per softmax exponential block as the FA kernels run
// it (FFMA2 scale, ex2 on MUFU or the FMA-pipe polynomial for EMU of every 8
// pairs, FADD2 row sum, F2FP bf16 pack), 128 scores per thread, with W warps
// per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/exp_rate.cu -o /tmp/er
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/softmax.cuh"
using namespace mimw;

template <int EMU, int N>
__global__ void __launch_bounds__(512, 1) k(float *out, long long *cyc, int iters, float seed) {
  uint32_t s[N];
#pragma unroll
  for (int c = 0; c < N; ++c) s[c] = __float_as_uint(seed * (float)((threadIdx.x * 7 + c * 13) % 97) - 3.f);
  float l = 0.f;
  uint32_t keep = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float nm = -0.25f * (float)(it & 3);
    const uint64_t sl2 = f2_pack(0.18f, 0.18f), nm2 = f2_pack(nm, nm);
    uint64_t acc[4] = {0, 0, 0, 0};
    uint32_t pk[N / 2];
#pragma unroll
    for (int e = 0; e < N / 2; ++e) {
      const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), sl2, nm2);
      const uint64_t p2 = ((e & 7) < EMU) ? ex2_poly2(x2) : ex2_mufu2(x2);
      acc[e & 3] = f2_add(acc[e & 3], p2);
      pk[e] = pack_bf16_2(p2);
    }
    float a0, a1, b0, b1;
    f2_unpack(f2_add(acc[0], acc[1]), a0, a1);
    f2_unpack(f2_add(acc[2], acc[3]), b0, b1);
    l += (a0 + a1) + (b0 + b1);
#pragma unroll
    for (int e = 0; e < N / 2; ++e) keep ^= pk[e];
    // feed back so the loop is not hoisted
    s[it % N] ^= (keep & 1);
  }
  const long long t1 = clock64();
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 16 + threadIdx.x / 32] = t1 - t0;
  if (l == 12345.f || keep == 0xdeadbeef) out[threadIdx.x] = l;
}

template <int EMU, int N>
void run(int warps_per_smsp, float *o, long long *c) {
  const int iters = 2000;
  k<EMU, N><<<148, 128 * warps_per_smsp>>>(o, c, iters, 0.37f);
  cudaDeviceSynchronize();
  long long h[148 * 16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double sum = 0;
  int n = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < 4 * warps_per_smsp; ++w) { sum += h[b * 16 + w]; ++n; }
  const double per = sum / n / iters;
  printf("EMU %d  N %3d  warps/SMSP %d: %7.1f cycles per block of %d scores per warp  (%.2f per score; MUFU floor %d)\n",
         EMU, N, warps_per_smsp, per, N, per / N, (N - N * EMU / 8) * 8 * warps_per_smsp / warps_per_smsp);
}

int main() {
  float *o; long long *c;
  cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 148 * 16 * 8);
  for (int w : {1, 2, 3}) {
    run<0, 128>(w, o, c); run<1, 128>(w, o, c); run<2, 128>(w, o, c); run<3, 128>(w, o, c);
    run<0, 64>(w, o, c); run<2, 64>(w, o, c); run<3, 64>(w, o, c);
  }
  return 0;
}
