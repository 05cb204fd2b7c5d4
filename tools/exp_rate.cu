// Microbenchmark: cycles per softmax exponential block as the FA kernels run
// it (FFMA2 scale, ex2 on MUFU or the FMA-pipe polynomial for EMU of every 8
// pairs, FADD2 row sum, F2FP bf16 pack), 128 scores per thread, with W warps
// per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/exp_rate.cu -o /tmp/er
#include <cstdio>
#include "../paper_2605_10905_b200/csrc/softmax.cuh"
using namespace mimw;

// variants of the FMA-pipe exp2: V 0 = softmax.cuh's ex2_poly2; 1 = the 2^n
// fold as shift + add (ALU) instead of IMAD (FMA pipe); 2 = degree-2
// polynomial; 3 = both
template <int V>
__device__ __forceinline__ uint64_t ex2_poly_v(uint64_t x2) {
  if (V == 0) return ex2_poly2(x2);
  float a, b;
  f2_unpack(x2, a, b);
  a = fmaxf(a, -126.f);
  b = fmaxf(b, -126.f);
  const uint64_t x = f2_pack(a, b);
  const uint64_t t = f2_add(x, f2_pack(12582912.f, 12582912.f));
  const uint64_t r = f2_add(t, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = f2_fma(r, f2_pack(-1.f, -1.f), x);
  uint64_t q;
  if (V >= 2) {  // degree 2 minimax on [-0.5, 0.5]
    q = f2_fma(f2_pack(0.2402265f, 0.2402265f), f, f2_pack(0.6931472f, 0.6931472f));
    q = f2_fma(q, f, f2_pack(1.0f, 1.0f));
  } else {
    q = f2_fma(f2_pack(0.0551824f, 0.0551824f), f, f2_pack(0.24261211f, 0.24261211f));
    q = f2_fma(q, f, f2_pack(0.693259f, 0.693259f));
    q = f2_fma(q, f, f2_pack(0.99992794f, 0.99992794f));
  }
  float t0, t1, q0, q1;
  f2_unpack(t, t0, t1);
  f2_unpack(q, q0, q1);
  uint32_t y0, y1;
  if (V & 1) {
    asm("{\n\t.reg .b32 s;\n\tbfi.b32 s, %1, 0, 23, 9;\n\tadd.u32 %0, s, %2;\n\t}" : "=r"(y0) : "r"(__float_as_uint(t0)), "r"(__float_as_uint(q0)));
    asm("{\n\t.reg .b32 s;\n\tbfi.b32 s, %1, 0, 23, 9;\n\tadd.u32 %0, s, %2;\n\t}" : "=r"(y1) : "r"(__float_as_uint(t1)), "r"(__float_as_uint(q1)));
  } else {
    y0 = (__float_as_uint(t0) << 23) + __float_as_uint(q0);
    y1 = (__float_as_uint(t1) << 23) + __float_as_uint(q1);
  }
  return f2_pack(__uint_as_float(y0), __uint_as_float(y1));
}

template <int EMU, int N, int V = 0>
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
      const uint64_t p2 = ((e & 7) < EMU) ? ex2_poly_v<V>(x2) : ex2_mufu2(x2);
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

template <int EMU, int N, int V = 0>
void run(int warps_per_smsp, float *o, long long *c) {
  const int iters = 2000;
  k<EMU, N, V><<<148, 128 * warps_per_smsp>>>(o, c, iters, 0.37f);
  cudaDeviceSynchronize();
  long long h[148 * 16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double sum = 0;
  int n = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < 4 * warps_per_smsp; ++w) { sum += h[b * 16 + w]; ++n; }
  const double per = sum / n / iters;
  printf("V %d EMU %d  N %3d  warps/SMSP %d: %7.1f cycles per block of %d scores per warp  (%.2f per score; MUFU floor %d)\n",
         V, EMU, N, warps_per_smsp, per, N, per / N, (N - N * EMU / 8) * 8 * warps_per_smsp / warps_per_smsp);
}

int main() {
  float *o; long long *c;
  cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 148 * 16 * 8);
  for (int w : {1, 2, 3}) {
    run<0, 128>(w, o, c); run<1, 128>(w, o, c); run<2, 128>(w, o, c); run<3, 128>(w, o, c);
    run<0, 64>(w, o, c); run<2, 64>(w, o, c); run<3, 64>(w, o, c);
  }
  for (int w : {4}) {
    run<0, 64>(w, o, c); run<2, 64>(w, o, c); run<3, 64>(w, o, c);
    run<0, 128>(w, o, c); run<3, 128>(w, o, c);
  }
  for (int w : {2, 3})
    for (int dummy = 0; dummy < 1; ++dummy) {
      run<2, 128, 1>(w, o, c); run<3, 128, 1>(w, o, c); run<4, 128, 1>(w, o, c);
      run<2, 128, 2>(w, o, c); run<3, 128, 2>(w, o, c); run<4, 128, 2>(w, o, c);
      run<2, 128, 3>(w, o, c); run<3, 128, 3>(w, o, c); run<4, 128, 3>(w, o, c);
    }
  return 0;
}
