// Packed fp32x2 softmax arithmetic shared by the attention kernels
// (FFMA2 / FADD2 on sm_100a, MUFU ex2, an FMA-pipe exp2 polynomial).
#pragma once
#include "ptx.cuh"

namespace mimw {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ uint64_t ex2_mufu2(uint64_t x2) {
  float a, b;
  f2_unpack(x2, a, b);
  return f2_pack(ex2(a), ex2(b));
}

// exp2 on the FMA pipe (offloads the MUFU, the FA-forward co-bottleneck):
// x = n + f, n = rint(x) via the 1.5*2^23 magic, f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. err 7.5e-5, far below the
// bf16 rounding of P); 2^n folded into the exponent bits.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float a, b;
  f2_unpack(x2, a, b);
  a = fmaxf(a, -126.f);  // 2^-126 keeps the exponent field >= 0 (no wrap to NaN)
  b = fmaxf(b, -126.f);
  const uint64_t x = f2_pack(a, b);
  const uint64_t t = f2_add(x, f2_pack(12582912.f, 12582912.f));
  const uint64_t r = f2_add(t, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = f2_fma(r, f2_pack(-1.f, -1.f), x);
  uint64_t q = f2_fma(f2_pack(0.0551824f, 0.0551824f), f, f2_pack(0.24261211f, 0.24261211f));
  q = f2_fma(q, f, f2_pack(0.693259f, 0.693259f));
  q = f2_fma(q, f, f2_pack(0.99992794f, 0.99992794f));
  float t0, t1, q0, q1;
  f2_unpack(t, t0, t1);
  f2_unpack(q, q0, q1);
  const float y0 = __int_as_float((__float_as_int(t0) << 23) + __float_as_int(q0));
  const float y1 = __int_as_float((__float_as_int(t1) << 23) + __float_as_int(q1));
  return f2_pack(y0, y1);
}

__device__ __forceinline__ uint32_t pack_bf16_2(uint64_t v) {
  float a, b;
  f2_unpack(v, a, b);
  return pack_bf16(a, b);
}

}  // namespace mimw
