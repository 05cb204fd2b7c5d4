// Internal launcher of the reference-precision attention (MIMW_PREC_F32).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct AttnF32Args {
  const float *q, *k1, *v1;  // device [seq, d] f32 (attention: k = k1, v = v1)
  const float *k2, *v2;      // simplicial only
  float *o;                  // [seq, d]
  float *lse;                // [seq] or null
  int64_t seq, d;            // d <= 128
  int64_t w1, w2;            // attention: w1 = window; simplicial: both windows
  bool causal;               // attention: false = every key
  bool simplicial;
  double scale;
};

cudaError_t attention_f32_launch(const AttnF32Args &a, cudaStream_t stream);

}  // namespace mimw
