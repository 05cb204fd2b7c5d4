// Internal launcher interface for the warp-specialized flash-attention forward.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct AttnArgs {
  const void *q, *k, *v;  // [batch, heads, seq, 128] bf16, contiguous
  void *o;                // [batch, heads, seq, 128] bf16
  float *lse;             // [batch, heads, seq] fp32 (natural log) or null
  int64_t batch, heads, seq;
  int64_t window;         // keys j in [i - window + 1, i]; >= seq plain causal; <= 0 non-causal
  double scale;
  int max_ctas;           // 0 = one persistent CTA per SM
  unsigned long long *trace = nullptr;  // optional [grid][12 warps][8] cycle counters
  int emu = -1;           // exp2 pairs of 8 on the FMA pipe (-1 = default)
  int cta_group = 1;      // 1: one-CTA kernel (two Q tiles per SM); 2: the 2-CTA kernel (attention_fwd_cg2.cuh)
};

cudaError_t attention_fwd_launch(const AttnArgs &a, cudaStream_t stream);

}  // namespace mimw
