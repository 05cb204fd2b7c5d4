// Internal launcher interface for the warp-specialized flash-attention backward.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct AttnBwdArgs {
  const void *q, *k, *v, *o, *dout;  // [batch, heads, seq, 128] bf16, contiguous
  const float *lse;                  // [batch, heads, seq] fp32 (natural log, from the forward)
  void *dq, *dk, *dv;                // [batch, heads, seq, 128] bf16
  int64_t batch, heads, seq;
  int64_t window;                    // as AttnArgs: >= seq causal, <= 0 non-causal
  double scale;
};

cudaError_t attention_bwd_launch(const AttnBwdArgs &a, cudaStream_t stream);

}  // namespace mimw
