// Internal launcher interface for the 2-simplicial attention forward.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct SimplicialArgs {
  const void *q, *k1, *v1, *k2, *v2;  // [bh, seq, 128] bf16, contiguous
  void *o;                            // [bh, seq, 128] bf16
  float *lse;                         // [bh, seq] fp32 (natural log) or null
  int64_t bh, seq, w1, w2;
  double scale;
};

cudaError_t simplicial_fwd_launch(const SimplicialArgs &a, cudaStream_t stream);

}  // namespace mimw
