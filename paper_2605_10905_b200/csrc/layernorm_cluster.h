// Internal launcher interface for the cluster-cooperative LayerNorm.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct LayerNormArgs {
  const float *x;   // [rows, n]
  const float *w;   // [n]
  const float *b;   // [n]
  float *y;         // [rows, n]
  float *mean;      // [rows] or null
  float *rstd;      // [rows] or null
  int64_t rows, n;
  double eps;
  int cluster;      // 0 = automatic (CTAs per row)
};

cudaError_t layernorm_cluster_launch(const LayerNormArgs &a, cudaStream_t stream);

}  // namespace mimw
