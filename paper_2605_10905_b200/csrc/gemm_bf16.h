// Internal launcher interface for the persistent warp-specialized bf16 GEMM.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct GemmArgs {
  const void *a;   // [m, k] bf16, row stride lda (elements)
  const void *b;   // b_kn ? [k, n] (row stride ldb) : [n, k] (row stride ldb), bf16
  void *c;         // [m, n], row stride ldc; f32 when c_f32 else bf16
  int64_t m, n, k, lda, ldb, ldc;
  bool b_kn;       // B given as [K, N] row-major (the reference's layout, oracles.cpp:21-22)
  bool c_f32;
  int cta_group;   // 2 (default, CTA pair) or 1
  int raster_group;  // tile-row group for L2-friendly rasterisation (0 = default 8)
  int max_clusters;  // 0 = one cluster per SM pair
};

cudaError_t gemm_bf16_launch(const GemmArgs &g, cudaStream_t stream);

}  // namespace mimw
