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
  int cluster_pairs; // 2: clusters of two CTA pairs sharing B by TMA multicast; else 1
};

cudaError_t gemm_bf16_launch(const GemmArgs &g, cudaStream_t stream);

// Grouped (MoE) GEMM: for e < n_groups,
//   y[off_e : off_{e+1}, :] = x[off_e : off_{e+1}, :] . W_e
// with off = m_offsets (HOST array of n_groups + 1 non-decreasing rows),
// x bf16 [off_G, k], w bf16 [G, k, n] (w_kn) or [G, n, k], y bf16 [off_G, n].
struct GroupedGemmArgs {
  const void *x;
  const int64_t *m_offsets;
  const void *w;
  void *y;
  int64_t n_groups, n, k;
  bool w_kn;
  int cta_group;
  int max_clusters;
  bool swap_tails;  // each group's < 256-row tail as a swapped-operand tile (Y^T = W^T X^T)
};

cudaError_t grouped_gemm_bf16_launch(const GroupedGemmArgs &g, cudaStream_t stream);

}  // namespace mimw
