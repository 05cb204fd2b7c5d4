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
  int tile_n;        // C columns per CTA-pair tile: 0 auto, 256, or 512 (bf16 out, cta_group 2)
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
  int swap_tails;   // each group's < 256-row tail as a swapped-operand tile (Y^T = W^T X^T):
                    // 1 yes, 0 padded, -1 default (swapped)
  int tile_n;       // output columns per CTA-pair tile: 0 auto (512 when n >= 512), 256, 512
};

cudaError_t grouped_gemm_bf16_launch(const GroupedGemmArgs &g, cudaStream_t stream);

// K-gathered multi-device GEMM (proj/kernels/multi_device_gemm.mimw,
// oracle_multi_device_gemm oracles.cpp:57-80, generalised to `world` splits):
//   c[rows, n] = sum_s a[s][row0 : row0 + rows, :] . b[s]
// a[s] bf16 [m, k[s]] and b[s] bf16 [k[s], n] are the splits held by device
// s, as pointers valid in this process (local, or peer memory mapped through
// CUDA IPC).  The local split a[rank]/b[rank] is read in place; the others are
// pulled over NVLink by comm CTAs into `ws` while the GEMM runs.  pads[p]:
// device p's signal pad (2 * 8 u32, zeroed once at allocation, IPC-mapped) for
// the entry/exit barrier, with `epoch` strictly increasing per call; all-null
// pads = no device barrier (caller guarantees the peers' inputs are ready and
// stay unchanged until this call completes, e.g. ranks emulated on one GPU).
struct MultiDeviceGemmArgs {
  int rank, world;
  const void *a[8];
  const void *b[8];
  int64_t k[8];
  int64_t n, row0, rows;
  void *c;
  int64_t ldc;
  void *ws;
  size_t ws_bytes;
  uint32_t *pads[8];
  uint32_t epoch;
  int comm_clusters;  // > 0 dedicated comm CTA pairs, < 0 a comm warp in every GEMM CTA, 0 default
  int max_clusters;   // cap on GEMM CTA pairs (0 = all co-resident minus comm)
  int comm_box;       // comm box rows 32 / 64 / 128 of 512-byte rows (0 = 64: 32 KiB boxes)
  int comm_agents;    // copy pipelines per comm CTA, 1..6 (0 = 2)
  int comm_lag;       // stores in flight before a slab signal waits (0 = 8)
};

size_t multi_device_gemm_workspace_bytes(int rank, int world, const int64_t *k, int64_t rows, int64_t n);
cudaError_t multi_device_gemm_launch(const MultiDeviceGemmArgs &g, cudaStream_t stream);

}  // namespace mimw
