// Internal launcher interface for the block-scaled FP8 (MXFP8) GEMM.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>

namespace mimw {

struct Mxfp8Args {
  const void *a;    // e4m3 [m, k], row stride lda bytes (K-major)
  const void *sfa;  // ue8m0 [m, k/32]
  const void *b;    // e4m3 [n, k], row stride ldb bytes (K-major, "NT")
  const void *sfb;  // ue8m0 [n, k/32]
  void *c;          // bf16 [m, n], row stride ldc
  int64_t m, n, k, lda, ldb, ldc;
  void *workspace;  // gemm_mxfp8_workspace(m, n, k) bytes (scale-factor atoms)
  int cta_group;    // 2 (default, CTA pair M=256) or 1
};

size_t gemm_mxfp8_workspace(int64_t m, int64_t n, int64_t k);
cudaError_t gemm_mxfp8_launch(const Mxfp8Args &g, cudaStream_t stream);

}  // namespace mimw
