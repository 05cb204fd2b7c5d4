// Operand staging kernels for the host-f32 (reference Tile) entry points:
// f32 -> bf16 (RNE) with zero padding, and the split-bf16 "x3" operands.
//
// bf16x3: x = hi + lo with hi = bf16(x), lo = bf16(x - hi).  Then
//   A.B ~= Ah.Bh + Ah.Bl + Al.Bh = [Ah | Ah | Al] . [Bh ; Bl ; Bh]
// i.e. ONE bf16 tensor-core GEMM with K' = 3K, fp32 accumulate.  The
// dropped Al.Bl term is ~2^-16 relative, so the result meets the
// reference's own f32 tolerance (1e-4, gemm_pipeline.case:5).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "convert.h"

namespace mimw {

namespace {

// dst[r, col_off + c] = part(src[r, c]) for r < rows, c < cols;
// zero for c in [cols, pad_cols).  part: 0 = hi, 1 = lo.
__global__ void stage_bf16_kernel(const float *__restrict__ src, int64_t rows, int64_t cols,
                                  int64_t pad_cols, __nv_bfloat16 *__restrict__ dst, int64_t ld,
                                  int64_t col_off, int part) {
  int64_t n = rows * pad_cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / pad_cols, c = i - r * pad_cols;
    float x = c < cols ? src[r * cols + c] : 0.0f;
    __nv_bfloat16 hi = __float2bfloat16_rn(x);
    __nv_bfloat16 v = part == 0 ? hi : __float2bfloat16_rn(x - __bfloat162float(hi));
    dst[r * ld + col_off + c] = v;
  }
}

// Row-block variant for stacking along K for B[K,N]: rows [0,rows) of src go
// to dst rows [row_off, row_off+rows); rows [rows, pad_rows) are zero.
__global__ void stage_rows_bf16_kernel(const float *__restrict__ src, int64_t rows, int64_t pad_rows,
                                       int64_t cols, int64_t pad_cols, __nv_bfloat16 *__restrict__ dst,
                                       int64_t ld, int64_t row_off, int part) {
  int64_t n = pad_rows * pad_cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / pad_cols, c = i - r * pad_cols;
    float x = (r < rows && c < cols) ? src[r * cols + c] : 0.0f;
    __nv_bfloat16 hi = __float2bfloat16_rn(x);
    __nv_bfloat16 v = part == 0 ? hi : __float2bfloat16_rn(x - __bfloat162float(hi));
    dst[(row_off + r) * ld + c] = v;
  }
}

__global__ void unpad_f32_kernel(const float *__restrict__ src, int64_t ld, float *__restrict__ dst,
                                 int64_t rows, int64_t cols) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i - r * cols;
    dst[i] = src[r * ld + c];
  }
}

__global__ void unpad_bf16_kernel(const __nv_bfloat16 *__restrict__ src, int64_t ld,
                                  float *__restrict__ dst, int64_t rows, int64_t cols) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i - r * cols;
    dst[i] = __bfloat162float(src[r * ld + c]);
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 4096 ? (g > 0 ? g : 1) : 4096);
}

}  // namespace

void stage_cols_bf16(const float *src, int64_t rows, int64_t cols, int64_t pad_cols, void *dst,
                     int64_t ld, int64_t col_off, int part, cudaStream_t s) {
  stage_bf16_kernel<<<grid_for(rows * pad_cols), 256, 0, s>>>(
      src, rows, cols, pad_cols, static_cast<__nv_bfloat16 *>(dst), ld, col_off, part);
}

void stage_rows_bf16(const float *src, int64_t rows, int64_t pad_rows, int64_t cols,
                     int64_t pad_cols, void *dst, int64_t ld, int64_t row_off, int part,
                     cudaStream_t s) {
  stage_rows_bf16_kernel<<<grid_for(pad_rows * pad_cols), 256, 0, s>>>(
      src, rows, pad_rows, cols, pad_cols, static_cast<__nv_bfloat16 *>(dst), ld, row_off, part);
}

void unpad_f32(const float *src, int64_t ld, float *dst, int64_t rows, int64_t cols,
               cudaStream_t s) {
  unpad_f32_kernel<<<grid_for(rows * cols), 256, 0, s>>>(src, ld, dst, rows, cols);
}

void unpad_bf16_to_f32(const void *src, int64_t ld, float *dst, int64_t rows, int64_t cols,
                       cudaStream_t s) {
  unpad_bf16_kernel<<<grid_for(rows * cols), 256, 0, s>>>(static_cast<const __nv_bfloat16 *>(src), ld,
                                                           dst, rows, cols);
}

}  // namespace mimw
