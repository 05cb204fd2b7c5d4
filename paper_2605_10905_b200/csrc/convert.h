#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {
// part: 0 = bf16(x) ("hi"), 1 = bf16(x - bf16(x)) ("lo")
void stage_cols_bf16(const float *src, int64_t rows, int64_t cols, int64_t pad_cols, void *dst,
                     int64_t ld, int64_t col_off, int part, cudaStream_t s);
void stage_rows_bf16(const float *src, int64_t rows, int64_t pad_rows, int64_t cols,
                     int64_t pad_cols, void *dst, int64_t ld, int64_t row_off, int part,
                     cudaStream_t s);
void unpad_f32(const float *src, int64_t ld, float *dst, int64_t rows, int64_t cols,
               cudaStream_t s);
void unpad_bf16_to_f32(const void *src, int64_t ld, float *dst, int64_t rows, int64_t cols,
                       cudaStream_t s);
}  // namespace mimw
