// Host-side bf16 staging for the host-f32 Tile entries (MIMW_PREC_BF16): the
// f32 -> bf16 round-to-nearest-even conversion runs on the host threads into
// pinned buffers, so PCIe carries 2 bytes per element instead of 4 (the e2e
// path is bound by the H2D stream).  Bit-identical to the device staging
// kernels (__float2bfloat16_rn; NaN -> 0x7FFF).
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>

namespace mimw {

// dst[r * ld_dst + col_off + j] = bf16_rne(src[r * ld_src + j]), r < rows, j < cols
void host_rows_to_bf16(const float *src, int64_t ld_src, int64_t rows, int64_t cols, uint16_t *dst,
                       int64_t ld_dst, int64_t col_off);

// dst[r * ld_dst + j] = f32(src[r * ld_src + j]) for bf16 src (exact widening)
void host_rows_bf16_to_f32(const uint16_t *src, int64_t ld_src, int64_t rows, int64_t cols, float *dst,
                           int64_t ld_dst);

// dst[0, n) = src[0, n) with streaming stores (the drain of a pinned result
// slot into the caller's pageable buffer)
void host_copy_f32(float *dst, const float *src, int64_t n);

// Runs f(lo, hi) over [0, n) split across the process-wide host thread pool
// (the caller participates) and returns when every range is done.
void host_parallel_for(int64_t n, const std::function<void(int64_t, int64_t)> &f);

// A pinned (page-locked) host buffer of at least `bytes` owned by the calling
// thread, reused across its calls with the same slot index.
void *pinned_slot(int slot, size_t bytes);

}  // namespace mimw
