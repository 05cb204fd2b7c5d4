// Split-bf16 x3 attention (MIMW_PREC_F32_BF16X3) for one causal-window head of
// f32 device tensors; see attention_x3.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mimw {

struct AttnX3Args {
  const float *q, *k, *v;  // [seq, d] f32 device
  float *o;                // [seq, d] f32 device
  float *lse;              // [seq] f32 device or nullptr
  int64_t seq, d, w;       // d <= 128 (any), w >= 1
  double scale;
  void *workspace;         // attention_x3_workspace_bytes(seq, d) bytes, 256-B aligned
};

int64_t attention_x3_row_block(int64_t seq);
size_t attention_x3_workspace_bytes(int64_t seq, int64_t d);
cudaError_t attention_x3_launch(const AttnX3Args &a, cudaStream_t s);

}  // namespace mimw
