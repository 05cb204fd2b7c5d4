// Split-bf16 x3 attention for the host-Tile entry points (MIMW_PREC_F32_BF16X3):
// oracle_attention (proj/core/src/oracles.cpp:119-145) at the reference's own
// f32 tolerance (1e-4, acceptance.cpp:333-355) on the tcgen05 tensor cores.
//
// Same algebra as the GEMM's x3 mode (convert.cu): x = hi + lo, hi = bf16(x),
// lo = bf16(x - hi), and A.B ~= Ah.Bh + Ah.Bl + Al.Bh as ONE bf16 GEMM with
// K' = 3K and fp32 accumulate (the dropped Al.Bl term is ~2^-16 relative).
// Per query-row block [r0, r0 + R) of one head, over the block's key range
// [klo, khi) = [max(0, r0 - w + 1), r0 + R) (the causal window of its rows):
//
//   S  = [Qh | Qh | Ql] . [Kh | Kl | Kh]^T        (gemm_bf16, B_NK, f32 out)
//   P  = exp(scale S - m) / l per row, within i - w < j <= i, else 0;
//        lse = m + log l                           (softmax_split3_kernel, f32 / f64 sum)
//   O  = Px . Vx, Px[i, 3j + t] = (Ph, Ph, Pl)[t], Vx[3j + t] = (Vh, Vl, Vh)[t]
//                                                  (gemm_bf16, B_KN, f32 out)
//
// Interleaving the three parts per key keeps any key range one contiguous
// K' range of Px / Vx, so a row block only multiplies the keys its window
// can reach.  Scores and P are materialised (R x (khi - klo) f32), which is
// the right trade for the reference's Tile sizes; the fused one-pass kernel
// (attention_fwd.cu) is the bf16 production path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "attention_x3.h"
#include "gemm_bf16.h"

namespace mimw {

namespace {

__device__ __forceinline__ __nv_bfloat16 part_of(float x, int lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  return lo ? __float2bfloat16_rn(x - __bfloat162float(h)) : h;
}

// dst[r, t * dp + c] = part_t(src[r, c]) (0 for c >= d); part t is lo iff bit t of lo_mask.
__global__ void split3_cols_kernel(const float *__restrict__ src, int64_t rows, int d, int dp,
                                   __nv_bfloat16 *__restrict__ dst, int lo_mask) {
  const int64_t n = rows * 3 * dp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (3 * dp);
    const int cc = (int)(i - r * 3 * dp), t = cc / dp, c = cc - t * dp;
    dst[i] = part_of(c < d ? src[r * d + c] : 0.f, (lo_mask >> t) & 1);
  }
}

// dst[3 j + t, c] = (Vh, Vl, Vh)[t][j, c] (0 for c >= d).
__global__ void split3_rows_kernel(const float *__restrict__ src, int64_t rows, int d, int dp,
                                   __nv_bfloat16 *__restrict__ dst) {
  const int64_t n = rows * 3 * dp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = i / dp;
    const int c = (int)(i - rr * dp);
    const int64_t j = rr / 3;
    const int t = (int)(rr - 3 * j);
    dst[i] = part_of(c < d ? src[j * d + c] : 0.f, t == 1);
  }
}

// One warp per query row i = r0 + blockIdx.x * 8 + warp.  S row pitch lds
// (f32), key columns relative to klo; writes the whole Px row [0, 3 nk).
__global__ void __launch_bounds__(256)
softmax_split3_kernel(const float *__restrict__ S, int64_t lds, __nv_bfloat16 *__restrict__ px, int64_t ldp,
                      int64_t r0, int64_t rows, int64_t klo, int64_t nk, int64_t w, float scale,
                      float *__restrict__ lse) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rr = (int64_t)blockIdx.x * 8 + warp;
  if (rr >= rows) return;
  const int64_t i = r0 + rr;
  const int64_t lo = (i - w + 1 > klo ? i - w + 1 : klo) - klo, hi = i - klo;  // window, inclusive
  const float *s = S + rr * lds;
  float m = -INFINITY;
  for (int64_t j = lo + lane; j <= hi; j += 32) m = fmaxf(m, s[j] * scale);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  double l = 0.0;
  for (int64_t j = lo + lane; j <= hi; j += 32) l += (double)expf(s[j] * scale - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  const float inv = (float)(1.0 / l);
  __nv_bfloat16 *p = px + rr * ldp;
  for (int64_t j = lane; j < nk; j += 32) {
    const float v = (j >= lo && j <= hi) ? expf(s[j] * scale - m) * inv : 0.f;
    const __nv_bfloat16 h = part_of(v, 0), q = part_of(v, 1);
    p[3 * j] = h;
    p[3 * j + 1] = h;
    p[3 * j + 2] = q;
  }
  if (lse != nullptr && lane == 0) lse[i] = (float)((double)m + log(l));
}

int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

size_t attention_x3_workspace_bytes(int64_t seq, int64_t d) {
  const int64_t dp = round_up(d, 8);
  const int64_t rb = attention_x3_row_block(seq);
  const int64_t nk = round_up(seq, 8);
  return (size_t)2 * seq * 3 * dp * 2      // Qx, Kx
         + (size_t)3 * seq * dp * 2        // Vx
         + (size_t)seq * dp * 4            // O (f32, padded columns)
         + (size_t)rb * round_up(nk, 4) * 4  // S block
         + (size_t)rb * round_up(3 * nk, 8) * 2 + 1024;  // Px block, alignment slack
}

int64_t attention_x3_row_block(int64_t seq) {
  // S + Px cost 10 B per (row, key): keep a block's pair under ~64 MiB (L2-sized
  // blocks; S = 8192 runs as 768-row blocks, each a 768 x <= 8192 x 3D GEMM)
  const int64_t cap = (64ll << 20) / (10 * (seq > 0 ? seq : 1));
  int64_t rb = cap < 256 ? 256 : cap / 256 * 256;
  return rb < seq ? rb : seq;
}

cudaError_t attention_x3_launch(const AttnX3Args &a, cudaStream_t s) {
  if (a.seq <= 0) return cudaSuccess;
  const int64_t seq = a.seq, d = a.d, dp = round_up(d, 8);
  const int64_t rb = attention_x3_row_block(seq);
  const int64_t w = a.w < seq ? a.w : seq;
  char *ws = static_cast<char *>(a.workspace);
  auto take = [&](size_t bytes) {
    char *p = ws;
    ws += (bytes + 255) / 256 * 256;
    return p;
  };
  auto *qx = reinterpret_cast<__nv_bfloat16 *>(take((size_t)seq * 3 * dp * 2));
  auto *kx = reinterpret_cast<__nv_bfloat16 *>(take((size_t)seq * 3 * dp * 2));
  auto *vx = reinterpret_cast<__nv_bfloat16 *>(take((size_t)3 * seq * dp * 2));
  auto *of = reinterpret_cast<float *>(take((size_t)seq * dp * 4));
  const int64_t nk_max = round_up(seq, 8);
  auto *sb = reinterpret_cast<float *>(take((size_t)rb * round_up(nk_max, 4) * 4));
  auto *pb = reinterpret_cast<__nv_bfloat16 *>(take((size_t)rb * round_up(3 * nk_max, 8) * 2));
  split3_cols_kernel<<<grid_for(seq * 3 * dp), 256, 0, s>>>(a.q, seq, (int)d, (int)dp, qx, 0b100);  // Qh Qh Ql
  split3_cols_kernel<<<grid_for(seq * 3 * dp), 256, 0, s>>>(a.k, seq, (int)d, (int)dp, kx, 0b010);  // Kh Kl Kh
  split3_rows_kernel<<<grid_for(seq * 3 * dp), 256, 0, s>>>(a.v, seq, (int)d, (int)dp, vx);
  cudaError_t err = cudaGetLastError();
  for (int64_t r0 = 0; r0 < seq && err == cudaSuccess; r0 += rb) {
    const int64_t rows = seq - r0 < rb ? seq - r0 : rb;
    const int64_t klo = r0 - w + 1 > 0 ? r0 - w + 1 : 0, khi = r0 + rows, nk = khi - klo;
    const int64_t lds = round_up(nk, 4), ldp = round_up(3 * nk, 8);
    GemmArgs g{};
    g.a = qx + r0 * 3 * dp;
    g.b = kx + klo * 3 * dp;
    g.c = sb;
    g.m = rows;
    g.n = nk;
    g.k = 3 * dp;
    g.lda = g.ldb = 3 * dp;
    g.ldc = lds;
    g.b_kn = false;
    g.c_f32 = true;
    g.cta_group = 2;
    err = gemm_bf16_launch(g, s);
    if (err != cudaSuccess) break;
    softmax_split3_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(sb, lds, pb, ldp, r0, rows, klo, nk, w,
                                                                    (float)a.scale, a.lse);
    err = cudaGetLastError();
    if (err != cudaSuccess) break;
    GemmArgs h{};
    h.a = pb;
    h.b = vx + 3 * klo * dp;
    h.c = of + r0 * dp;
    h.m = rows;
    h.n = dp;
    h.k = 3 * nk;
    h.lda = ldp;
    h.ldb = dp;
    h.ldc = dp;
    h.b_kn = true;
    h.c_f32 = true;
    h.cta_group = 2;
    err = gemm_bf16_launch(h, s);
  }
  if (err != cudaSuccess) return err;
  if (dp == d) return cudaMemcpyAsync(a.o, of, (size_t)seq * d * 4, cudaMemcpyDeviceToDevice, s);
  return cudaMemcpy2DAsync(a.o, (size_t)d * 4, of, (size_t)dp * 4, (size_t)d * 4, (size_t)seq,
                           cudaMemcpyDeviceToDevice, s);
}

}  // namespace mimw
