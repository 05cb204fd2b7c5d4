// Reference-precision attention for the host-Tile entry points
// (MIMW_PREC_F32): the arithmetic of the reference's oracles kept on the GPU,
// for callers that need the reference's own tolerances (1e-4 / 1e-3,
// acceptance.cpp:333-355, simplicial_attention.case) rather than the bf16
// tensor-core path's 1e-2.
//
//   attention:  oracle_attention            (proj/core/src/oracles.cpp:119-145)
//   simplicial: oracle_simplicial_attention (proj/core/src/oracles.cpp:82-117)
//
// One CTA per query row, CUDA cores: scores and the softmax bookkeeping in
// f64 as the oracles compute them, the output accumulated in f32, over the
// row's key set in chunks of 256 with an online max (the oracles' two-pass
// max / normalise gives the same result up to f32 rounding).  Sized for the
// reference's Tiles (S = 32 .. a few thousand); the production path for real
// workloads is the tcgen05 kernels (attention_fwd.cu, simplicial_fwd.cu).
#include "attention_f32.h"

#include <cmath>

namespace mimw {

namespace {

constexpr int THREADS = 128;  // thread x owns output column x (d <= 128)
constexpr int CHUNK = 256;

__device__ __forceinline__ double block_reduce(double v, double *red, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < THREADS / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
  return r;
}

// Row i of either oracle.  mode 0: keys j in [lo1, hi1] (attention, v = v1);
// mode 1: pairs (j1, j2) in [lo1, hi1] x [lo2, hi2] (simplicial, v = v1 (.) v2).
__global__ void __launch_bounds__(THREADS)
attention_f32_kernel(const float *__restrict__ q, const float *__restrict__ k1, const float *__restrict__ v1,
                     const float *__restrict__ k2, const float *__restrict__ v2, float *__restrict__ o,
                     float *__restrict__ lse, int seq, int d, int w1, int w2, int causal, int mode,
                     double scale) {
  __shared__ double qs[THREADS];
  __shared__ double sc[CHUNK];
  __shared__ int j1s[CHUNK], j2s[CHUNK];
  __shared__ double red[THREADS / 32];
  const int i = blockIdx.x;
  const int x = threadIdx.x;
  qs[x] = x < d ? (double)q[(size_t)i * d + x] : 0.0;
  const int lo1 = causal ? max(0, i - w1 + 1) : 0, hi1 = causal ? i : seq - 1;
  const int lo2 = max(0, i - w2 + 1), hi2 = i;
  const int n1 = hi1 - lo1 + 1;
  const int n2 = mode ? hi2 - lo2 + 1 : 1;
  const long long npairs = (long long)n1 * n2;
  double m = -INFINITY, l = 0.0;
  float acc = 0.f;
  __syncthreads();
  for (long long c0 = 0; c0 < npairs; c0 += CHUNK) {
    const int cnt = (int)(npairs - c0 < CHUNK ? npairs - c0 : CHUNK);
    // scores of this chunk, two pairs per thread
    for (int t = x; t < cnt; t += THREADS) {
      const long long pidx = c0 + t;
      const int j1 = lo1 + (int)(pidx / n2);
      const int j2 = mode ? lo2 + (int)(pidx % n2) : 0;
      double s = 0.0;
      const float *a = k1 + (size_t)j1 * d;
      if (mode) {
        const float *b = k2 + (size_t)j2 * d;
        for (int e = 0; e < d; ++e) s += qs[e] * (double)a[e] * (double)b[e];
      } else {
        for (int e = 0; e < d; ++e) s += qs[e] * (double)a[e];
      }
      sc[t] = s * scale;
      j1s[t] = j1;
      j2s[t] = j2;
    }
    __syncthreads();
    double cm = -INFINITY;
    for (int t = x; t < cnt; t += THREADS) cm = fmax(cm, sc[t]);
    cm = block_reduce(cm, red, true);
    const double mn = fmax(m, cm);
    const double corr = (m == -INFINITY) ? 0.0 : exp(m - mn);
    l *= corr;
    acc = (float)((double)acc * corr);
    double cs = 0.0;
    for (int t = x; t < cnt; t += THREADS) cs += exp(sc[t] - mn);
    l += block_reduce(cs, red, false);
    if (x < d) {
      for (int t = 0; t < cnt; ++t) {
        const double p = exp(sc[t] - mn);
        const float vv = mode ? v1[(size_t)j1s[t] * d + x] * v2[(size_t)j2s[t] * d + x] : v1[(size_t)j1s[t] * d + x];
        acc += (float)(p * (double)vv);
      }
    }
    m = mn;
    __syncthreads();  // sc / j reused by the next chunk
  }
  if (x < d) o[(size_t)i * d + x] = l > 0.0 ? (float)((double)acc / l) : 0.f;
  if (lse != nullptr && x == 0) lse[i] = (float)(m + log(l));
}

}  // namespace

cudaError_t attention_f32_launch(const AttnF32Args &a, cudaStream_t stream) {
  if (a.seq <= 0) return cudaSuccess;
  attention_f32_kernel<<<(unsigned)a.seq, THREADS, 0, stream>>>(
      a.q, a.k1, a.v1, a.k2, a.v2, a.o, a.lse, (int)a.seq, (int)a.d,
      (int)(a.w1 < a.seq ? a.w1 : a.seq), (int)(a.w2 < a.seq ? a.w2 : a.seq),  // windows >= seq: every key (no int overflow)
      a.causal ? 1 : 0,
      a.simplicial ? 1 : 0, a.scale);
  return cudaGetLastError();
}

}  // namespace mimw
