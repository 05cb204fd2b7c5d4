// Cluster-cooperative LayerNorm for sm_100a:
//     y[r, j] = (x[r, j] - mean_r) * rstd_r * w[j] + b[j],
//     mean_r = sum_j x / n,  var_r = sum_j (x - mean_r)^2 / n,  rstd_r = 1 / sqrt(var_r + eps)
// i.e. oracle_layernorm (proj/core/src/oracles.cpp:28-55, two-pass mean then
// deviations), computed the way the reference's MIMW program distributes it
// (proj/kernels/layernorm_cluster.mimw:1-62): one thread-block cluster owns a
// row, CTA rank r owns a contiguous column slice, and the per-CTA partial
// reductions are exchanged through distributed shared memory with
// "arrive remote, wait local": every CTA st.async's its partial
// into each peer's smem slot, completing bytes on the PEER's mbarrier, then
// waits on its own.
//
// HBM-bound: the row slice is read once into registers (float4, coalesced),
// reduced twice (mean, then squared deviations: the oracle's two passes, from
// registers instead of a second HBM read) and written once.  Algorithmic
// bytes per element: 4 (x) + 4 (y); w and b are re-read per row from L2.
#include "layernorm_cluster.h"
#include "ptx.cuh"

#include <algorithm>
#include <cstdlib>

namespace mimw {

namespace {

constexpr int THREADS = 256;
constexpr int MAX_CLUSTER = 16;

__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   remote_addr),
               "r"(__float_as_uint(v)), "r"(remote_bar)
               : "memory");
}

// Block-wide sum; every thread gets the result (xor butterfly over all 32 lanes).
__device__ __forceinline__ float block_sum(float v, float *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // `red` reuse across calls
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = lane < THREADS / 32 ? red[lane] : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // every lane gets the total
  return t;
}

// All-gather of one float per CTA across the cluster through DSM; returns the
// cluster-wide sum (in rank order, so every CTA computes the identical value).
// `parity` is the barrier phase of this use (one use per row and round).
__device__ __forceinline__ float cluster_sum(float part, int round, int csize, uint32_t rank,
                                             float *slots, uint32_t bar, uint32_t parity,
                                             float *bcast) {
  if (threadIdx.x < 32) {  // warp 0: lane p sends to peer p, then the lanes sum the slots
    const int p = (int)threadIdx.x;
    const uint32_t my_slot = smem_u32(slots + round * MAX_CLUSTER + rank);
    if (p == 0) {
      slots[round * MAX_CLUSTER + rank] = part;
      mbar_arrive_expect_tx(bar, 4u * (uint32_t)(csize - 1));
    }
    if (p < csize && p != (int)rank) st_async_f32(map_to_rank(my_slot, (uint32_t)p), part, map_to_rank(bar, (uint32_t)p));
    mbar_wait(bar, parity, 60 + round);
    __syncwarp();  // lane 0's own-slot write visible to lane `rank`
    float s = p < csize ? slots[round * MAX_CLUSTER + p] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (p == 0) *bcast = s;
  }
  __syncthreads();
  return *bcast;
}

template <int VPT>
__device__ __forceinline__ void load_slice(float4 (&v)[VPT], const float *xr, int c0, int c1, int vec_ok) {
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = c0 + (i * THREADS + (int)threadIdx.x) * 4;
    if (vec_ok && c + 3 < c1) {
      v[i] = __ldcs(reinterpret_cast<const float4 *>(xr + c));
    } else {
      v[i].x = c < c1 ? xr[c] : 0.f;
      v[i].y = c + 1 < c1 ? xr[c + 1] : 0.f;
      v[i].z = c + 2 < c1 ? xr[c + 2] : 0.f;
      v[i].w = c + 3 < c1 ? xr[c + 3] : 0.f;
    }
  }
}

// Persistent: each cluster walks rows cluster_id, cluster_id + nclusters, ...
// and issues the loads of its next row before reducing the current one, so
// HBM reads overlap the two DSM exchange rounds and the stores.
template <int VPT>  // float4 vectors per thread (slice = VPT * 4 * THREADS columns)
__global__ void __launch_bounds__(THREADS)
layernorm_cluster_kernel(const float *__restrict__ x, const float *__restrict__ w,
                         const float *__restrict__ b, float *__restrict__ y, float *__restrict__ mean,
                         float *__restrict__ rstd, int rows, int n, int slice, float eps, int vec_ok) {
  __shared__ float red[THREADS / 32];
  __shared__ float slots[2 * MAX_CLUSTER];
  __shared__ alignas(8) uint64_t bars[2];
  __shared__ float bcast;
  const uint32_t rank = cluster_ctarank();
  const int nclusters = (int)nclusters_x();
  const int csize = (int)(gridDim.x / nclusters);
  const int c0 = (int)rank * slice;
  const int c1 = min(n, c0 + slice);
  const float inv_n = 1.f / (float)n;

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_mbar_init();
  }
  cluster_sync();  // peers' barriers are initialised before any st.async targets them

  int row = (int)cluster_id_x();
  float4 v[VPT], nx[VPT];
  if (row < rows) load_slice<VPT>(v, x + (size_t)row * n, c0, c1, vec_ok);
  uint32_t parity = 0;
  for (; row < rows; row += nclusters) {
    const int nrow = row + nclusters;
    if (nrow < rows) load_slice<VPT>(nx, x + (size_t)nrow * n, c0, c1, vec_ok);  // in flight

    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mu =
        cluster_sum(block_sum(s, red), 0, csize, rank, slots, smem_u32(&bars[0]), parity, &bcast) * inv_n;
    // second pass (the oracle's sum of squared deviations), from registers
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = c0 + (i * THREADS + (int)threadIdx.x) * 4;
      const float dx = c < c1 ? v[i].x - mu : 0.f;
      const float dy = c + 1 < c1 ? v[i].y - mu : 0.f;
      const float dz = c + 2 < c1 ? v[i].z - mu : 0.f;
      const float dw = c + 3 < c1 ? v[i].w - mu : 0.f;
      q += (dx * dx + dy * dy) + (dz * dz + dw * dw);
    }
    const float var =
        cluster_sum(block_sum(q, red), 1, csize, rank, slots, smem_u32(&bars[1]), parity, &bcast) * inv_n;
    const float rs = rsqrtf(var + eps);
    if (rank == 0 && threadIdx.x == 0) {
      if (mean) mean[row] = mu;
      if (rstd) rstd[row] = rs;
    }
    float *yr = y + (size_t)row * n;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = c0 + (i * THREADS + (int)threadIdx.x) * 4;
      if (vec_ok && c + 3 < c1) {
        const float4 ww = __ldg(reinterpret_cast<const float4 *>(w + c));
        const float4 bb = __ldg(reinterpret_cast<const float4 *>(b + c));
        float4 o;
        o.x = (v[i].x - mu) * rs * ww.x + bb.x;
        o.y = (v[i].y - mu) * rs * ww.y + bb.y;
        o.z = (v[i].z - mu) * rs * ww.z + bb.z;
        o.w = (v[i].w - mu) * rs * ww.w + bb.w;
        __stcs(reinterpret_cast<float4 *>(yr + c), o);
      } else {
        const float e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        for (int k = 0; k < 4; ++k)
          if (c + k < c1) yr[c + k] = (e[k] - mu) * rs * w[c + k] + b[c + k];
      }
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) v[i] = nx[i];
    parity ^= 1;
  }
  cluster_sync();  // no CTA leaves while a peer's st.async may still target it
}


__device__ __forceinline__ void st_async_f32x2(uint32_t remote_addr, float a, float b, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                   remote_addr),
               "f"(a), "f"(b), "r"(remote_bar)
               : "memory");
}

// Look-ahead variant: ONE exchange per row (each CTA sends its slice's sum
// and sum of squared deviations from the slice mean; Chan's pairwise
// combination gives the row's mean and variance), sent one row AHEAD: row
// k+1's partial statistics go out before row k is normalised, and row k's
// were sent an iteration earlier, so a CTA only waits when a peer is a whole
// row behind.  Rows k (normalising), k+1 (statistics) and k+2 (loads in
// flight) are in registers.  Three exchange slots (row mod 3): a CTA sends
// row k+1 only after receiving every peer's row k, by which time each peer
// has consumed row k-2 from the slot being overwritten.  Needs vec_ok.
template <int VPT>
__global__ void __launch_bounds__(THREADS, 2)
layernorm_cluster_la_kernel(const float *__restrict__ x, const float *__restrict__ w,
                            const float *__restrict__ b, float *__restrict__ y, float *__restrict__ mean,
                            float *__restrict__ rstd, int rows, int n, int slice, float eps) {
  __shared__ float red[THREADS / 32];
  __shared__ float2 xs[3][MAX_CLUSTER];
  __shared__ alignas(8) uint64_t bars[3];
  __shared__ float2 bc;
  const uint32_t rank = cluster_ctarank();
  const int nclusters = (int)nclusters_x();
  const int csize = (int)(gridDim.x / nclusters);
  const int c0 = (int)rank * slice;
  const int c1 = min(n, c0 + slice);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  cluster_sync();

  // local (sum, M2) of a slice in registers, sent to every peer's slot k % 3
  auto send_stats = [&](const float4 (&v)[VPT], int k) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float ssum = block_sum(s, red);
    const int nl = max(c1 - c0, 0);
    const float lmu = nl > 0 ? ssum / (float)nl : 0.f;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = c0 + (i * THREADS + (int)threadIdx.x) * 4;
      if (c < c1) {
        const float dx = v[i].x - lmu, dy = v[i].y - lmu, dz = v[i].z - lmu, dw = v[i].w - lmu;
        q += (dx * dx + dy * dy) + (dz * dz + dw * dw);
      }
    }
    const float m2 = block_sum(q, red);
    if (threadIdx.x < 32) {  // warp 0: lane p sends to peer p
      const int slot = k % 3;
      const uint32_t bar = smem_u32(&bars[slot]);
      const uint32_t mine = smem_u32(&xs[slot][rank]);
      if (threadIdx.x == 0) {
        xs[slot][rank] = make_float2(ssum, m2);
        mbar_arrive_expect_tx(bar, 8u * (uint32_t)(csize - 1));
      }
      const int p = (int)threadIdx.x;
      if (p < csize && p != (int)rank)
        st_async_f32x2(map_to_rank(mine, (uint32_t)p), ssum, m2, map_to_rank(bar, (uint32_t)p));
    }
  };

  const int row0 = (int)cluster_id_x();
  float4 A[VPT], B[VPT], C[VPT];
  if (row0 < rows) load_slice<VPT>(A, x + (size_t)row0 * n, c0, c1, 1);
  if (row0 + nclusters < rows) load_slice<VPT>(B, x + (size_t)(row0 + nclusters) * n, c0, c1, 1);
  if (row0 < rows) send_stats(A, 0);
  int k = 0;
  for (int row = row0; row < rows; row += nclusters, ++k) {
    const int r1 = row + nclusters, r2 = row + 2 * nclusters;
    if (r2 < rows) load_slice<VPT>(C, x + (size_t)r2 * n, c0, c1, 1);
    if (threadIdx.x < 32) {  // warp 0 combines: lane p holds peer p's (sum, M2)
      const int slot = k % 3;
      const int p = (int)threadIdx.x;
      mbar_wait(smem_u32(&bars[slot]), (uint32_t)(k / 3) & 1, 63);
      const float2 sp = p < csize ? xs[slot][p] : make_float2(0.f, 0.f);
      float tot = sp.x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const float mu = tot / (float)n;
      const int np = p < csize ? max(0, min(n, (p + 1) * slice) - p * slice) : 0;
      const float d = np > 0 ? sp.x / (float)np - mu : 0.f;
      float m2 = np > 0 ? sp.y + (float)np * d * d : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m2 += __shfl_xor_sync(0xffffffffu, m2, o);
      if (p == 0) {
        const float rs = rsqrtf(m2 / (float)n + eps);
        bc = make_float2(mu, rs);
        if (rank == 0) {
          if (mean) mean[row] = mu;
          if (rstd) rstd[row] = rs;
        }
      }
    }
    __syncthreads();
    const float2 st = bc;
    if (r1 < rows) send_stats(B, k + 1);  // its block reductions also order every read of bc before the next write
    float *yr = y + (size_t)row * n;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = c0 + (i * THREADS + (int)threadIdx.x) * 4;
      if (c < c1) {
        const float4 ww = __ldg(reinterpret_cast<const float4 *>(w + c));
        const float4 bb = __ldg(reinterpret_cast<const float4 *>(b + c));
        float4 o;
        o.x = (A[i].x - st.x) * st.y * ww.x + bb.x;
        o.y = (A[i].y - st.x) * st.y * ww.y + bb.y;
        o.z = (A[i].z - st.x) * st.y * ww.z + bb.z;
        o.w = (A[i].w - st.x) * st.y * ww.w + bb.w;
        __stcs(reinterpret_cast<float4 *>(yr + c), o);
      }
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      A[i] = B[i];
      B[i] = C[i];
    }
  }
  cluster_sync();  // no CTA leaves while a peer's st.async may still target it
}

}  // namespace

cudaError_t layernorm_cluster_launch(const LayerNormArgs &a, cudaStream_t stream) {
  if (a.rows <= 0 || a.n <= 0) return cudaSuccess;
  // cluster size: enough CTAs that each slice fits VPT <= 8 float4 per
  // thread (8K columns per CTA, up to 16K at the 16-CTA limit); for few rows, more CTAs per row (slices of
  // >= 256 columns) so the whole chip streams the rows; a power of two <= 16
  // (16 is the opt-in non-portable size).  4 x 1024 gives the reference's
  // 4-CTA cluster of 256-column slices (layernorm_cluster.mimw:1-4).
  // (8K-column slices measured fastest: tools/ln_sweep.py; 16K only when a
  // 16-CTA cluster is not enough)
  const int64_t per_cta_max = 8LL * 4 * THREADS;
  int64_t want = std::max<int64_t>((a.n + per_cta_max - 1) / per_cta_max,
                                   std::min<int64_t>((148 + a.rows - 1) / a.rows, a.n / 256));
  int csize = 1;
  while (csize < want && csize < MAX_CLUSTER) csize *= 2;
  if (a.cluster > 0) csize = a.cluster;
  int slice = (int)((a.n + csize - 1) / csize);
  slice = (slice + 3) / 4 * 4;
  const int vec = (slice + 4 * THREADS - 1) / (4 * THREADS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.rows * csize), 1, 1);  // sized below (persistent)
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> cudaError_t {
    if (csize > 8) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    const int vec_ok = (a.n % 4 == 0) &&
                       ((((uintptr_t)a.x | (uintptr_t)a.w | (uintptr_t)a.b | (uintptr_t)a.y) & 15) == 0);
    // persistent: as many clusters as are co-resident, at most one per row
    int active = 0;
    cfg.gridDim = dim3((unsigned)(std::min<int64_t>(a.rows, 4096) * csize), 1, 1);
    if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) != cudaSuccess || active <= 0) {
      cudaGetLastError();
      active = std::max(1, 148 / csize);
    }
    const int64_t clusters = std::min<int64_t>(a.rows, active);
    cfg.gridDim = dim3((unsigned)(clusters * csize), 1, 1);
    return cudaLaunchKernelEx(&cfg, kern, a.x, a.w, a.b, a.y, a.mean, a.rstd, (int)a.rows, (int)a.n,
                              slice, (float)a.eps, vec_ok);
  };
  auto go_la = [&](auto kern) -> cudaError_t {
    if (csize > 8) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    int active = 0;
    cfg.gridDim = dim3((unsigned)(std::min<int64_t>(a.rows, 4096) * csize), 1, 1);
    if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) != cudaSuccess || active <= 0) {
      cudaGetLastError();
      active = std::max(1, 148 / csize);
    }
    cfg.gridDim = dim3((unsigned)(std::min<int64_t>(a.rows, active) * csize), 1, 1);
    return cudaLaunchKernelEx(&cfg, kern, a.x, a.w, a.b, a.y, a.mean, a.rstd, (int)a.rows, (int)a.n, slice,
                              (float)a.eps);
  };
  static const int la_env = getenv("MIMW_LN_LOOKAHEAD") ? atoi(getenv("MIMW_LN_LOOKAHEAD")) : 1;  // A/B knob (1: measured +15%)
  const bool vec_ok = (a.n % 4 == 0) &&
                      ((((uintptr_t)a.x | (uintptr_t)a.w | (uintptr_t)a.b | (uintptr_t)a.y) & 15) == 0);
  if (la_env && vec_ok) {
    if (vec <= 1) return go_la(layernorm_cluster_la_kernel<1>);
    if (vec <= 2) return go_la(layernorm_cluster_la_kernel<2>);
    if (vec <= 4) return go_la(layernorm_cluster_la_kernel<4>);
    if (vec <= 8) return go_la(layernorm_cluster_la_kernel<8>);
  }
  if (vec <= 1) return go(layernorm_cluster_kernel<1>);
  if (vec <= 2) return go(layernorm_cluster_kernel<2>);
  if (vec <= 4) return go(layernorm_cluster_kernel<4>);
  if (vec <= 8) return go(layernorm_cluster_kernel<8>);
  if (vec <= 16) return go(layernorm_cluster_kernel<16>);
  return cudaErrorInvalidValue;  // n > 16 * 16K columns
}

}  // namespace mimw
