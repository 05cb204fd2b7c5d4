// Microbenchmark: per-SM throughput of a single-thread TMA copy pipeline
// (global -> smem -> global), the comm role of the all-gather GEMM.
// Each CTA copies its contiguous share of a buffer with `nb` smem buffers of
// `box` bytes (1-D cp.async.bulk), a buffer refilled once its store has read
// it; MODE 1 also waits for full store completion `lag` stores behind (the
// slab-signal wait); MODE 2 splits the CTA's work over `agents` threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_copy tools/tma_copy.cu
//   tools/tma_copy [ctas]
#include <cstdio>
#include <vector>
#include "../paper_2605_10905_b200/csrc/ptx.cuh"
using namespace mimw;

__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}

template <int LAG>
__device__ void agent(const char *src, char *dst, size_t bytes, uint32_t buf0, uint32_t bar0, int nb,
                      uint32_t box, bool wait_full) {
  for (int i = 0; i < nb; ++i) mbar_init(bar0 + 8 * i, 1);
  fence_mbar_init();
  const int n = (int)(bytes / box);
  int nl = 0;
  auto load = [&](int idx) {
    const int slot = idx % nb;
    mbar_arrive_expect_tx(bar0 + 8 * slot, box);
    bulk_load(buf0 + slot * box, src + (size_t)idx * box, box, bar0 + 8 * slot);
  };
  while (nl < nb && nl < n) load(nl++);
  for (int ns = 0; ns < n; ++ns) {
    const int slot = ns % nb;
    mbar_wait(bar0 + 8 * slot, (uint32_t)((ns / nb) & 1));
    bulk_store(dst + (size_t)ns * box, buf0 + slot * box, box);
    bulk_commit();
    if (ns >= 1) {
      bulk_wait_read<1>();
      if (nl < n) load(nl++);
    }
    if (wait_full && ns >= LAG) bulk_wait<LAG>();
  }
  bulk_wait<0>();
}

// all threads: 16-byte LDG x U in flight, then STG (the LSU path)
template <int U>
__device__ void ldg_copy(const char *src, char *dst, size_t bytes) {
  const int4 *s = reinterpret_cast<const int4 *>(src);
  int4 *d = reinterpret_cast<int4 *>(dst);
  const size_t n = bytes / 16;
  for (size_t i = threadIdx.x; i < n; i += (size_t)blockDim.x * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + (size_t)u * blockDim.x;
      if (j < n) v[u] = __ldcs(s + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + (size_t)u * blockDim.x;
      if (j < n) __stcs(d + j, v[u]);
    }
  }
}

__global__ void __launch_bounds__(192, 1) copy_kernel(const char *src, char *dst, size_t per_cta,
                                                      int nb, uint32_t box, int mode, int agents) {
  extern __shared__ uint8_t sm[];
  __shared__ uint64_t bars[32];
  const uint32_t buf = (smem_u32(sm) + 1023) & ~1023u;
  const char *s = src + blockIdx.x * per_cta;
  char *d = dst + blockIdx.x * per_cta;
  const int warp = threadIdx.x / 32;
  if (mode == 3) { ldg_copy<8>(s, d, per_cta); return; }
  if (mode == 4) { ldg_copy<16>(s, d, per_cta); return; }
  if (threadIdx.x % 32 == 0 && warp < agents) {
    const int nba = nb / agents;
    const size_t share = per_cta / agents;
    agent<8>(s + warp * share, d + warp * share, share, buf + warp * nba * box,
             smem_u32(&bars[warp * nba]), nba, box, mode == 1);
  }
}

int main(int argc, char **argv) {
  int ctas_list[] = {8, 16, 148};
  size_t per_cta = 8u << 20;
  char *src, *dst;
  cudaMalloc(&src, per_cta * 148);
  cudaMalloc(&dst, per_cta * 148);
  cudaMemset(src, 1, per_cta * 148);
  cudaFuncSetAttribute(copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int nb; uint32_t box; int mode; int agents; };
  std::vector<Cfg> cfgs = {{6, 32768, 0, 1}, {6, 32768, 1, 1}, {12, 16384, 0, 1}, {12, 16384, 1, 1},
                           {24, 8192, 0, 1},  {12, 16384, 0, 2}, {3, 65536, 0, 1},
                           {2, 65536, 0, 1}, {6, 32768, 3, 1}, {6, 32768, 4, 1}};
  for (int ctas : ctas_list) {
    for (auto c : cfgs) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<ctas, 192, 200 * 1024>>>(src, dst, per_cta, c.nb, c.box, c.mode, c.agents);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      printf("ctas %3d nb %2d box %6u mode %d agents %d: %7.3f ms  %7.1f GB/s/SM (copy)  total %7.1f GB/s %s\n",
             ctas, c.nb, c.box, c.mode, c.agents, ms, per_cta / (ms * 1e6), per_cta * ctas / (ms * 1e6),
             err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  }
  return 0;
}
