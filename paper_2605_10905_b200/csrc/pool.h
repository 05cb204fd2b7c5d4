// Library-private stream-ordered memory pool (one per device).
//
// Scratch (staging buffers of the host-Tile entries, the attention-backward
// dQ accumulator, the MXFP8 scale atoms) comes from a cudaMemPool_t this
// library creates, with its release threshold set to keep freed memory: the
// default threshold (0) hands memory back to the driver at every
// synchronisation and the next call re-maps it (measured: tens of ms of jitter
// for the 0.8 GB backward accumulator).  The device's DEFAULT pool, which the
// host application's own cudaMallocAsync uses, is never touched
// (tests/test_capi_gpu.py checks its release threshold is unchanged).
// mimw_b200_trim_pool() returns the cached memory to the driver.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>

namespace mimw {

inline cudaMemPool_t scratch_pool() {
  static std::once_flag once[64];
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::call_once(once[dev], [dev] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = p;
    } else {
      cudaGetLastError();
    }
  });
  return pools[dev];
}

// Stream-ordered scratch from the private pool (freed with cudaFreeAsync).
inline cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = scratch_pool();
  if (pool == nullptr) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

}  // namespace mimw
