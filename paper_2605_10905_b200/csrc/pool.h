// Stream-ordered scratch comes from the device's default memory pool.  Its
// default release threshold (0) hands freed memory back to the driver at every
// synchronisation, and the next call re-maps it: measured as tens of ms of
// jitter for the attention-backward accumulator.  Every entry that allocates
// scratch calls this first, so the pool keeps its memory.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

namespace mimw {

inline void keep_pool_memory() {
  static std::once_flag once[64];  // host entries may be called from several threads
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
}

}  // namespace mimw
