// Host-side TMA descriptor encoding through the driver entry point (no -lcuda
// at link time: the symbol is resolved from the loaded driver at run time).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace mimw {

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Row-major 2-D tensor [rows, cols] with leading dimension `ld` (elements),
// box {box_cols, box_rows}.  dim0 = cols (contiguous).
inline CUtensorMap make_tmap_2d(const void *base, CUtensorMapDataType dt, int elem_bytes,
                                uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                                uint32_t box_rows, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled_fn()(&m, dt, 2, const_cast<void *>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) +
                             ") rows=" + std::to_string(rows) + " cols=" + std::to_string(cols) +
                             " ld=" + std::to_string(ld));
  return m;
}

// 3-D tensor [d2, d1, d0] with strides (elements) s1 (dim1), s2 (dim2).
inline CUtensorMap make_tmap_3d(const void *base, CUtensorMapDataType dt, int elem_bytes,
                                uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                                uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * (uint64_t)elem_bytes, s2 * (uint64_t)elem_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_tiled_fn()(&m, dt, 3, const_cast<void *>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled(3d) failed (" + std::to_string((int)r) + ")");
  return m;
}

inline int sm_count(int device = -1) {
  static int cached[64] = {0};
  if (device < 0) cudaGetDevice(&device);
  if (device < 64 && cached[device]) return cached[device];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (device < 64) cached[device] = n;
  return n;
}

}  // namespace mimw
