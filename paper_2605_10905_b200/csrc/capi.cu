// extern "C" boundary of libmimw_b200.so (declared in include/mimw_b200.h).
//
// Each mimw_b200_oracle_* entry replaces one function of the reference's
// operator API, proj/core/include/mimw/oracles.hpp, with the same argument
// meaning (row-major f32 host Tiles).  The mimw_b200_* device entries are the
// production path.  No exception crosses the ABI; no CPU fallback exists.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mimw_b200.h"
#include "convert.h"
#include "gemm_bf16.h"

namespace {

thread_local std::string g_last_error;

struct MimwError : std::runtime_error {
  int code;
  MimwError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw MimwError(MIMW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F &&f) {
  try {
    f();
    return MIMW_OK;
  } catch (const MimwError &e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception &e) {
    g_last_error = e.what();
    return MIMW_ERR_CUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return MIMW_ERR_CUDA;
  }
}

void require_sm100() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0;
    cudaDeviceProp p;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    } else {
      ok = (p.major == 10) ? 1 : 0;
    }
  }
  if (!ok) throw MimwError(MIMW_ERR_CUDA, "no sm_100 (B200) device visible; libmimw_b200 has no CPU fallback");
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

void require(bool c, int code, const std::string &msg) {
  if (!c) throw MimwError(code, msg);
}

void require_pitch(const void *p, int64_t ld, int64_t es, const char *name) {
  require(((uintptr_t)p & 15) == 0, MIMW_ERR_UNSUPPORTED, std::string(name) + ": base not 16-byte aligned");
  require((ld * es) % 16 == 0, MIMW_ERR_UNSUPPORTED,
          std::string(name) + ": row pitch must be a multiple of 16 bytes (TMA)");
}

// RAII device scratch on a stream.
struct DevBuf {
  void *p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) check_cuda(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T *as() const { return static_cast<T *>(p); }
};

// C[m,n] (host f32) = sum_parts A_i[m,k_i] . B_i[k_i,n] on tensor cores.
// The K-parts are concatenated along K (oracle_multi_device_gemm,
// oracles.cpp:57-80); with MIMW_PREC_F32_BF16X3 every part is expanded to its
// three split-bf16 products (convert.cu).
void host_gemm(const std::vector<const float *> &a_parts, const std::vector<const float *> &b_parts,
               const std::vector<int64_t> &k_parts, int64_t m, int64_t n, float *c, int precision) {
  require(precision == MIMW_PREC_BF16 || precision == MIMW_PREC_F32_BF16X3, MIMW_ERR_ARG,
          "precision must be MIMW_PREC_BF16 or MIMW_PREC_F32_BF16X3");
  require(m >= 0 && n >= 0, MIMW_ERR_SHAPE, "negative extent");
  int64_t k = 0;
  for (auto kk : k_parts) {
    require(kk >= 0, MIMW_ERR_SHAPE, "negative extent");
    k += kk;
  }
  if (m == 0 || n == 0) return;
  require(c != nullptr, MIMW_ERR_ARG, "null output");
  if (k == 0) {  // float accumulator starts at 0.0f (oracles.cpp:19)
    std::memset(c, 0, sizeof(float) * m * n);
    return;
  }
  for (size_t i = 0; i < a_parts.size(); ++i)
    require(k_parts[i] == 0 || (a_parts[i] && b_parts[i]), MIMW_ERR_ARG, "null input");
  require_sm100();

  cudaStream_t s = cudaStreamPerThread;
  const int nseg = precision == MIMW_PREC_F32_BF16X3 ? 3 : 1;
  const int64_t kp = round_up(k, 8);  // bf16 row pitch multiple of 16 B
  const int64_t np = round_up(n, 8);
  const int64_t kt = nseg * kp;
  size_t in_elems = 0;
  for (size_t i = 0; i < a_parts.size(); ++i) in_elems += (m + n) * k_parts[i];
  DevBuf din(sizeof(float) * in_elems, s);
  DevBuf dA(2 * m * kt, s), dB(2 * kt * np, s), dC(sizeof(float) * m * np, s);

  // segment products: (A part, B part) for hi.hi [, hi.lo, lo.hi]
  const int a_part_of_seg[3] = {0, 0, 1};
  const int b_part_of_seg[3] = {0, 1, 0};
  float *cursor = din.as<float>();
  int64_t koff = 0;
  for (size_t i = 0; i < a_parts.size(); ++i) {
    const int64_t ki = k_parts[i];
    if (ki == 0) continue;
    float *da = cursor;
    float *db = cursor + m * ki;
    cursor += (m + n) * ki;
    check_cuda(cudaMemcpyAsync(da, a_parts[i], sizeof(float) * m * ki, cudaMemcpyHostToDevice, s), "H2D a");
    check_cuda(cudaMemcpyAsync(db, b_parts[i], sizeof(float) * ki * n, cudaMemcpyHostToDevice, s), "H2D b");
    const bool last = (i + 1 == a_parts.size()) || (koff + ki == k);
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int64_t base = sgi * kp + koff;
      // the last part also zero-fills the K padding of its segment
      const int64_t a_pad = last ? (kp - koff) : ki;
      mimw::stage_cols_bf16(da, m, ki, a_pad, dA.p, kt, base, a_part_of_seg[sgi], s);
      mimw::stage_rows_bf16(db, ki, a_pad, n, np, dB.p, np, base, b_part_of_seg[sgi], s);
    }
    koff += ki;
  }
  check_cuda(cudaGetLastError(), "staging kernels");

  mimw::GemmArgs g{};
  g.a = dA.p;
  g.b = dB.p;
  g.c = dC.p;
  g.m = m;
  g.n = np;
  g.k = kt;
  g.lda = kt;
  g.ldb = np;
  g.ldc = np;
  g.b_kn = true;
  g.c_f32 = true;
  g.cta_group = 2;
  check_cuda(mimw::gemm_bf16_launch(g, s), "gemm launch");
  check_cuda(cudaMemcpy2DAsync(c, sizeof(float) * n, dC.p, sizeof(float) * np, sizeof(float) * n, m,
                               cudaMemcpyDeviceToHost, s),
             "D2H c");
  check_cuda(cudaStreamSynchronize(s), "gemm execution");
}

}  // namespace

extern "C" {

int mimw_b200_version(void) { return 1; }

const char *mimw_b200_last_error(void) { return g_last_error.c_str(); }

int mimw_b200_oracle_gemm(const float *a, const float *b, float *c, int64_t m, int64_t n, int64_t k,
                          int32_t precision) {
  return guarded([&] { host_gemm({a}, {b}, {k}, m, n, c, precision); });
}

int mimw_b200_oracle_multi_device_gemm(const float *a0, const float *a1, const float *b0,
                                       const float *b1, float *c, int64_t m, int64_t k0, int64_t k1,
                                       int64_t n, int32_t precision) {
  return guarded([&] { host_gemm({a0, a1}, {b0, b1}, {k0, k1}, m, n, c, precision); });
}

int mimw_b200_gemm_bf16(const void *a, const void *b, void *c, int64_t m, int64_t n, int64_t k,
                        int64_t lda, int64_t ldb, int64_t ldc, int32_t b_layout, int32_t c_dtype,
                        void *stream) {
  return guarded([&] {
    require(b_layout == MIMW_B_KN || b_layout == MIMW_B_NK, MIMW_ERR_ARG, "bad b_layout");
    require(c_dtype == MIMW_F32 || c_dtype == MIMW_BF16, MIMW_ERR_ARG, "bad c_dtype");
    require(m >= 0 && n >= 0 && k >= 0, MIMW_ERR_SHAPE, "negative extent");
    require(m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31), MIMW_ERR_UNSUPPORTED, "extent >= 2^31");
    if (m == 0 || n == 0) return;
    if (k == 0) {  // C = 0 (oracles.cpp:19)
      require(c != nullptr, MIMW_ERR_ARG, "null pointer");
      require_sm100();
      const int64_t es = c_dtype == MIMW_F32 ? 4 : 2;
      check_cuda(cudaMemset2DAsync(c, ldc * es, 0, n * es, m, static_cast<cudaStream_t>(stream)), "memset");
      return;
    }
    require(a && b && c, MIMW_ERR_ARG, "null pointer");
    require(lda >= k && ldc >= n && ldb >= (b_layout == MIMW_B_KN ? n : k), MIMW_ERR_SHAPE,
            "leading dimension smaller than the row");
    require_pitch(a, lda, 2, "a");
    require_pitch(b, ldb, 2, "b");
    require_pitch(c, ldc, c_dtype == MIMW_F32 ? 4 : 2, "c");
    require_sm100();
    mimw::GemmArgs g{};
    g.a = a;
    g.b = b;
    g.c = c;
    g.m = m;
    g.n = n;
    g.k = k;
    g.lda = lda;
    g.ldb = ldb;
    g.ldc = ldc;
    g.b_kn = b_layout == MIMW_B_KN;
    g.c_f32 = c_dtype == MIMW_F32;
    g.cta_group = 2;
    check_cuda(mimw::gemm_bf16_launch(g, static_cast<cudaStream_t>(stream)), "gemm launch");
  });
}

// Tuning / test hook (not part of the public header): force cta_group and
// raster group.  Used by the parity tests to cover the 1-CTA variant.
int mimw_b200_gemm_bf16_ex(const void *a, const void *b, void *c, int64_t m, int64_t n, int64_t k,
                           int64_t lda, int64_t ldb, int64_t ldc, int32_t b_layout, int32_t c_dtype,
                           int32_t cta_group, int32_t raster_group, int32_t max_clusters,
                           void *stream) {
  return guarded([&] {
    require(cta_group == 1 || cta_group == 2, MIMW_ERR_ARG, "cta_group must be 1 or 2");
    if (m == 0 || n == 0) return;
    if (k == 0) {  // C = 0 (oracles.cpp:19)
      require(c != nullptr, MIMW_ERR_ARG, "null pointer");
      require_sm100();
      const int64_t es = c_dtype == MIMW_F32 ? 4 : 2;
      check_cuda(cudaMemset2DAsync(c, ldc * es, 0, n * es, m, static_cast<cudaStream_t>(stream)), "memset");
      return;
    }
    require(a && b && c, MIMW_ERR_ARG, "null pointer");
    require_pitch(a, lda, 2, "a");
    require_pitch(b, ldb, 2, "b");
    require_pitch(c, ldc, c_dtype == MIMW_F32 ? 4 : 2, "c");
    require_sm100();
    mimw::GemmArgs g{};
    g.a = a;
    g.b = b;
    g.c = c;
    g.m = m;
    g.n = n;
    g.k = k;
    g.lda = lda;
    g.ldb = ldb;
    g.ldc = ldc;
    g.b_kn = b_layout == MIMW_B_KN;
    g.c_f32 = c_dtype == MIMW_F32;
    g.cta_group = cta_group;
    g.raster_group = raster_group;
    g.max_clusters = max_clusters;
    check_cuda(mimw::gemm_bf16_launch(g, static_cast<cudaStream_t>(stream)), "gemm launch");
  });
}

}  // extern "C"
