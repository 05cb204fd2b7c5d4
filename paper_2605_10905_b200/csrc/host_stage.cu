// Host thread pool + pinned staging slots + f32 -> bf16 (RNE) row conversion
// for the PCIe-bound host-Tile entries (host_stage.h).
#include "host_stage.h"

#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace mimw {

namespace {

inline uint16_t bf16_rne(uint32_t u) {
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;  // NaN (the device conversion's canonical NaN)
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

__attribute__((target("avx2"))) inline __m256i cvt8_avx2(__m256i u) {
  const __m256i is_nan = _mm256_cmpgt_epi32(_mm256_and_si256(u, _mm256_set1_epi32(0x7fffffff)),
                                            _mm256_set1_epi32(0x7f800000));
  const __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(u, 16), _mm256_set1_epi32(1));
  const __m256i r = _mm256_srli_epi32(_mm256_add_epi32(_mm256_add_epi32(u, _mm256_set1_epi32(0x7fff)), lsb), 16);
  return _mm256_blendv_epi8(r, _mm256_set1_epi32(0x7fff), is_nan);
}

// 16 elements per iteration, streaming (non-temporal) 32-B stores into the
// pinned slot: no read-for-ownership of the destination lines, which the DMA
// engine reads next anyway
__attribute__((target("avx2"))) void convert_row_avx2(const float *src, int64_t n, uint16_t *dst) {
  const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
  int64_t j = 0;
  while (j < n && (reinterpret_cast<uintptr_t>(dst + j) & 31)) {
    dst[j] = bf16_rne(s[j]);
    ++j;
  }
  for (; j + 16 <= n; j += 16) {
    const __m256i a = cvt8_avx2(_mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + j)));
    const __m256i b = cvt8_avx2(_mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + j + 8)));
    // packus works per 128-bit lane: a0-3 b0-3 | a4-7 b4-7 -> reorder the 64-bit quarters
    const __m256i p = _mm256_permute4x64_epi64(_mm256_packus_epi32(a, b), 0xD8);
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + j), p);
  }
  for (; j < n; ++j) dst[j] = bf16_rne(s[j]);
}

void convert_row_generic(const float *src, int64_t n, uint16_t *dst) {
  const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
  for (int64_t j = 0; j < n; ++j) dst[j] = bf16_rne(s[j]);
}

class Pool {
 public:
  static Pool &get() {
    static Pool p;
    return p;
  }
  void run(int64_t n, const std::function<void(int64_t, int64_t)> &f) {
    const int parts = (int)std::min<int64_t>(n, (int64_t)workers_.size() + 1);
    if (parts <= 1) {
      if (n > 0) f(0, n);
      return;
    }
    std::unique_lock<std::mutex> lk(call_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      n_ = n;
      parts_ = parts;
      next_ = 1;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0, n / parts);  // the caller takes part 0
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    int want = (int)std::min(hw ? hw : 4u, 16u);
    if (const char *e = getenv("MIMW_HOST_THREADS")) want = std::max(1, atoi(e));  // A/B knob
    const int nt = want - 1;
    for (int i = 0; i < nt; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t, int64_t)> *job;
      int part;
      int64_t n;
      int parts;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || (gen_ != seen && job_ != nullptr && next_ < parts_); });
        if (stop_) return;
        part = next_++;
        if (next_ >= parts_) seen = gen_;
        job = job_;
        n = n_;
        parts = parts_;
      }
      (*job)(n * part / parts, n * (part + 1) / parts);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t, int64_t)> *job_ = nullptr;
  int64_t n_ = 0;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

void host_parallel_for(int64_t n, const std::function<void(int64_t, int64_t)> &f) { Pool::get().run(n, f); }

void host_rows_to_bf16(const float *src, int64_t ld_src, int64_t rows, int64_t cols, uint16_t *dst,
                       int64_t ld_dst, int64_t col_off) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  for (int64_t r = 0; r < rows; ++r) {
    if (avx2) convert_row_avx2(src + r * ld_src, cols, dst + r * ld_dst + col_off);
    else convert_row_generic(src + r * ld_src, cols, dst + r * ld_dst + col_off);
  }
  if (avx2) _mm_sfence();  // streaming stores ordered before the caller hands the slot to the DMA
}

// bf16 -> f32 widening (exact) of device results staged into a pinned slot
// (regular stores: streaming stores measured slower here, 46-48 vs 49-50
// TFLOP/s attention e2e)
__attribute__((target("avx2"))) static void widen_row_avx2(const uint16_t *src, int64_t n, float *dst) {
  int64_t j = 0;
  for (; j + 8 <= n; j += 8) {
    const __m256i w = _mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i *>(src + j)));
    _mm256_storeu_si256(reinterpret_cast<__m256i *>(dst + j), _mm256_slli_epi32(w, 16));
  }
  for (; j < n; ++j) {
    const uint32_t u = (uint32_t)src[j] << 16;
    std::memcpy(dst + j, &u, 4);
  }
}

void host_rows_bf16_to_f32(const uint16_t *src, int64_t ld_src, int64_t rows, int64_t cols, float *dst,
                           int64_t ld_dst) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  for (int64_t r = 0; r < rows; ++r) {
    if (avx2) {
      widen_row_avx2(src + r * ld_src, cols, dst + r * ld_dst);
    } else {
      for (int64_t j = 0; j < cols; ++j) {
        const uint32_t u = (uint32_t)src[r * ld_src + j] << 16;
        std::memcpy(dst + r * ld_dst + j, &u, 4);
      }
    }
  }
}

// streaming (non-temporal) stores into the caller's buffer: no read for
// ownership of lines that are only written (host memory bandwidth limits the
// pageable e2e path: 67 -> 78-80 TFLOP/s GEMM e2e)
__attribute__((target("avx2"))) static void copy_f32_avx2(const float *src, int64_t n, float *dst) {
  int64_t j = 0;
  while (j < n && (reinterpret_cast<uintptr_t>(dst + j) & 31)) {
    dst[j] = src[j];
    ++j;
  }
  for (; j + 16 <= n; j += 16) {
    const __m256 a = _mm256_loadu_ps(src + j);
    const __m256 b = _mm256_loadu_ps(src + j + 8);
    _mm256_stream_ps(dst + j, a);
    _mm256_stream_ps(dst + j + 8, b);
  }
  for (; j < n; ++j) dst[j] = src[j];
}

void host_copy_f32(float *dst, const float *src, int64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (!avx2) {
    std::memcpy(dst, src, sizeof(float) * (size_t)n);
    return;
  }
  copy_f32_avx2(src, n, dst);
  _mm_sfence();
}

namespace {
// per calling thread: concurrent host entries (the reference's oracles are
// pure functions, safe to call from several threads) never share a buffer
struct PinnedSlots {
  std::vector<std::pair<void *, size_t>> v;
  ~PinnedSlots() {
    for (auto &s : v)
      if (s.first) cudaFreeHost(s.first);
  }
};
}  // namespace

void *pinned_slot(int slot, size_t bytes) {
  thread_local PinnedSlots slots;
  if ((int)slots.v.size() <= slot) slots.v.resize((size_t)slot + 1, {nullptr, 0});
  auto &s = slots.v[(size_t)slot];
  if (s.second < bytes) {
    if (s.first) cudaFreeHost(s.first);
    s.first = nullptr;
    s.second = 0;
    if (cudaHostAlloc(&s.first, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    s.second = bytes;
  }
  return s.first;
}

}  // namespace mimw
