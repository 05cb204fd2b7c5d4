// extern "C" boundary of libmimw_b200.so (declared in include/mimw_b200.h).
//
// Each mimw_b200_oracle_* entry replaces one function of the reference's
// operator API, proj/core/include/mimw/oracles.hpp, with the same argument
// meaning (row-major f32 host Tiles).  The mimw_b200_* device entries are the
// production path.  No exception crosses the ABI; no CPU fallback exists.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mimw_b200.h"
#include "attention_x3.h"
#include "convert.h"
#include "pool.h"
#include "host_stage.h"
#include "attention_fwd.h"
#include "attention_bwd.h"
#include "attention_f32.h"
#include "gemm_bf16.h"
#ifdef MIMW_TILE_TRACE
namespace mimw { cudaError_t set_tile_trace(void *buf); }
#endif
#include "gemm_mxfp8.h"
#include "layernorm_cluster.h"
#include "simplicial_fwd.h"

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

// RAII CUDA event (timing disabled).
struct Event {
  cudaEvent_t e = nullptr;
  Event() { check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create"); }
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  Event(const Event &) = delete;
  Event &operator=(const Event &) = delete;
  Event(Event &&o) noexcept : e(o.e) { o.e = nullptr; }
};

// Per-thread, per-device copy streams for the pipelined host-buffer entries,
// destroyed when the thread exits.
struct SideStreams {
  cudaStream_t st[64][2] = {};
  ~SideStreams() {
    int cur = -1;
    cudaGetDevice(&cur);
    for (int d = 0; d < 64; ++d)
      if (st[d][0] || st[d][1]) {
        cudaSetDevice(d);
        for (auto &x : st[d])
          if (x) cudaStreamDestroy(x);
      }
    if (cur >= 0) cudaSetDevice(cur);
  }
};

cudaStream_t side_stream(int which) {
  thread_local SideStreams ss;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!ss.st[dev][which])
    check_cuda(cudaStreamCreateWithFlags(&ss.st[dev][which], cudaStreamNonBlocking), "stream create");
  return ss.st[dev][which];
}

// RAII device scratch on a stream.
struct DevBuf {
  void *p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) check_cuda(mimw::scratch_alloc(&p, bytes, s), "scratch allocation (private pool)");
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T *as() const { return static_cast<T *>(p); }
};

// Synchronizes the side streams when a host entry unwinds on an error, before
// its DevBufs (declared earlier, destroyed later) free device scratch that an
// in-flight copy on cs / ds may still touch, and before the thread's pinned
// slots can be refilled by the next call.
struct UnwindSync {
  cudaStream_t st[3];
  int n0;
  UnwindSync(cudaStream_t a, cudaStream_t b, cudaStream_t c) : st{a, b, c}, n0(std::uncaught_exceptions()) {}
  ~UnwindSync() {
    if (std::uncaught_exceptions() > n0)
      for (auto x : st) cudaStreamSynchronize(x);
  }
};

// MIMW_PREC_BF16 path of host_gemm with the f32 -> bf16 rounding done on the
// host threads (host_stage.h) straight into the device layout in pinned
// slots: PCIe carries 2 bytes per input element instead of 4, and the
// conversion of chunk i+1 overlaps the DMA of chunk i.  Same bf16 values as
// the device staging kernels, so the results are bit-identical.
// A host pointer the DMA engines can use directly (pinned / registered /
// managed)?  Pageable memory (a std::vector Tile, a numpy array) is instead
// read and written by the host threads through pinned slots.
static bool dma_capable(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type != cudaMemoryTypeUnregistered;
}

static void host_gemm_host_staged(const std::vector<const float *> &a_parts,
                                  const std::vector<const float *> &b_parts, const std::vector<int64_t> &k_parts,
                                  int64_t m, int64_t n, int64_t k, float *c, cudaStream_t s, cudaStream_t cs,
                                  cudaStream_t ds, int mode, bool c_pageable) {
  // mode 1: every chunk rounded on the host; 2: B's odd row chunks (and all of
  // A) go over PCIe as f32 and are rounded by the device staging kernels, so
  // the host threads and the H2D stream share B's transfer; 3: also A's odd
  // chunks on the host
  const int64_t kp = round_up(k, 8);
  const int64_t np = round_up(n, 8);
  DevBuf dA(2 * m * kp, s), dB(2 * kp * np, s), dC(sizeof(float) * m * np, s);
  DevBuf dF(mode == 1 ? 0 : sizeof(float) * (m + n) * k, s);  // f32 landing for device-rounded chunks
  UnwindSync guard(s, cs, ds);
  float *dFb = dF.as<float>(), *dFa = dF.as<float>() ? dF.as<float>() + (size_t)k * n : nullptr;
  Event e_alloc, e_b;
  check_cuda(cudaEventRecord(e_alloc.e, s), "event");
  check_cuda(cudaStreamWaitEvent(cs, e_alloc.e, 0), "wait");
  check_cuda(cudaStreamWaitEvent(ds, e_alloc.e, 0), "wait");
  std::vector<int64_t> koff(a_parts.size());
  for (size_t i = 0, o = 0; i < a_parts.size(); o += k_parts[i], ++i) koff[i] = (int64_t)o;
  std::vector<int> part_of_row((size_t)k);
  for (size_t i = 0; i < a_parts.size(); ++i)
    for (int64_t r = 0; r < k_parts[i]; ++r) part_of_row[(size_t)(koff[i] + r)] = (int)i;

  const int64_t bchunk = std::max<int64_t>(64, round_up((k + 7) / 8, 8));
  const int64_t achunk = std::max<int64_t>(512, round_up((m + 7) / 8, 256));
  const size_t slot_bytes = (size_t)std::max(bchunk * np, achunk * kp) * 2;
  constexpr int NSLOT = 3;
  Event slot_ev[NSLOT];
  bool slot_used[NSLOT] = {false, false, false};
  int slot = 0;
  // fill a pinned slot on the host threads, then DMA it to dst on cs
  auto stage = [&](int64_t rows, const std::function<void(int64_t, uint16_t *)> &fill_row, int64_t pitch,
                   void *dst) {
    if (slot_used[slot]) check_cuda(cudaEventSynchronize(slot_ev[slot].e), "pinned slot reuse");
    uint16_t *h = static_cast<uint16_t *>(mimw::pinned_slot(slot, slot_bytes));
    require(h != nullptr, MIMW_ERR_CUDA, "cudaHostAlloc failed");
    mimw::host_parallel_for(rows, [&](int64_t lo, int64_t hi) {
      for (int64_t r = lo; r < hi; ++r) fill_row(r, h + r * pitch);
    });
    check_cuda(cudaMemcpyAsync(dst, h, (size_t)rows * pitch * 2, cudaMemcpyHostToDevice, cs), "H2D");
    check_cuda(cudaEventRecord(slot_ev[slot].e, cs), "event");
    slot_used[slot] = true;
    slot = (slot + 1) % NSLOT;
  };
  // B rows (every part stacked along K), zero columns [n, np); zero rows [k, kp)
  if (kp > k)
    check_cuda(cudaMemsetAsync(static_cast<char *>(dB.p) + (size_t)k * np * 2, 0, (size_t)(kp - k) * np * 2, cs),
               "memset");
  for (int64_t r0 = 0, bi = 0; r0 < k; r0 += bchunk, ++bi) {
    const int64_t rows = std::min(bchunk, k - r0);
    if (mode != 1 && (bi & 1)) {
      // f32 over PCIe, rounded by the device staging kernel (per K part)
      for (size_t i = 0; i < b_parts.size(); ++i) {
        const int64_t lo = std::max(r0, koff[i]), hi = std::min(r0 + rows, koff[i] + k_parts[i]);
        if (hi <= lo) continue;
        float *land = dFb + lo * n;
        check_cuda(cudaMemcpyAsync(land, b_parts[i] + (lo - koff[i]) * n, sizeof(float) * (hi - lo) * n,
                                   cudaMemcpyHostToDevice, cs), "H2D b");
        Event e;
        check_cuda(cudaEventRecord(e.e, cs), "event");
        check_cuda(cudaStreamWaitEvent(s, e.e, 0), "wait");
        mimw::stage_rows_bf16(land, hi - lo, hi - lo, n, np, dB.p, np, lo, 0, s);
      }
      continue;
    }
    stage(rows, [&](int64_t r, uint16_t *dst) {
      const int64_t kr = r0 + r;
      const int i = part_of_row[(size_t)kr];
      mimw::host_rows_to_bf16(b_parts[(size_t)i] + (kr - koff[(size_t)i]) * n, n, 1, n, dst, np, 0);
      if (np > n) std::memset(dst + n, 0, (size_t)(np - n) * 2);
    }, np, static_cast<char *>(dB.p) + (size_t)r0 * np * 2);
  }
  check_cuda(cudaEventRecord(e_b.e, cs), "event");
  check_cuda(cudaStreamWaitEvent(s, e_b.e, 0), "wait");
  const int nchunks = (int)((m + achunk - 1) / achunk);
  std::vector<Event> e_a(nchunks), e_c(nchunks), e_d(c_pageable ? nchunks : 0);
  auto drain = [&](int ci) {
    const int64_t r0 = ci * achunk, rows = std::min(achunk, m - r0);
    check_cuda(cudaEventSynchronize(e_d[ci].e), "gemm execution");
    const float *hc = static_cast<const float *>(mimw::pinned_slot(7 + (ci & 1), (size_t)achunk * n * 4));
    mimw::host_parallel_for(rows, [&](int64_t lo, int64_t hi) {
      mimw::host_copy_f32(c + (r0 + lo) * n, hc + lo * n, (hi - lo) * n);
    });
  };
  for (int ci = 0; ci < nchunks; ++ci) {
    const int64_t r0 = ci * achunk, rows = std::min(achunk, m - r0);
    char *dA_rows = static_cast<char *>(dA.p) + (size_t)r0 * kp * 2;
    if (mode == 2 || (mode == 3 && (ci & 1))) {
      // f32 over PCIe, rounded by the device staging kernel (per K part)
      for (size_t i = 0; i < a_parts.size(); ++i)
        if (k_parts[i])
          check_cuda(cudaMemcpyAsync(dFa + r0 * k + koff[i] * rows, a_parts[i] + r0 * k_parts[i],
                                     sizeof(float) * rows * k_parts[i], cudaMemcpyHostToDevice, cs),
                     "H2D a");
      check_cuda(cudaEventRecord(e_a[ci].e, cs), "event");
      check_cuda(cudaStreamWaitEvent(s, e_a[ci].e, 0), "wait");
      for (size_t i = 0; i < a_parts.size(); ++i) {
        const int64_t ki = k_parts[i];
        if (ki == 0) continue;
        const bool last = koff[i] + ki == k;
        mimw::stage_cols_bf16(dFa + r0 * k + koff[i] * rows, rows, ki, last ? (kp - koff[i]) : ki, dA_rows, kp,
                              koff[i], 0, s);
      }
    } else {
      stage(rows, [&](int64_t r, uint16_t *dst) {
        for (size_t i = 0; i < a_parts.size(); ++i)
          if (k_parts[i])
            mimw::host_rows_to_bf16(a_parts[i] + (r0 + r) * k_parts[i], k_parts[i], 1, k_parts[i], dst, kp,
                                    koff[i]);
        if (kp > k) std::memset(dst + k, 0, (size_t)(kp - k) * 2);
      }, kp, dA_rows);
      check_cuda(cudaEventRecord(e_a[ci].e, cs), "event");
      check_cuda(cudaStreamWaitEvent(s, e_a[ci].e, 0), "wait");
    }
    mimw::GemmArgs g{};
    g.a = dA_rows;
    g.b = dB.p;
    g.c = static_cast<char *>(dC.p) + (size_t)r0 * np * 4;
    g.m = rows;
    g.n = np;
    g.k = kp;
    g.lda = kp;
    g.ldb = np;
    g.ldc = np;
    g.b_kn = true;
    g.c_f32 = true;
    g.cta_group = 2;
    check_cuda(mimw::gemm_bf16_launch(g, s), "gemm launch");
    check_cuda(cudaEventRecord(e_c[ci].e, s), "event");
    check_cuda(cudaStreamWaitEvent(ds, e_c[ci].e, 0), "wait");
    if (!c_pageable) {
      check_cuda(cudaMemcpy2DAsync(c + r0 * n, sizeof(float) * n, static_cast<char *>(dC.p) + (size_t)r0 * np * 4,
                                   sizeof(float) * np, sizeof(float) * n, rows, cudaMemcpyDeviceToHost, ds),
                 "D2H c");
      continue;
    }
    // pageable C: D2H into a pinned slot, copied out by the host threads one
    // chunk behind (the slot of chunk ci - 2 was drained in iteration ci - 1)
    float *hc = static_cast<float *>(mimw::pinned_slot(7 + (ci & 1), (size_t)achunk * n * 4));
    require(hc != nullptr, MIMW_ERR_CUDA, "cudaHostAlloc failed");
    check_cuda(cudaMemcpy2DAsync(hc, sizeof(float) * n, static_cast<char *>(dC.p) + (size_t)r0 * np * 4,
                                 sizeof(float) * np, sizeof(float) * n, rows, cudaMemcpyDeviceToHost, ds),
               "D2H c");
    check_cuda(cudaEventRecord(e_d[ci].e, ds), "event");
    if (ci >= 1) drain(ci - 1);
  }
  if (c_pageable && nchunks > 0) drain(nchunks - 1);
  check_cuda(cudaStreamSynchronize(ds), "gemm execution");
  check_cuda(cudaStreamSynchronize(cs), "gemm execution");
  check_cuda(cudaStreamSynchronize(s), "gemm execution");
}

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

  // Pipelined over row chunks of A/C on three streams: H2D copies (cs),
  // staging + GEMM (s), D2H copies (ds), so PCIe traffic in both directions
  // overlaps the tensor-core work (the host-f32 Tile path is PCIe-bound).
  cudaStream_t s = cudaStreamPerThread;
  cudaStream_t cs = side_stream(0), ds = side_stream(1);
  const int nseg = precision == MIMW_PREC_F32_BF16X3 ? 3 : 1;
  static const int host_stage = getenv("MIMW_HOST_STAGE") ? atoi(getenv("MIMW_HOST_STAGE")) : 3;  // A/B knob (mode 3 9.9-10.0 ms vs device staging 11.2)
  if (nseg == 1 && host_stage) {
    // pageable inputs: every chunk is rounded by the host threads (mode 1), so
    // no cudaMemcpyAsync ever reads pageable memory (the driver would stage it
    // synchronously at a fraction of the PCIe rate); pageable C: D2H through
    // pinned slots
    bool in_pageable = false;
    for (size_t i = 0; i < a_parts.size(); ++i)
      if (k_parts[i]) in_pageable |= !dma_capable(a_parts[i]) || !dma_capable(b_parts[i]);
    host_gemm_host_staged(a_parts, b_parts, k_parts, m, n, k, c, s, cs, ds, in_pageable ? 1 : host_stage,
                          !dma_capable(c));
    return;
  }
  const int64_t kp = round_up(k, 8);  // bf16 row pitch multiple of 16 B
  const int64_t np = round_up(n, 8);
  const int64_t kt = nseg * kp;
  size_t in_elems = 0;
  for (size_t i = 0; i < a_parts.size(); ++i) in_elems += (m + n) * k_parts[i];
  DevBuf din(sizeof(float) * in_elems, s);
  DevBuf dA(2 * m * kt, s), dB(2 * kt * np, s), dC(sizeof(float) * m * np, s);
  UnwindSync guard(s, cs, ds);
  Event e_alloc, e_b;
  check_cuda(cudaEventRecord(e_alloc.e, s), "event");
  check_cuda(cudaStreamWaitEvent(cs, e_alloc.e, 0), "wait");
  check_cuda(cudaStreamWaitEvent(ds, e_alloc.e, 0), "wait");

  // segment products: (A part, B part) for hi.hi [, hi.lo, lo.hi]
  const int a_part_of_seg[3] = {0, 0, 1};
  const int b_part_of_seg[3] = {0, 1, 0};
  std::vector<float *> da(a_parts.size()), db(a_parts.size());
  {
    float *cursor = din.as<float>();
    for (size_t i = 0; i < a_parts.size(); ++i) {
      da[i] = cursor;
      db[i] = cursor + m * k_parts[i];
      cursor += (m + n) * k_parts[i];
    }
  }
  // B (every part) first: all chunks need it
  for (size_t i = 0; i < a_parts.size(); ++i)
    if (k_parts[i])
      check_cuda(cudaMemcpyAsync(db[i], b_parts[i], sizeof(float) * k_parts[i] * n,
                                 cudaMemcpyHostToDevice, cs), "H2D b");
  check_cuda(cudaEventRecord(e_b.e, cs), "event");
  check_cuda(cudaStreamWaitEvent(s, e_b.e, 0), "wait");
  {
    int64_t koff = 0;
    for (size_t i = 0; i < a_parts.size(); ++i) {
      const int64_t ki = k_parts[i];
      if (ki == 0) continue;
      const bool last = (i + 1 == a_parts.size()) || (koff + ki == k);
      const int64_t pad = last ? (kp - koff) : ki;  // the last part zero-fills the K padding
      for (int sgi = 0; sgi < nseg; ++sgi)
        mimw::stage_rows_bf16(db[i], ki, pad, n, np, dB.p, np, sgi * kp + koff, b_part_of_seg[sgi], s);
      koff += ki;
    }
  }
  const int64_t chunk = std::max<int64_t>(512, round_up((m + 7) / 8, 256));
  const int nchunks = (int)((m + chunk - 1) / chunk);
  std::vector<Event> e_a(nchunks), e_c(nchunks);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int64_t r0 = ci * chunk, rows = std::min(chunk, m - r0);
    for (size_t i = 0; i < a_parts.size(); ++i)
      if (k_parts[i])
        check_cuda(cudaMemcpyAsync(da[i] + r0 * k_parts[i], a_parts[i] + r0 * k_parts[i],
                                   sizeof(float) * rows * k_parts[i], cudaMemcpyHostToDevice, cs),
                   "H2D a");
    check_cuda(cudaEventRecord(e_a[ci].e, cs), "event");
    check_cuda(cudaStreamWaitEvent(s, e_a[ci].e, 0), "wait");
    char *dA_rows = static_cast<char *>(dA.p) + (size_t)r0 * kt * 2;
    int64_t koff = 0;
    for (size_t i = 0; i < a_parts.size(); ++i) {
      const int64_t ki = k_parts[i];
      if (ki == 0) continue;
      const bool last = (i + 1 == a_parts.size()) || (koff + ki == k);
      const int64_t pad = last ? (kp - koff) : ki;
      for (int sgi = 0; sgi < nseg; ++sgi)
        mimw::stage_cols_bf16(da[i] + r0 * ki, rows, ki, pad, dA_rows, kt, sgi * kp + koff,
                              a_part_of_seg[sgi], s);
      koff += ki;
    }
    check_cuda(cudaGetLastError(), "staging kernels");
    mimw::GemmArgs g{};
    g.a = dA_rows;
    g.b = dB.p;
    g.c = static_cast<char *>(dC.p) + (size_t)r0 * np * 4;
    g.m = rows;
    g.n = np;
    g.k = kt;
    g.lda = kt;
    g.ldb = np;
    g.ldc = np;
    g.b_kn = true;
    g.c_f32 = true;
    g.cta_group = 2;
    check_cuda(mimw::gemm_bf16_launch(g, s), "gemm launch");
    check_cuda(cudaEventRecord(e_c[ci].e, s), "event");
    check_cuda(cudaStreamWaitEvent(ds, e_c[ci].e, 0), "wait");
    check_cuda(cudaMemcpy2DAsync(c + r0 * n, sizeof(float) * n, static_cast<char *>(dC.p) + (size_t)r0 * np * 4,
                                 sizeof(float) * np, sizeof(float) * n, rows, cudaMemcpyDeviceToHost, ds),
               "D2H c");
  }
  check_cuda(cudaStreamSynchronize(ds), "gemm execution");
  check_cuda(cudaStreamSynchronize(cs), "gemm execution");
  check_cuda(cudaStreamSynchronize(s), "gemm execution");
}



// MIMW_PREC_F32 for the host attention Tiles: the oracles' f64 score /
// softmax arithmetic on CUDA cores (attention_f32.cu), for callers that hold
// the reference's own tolerances.
void host_attention_f32(const float *const *inputs, int n_inputs, float *o, float *lse, int64_t seq,
                        int64_t d, int64_t w1, int64_t w2, bool simplicial, double scale) {
  cudaStream_t s = cudaStreamPerThread;
  const int64_t n = seq * d;
  DevBuf din(sizeof(float) * (n_inputs * n + seq + n), s);
  float *f = din.as<float>();
  for (int t = 0; t < n_inputs; ++t)
    check_cuda(cudaMemcpyAsync(f + t * n, inputs[t], sizeof(float) * n, cudaMemcpyHostToDevice, s), "H2D");
  float *dout = f + n_inputs * n, *dlse = dout + n;
  mimw::AttnF32Args a{};
  a.q = f;
  a.k1 = f + n;
  a.v1 = f + 2 * n;
  a.k2 = simplicial ? f + 3 * n : nullptr;
  a.v2 = simplicial ? f + 4 * n : nullptr;
  a.o = dout;
  a.lse = dlse;
  a.seq = seq;
  a.d = d;
  a.w1 = w1;
  a.w2 = w2;
  a.causal = true;
  a.simplicial = simplicial;
  a.scale = scale;
  check_cuda(mimw::attention_f32_launch(a, s), "attention f32 launch");
  check_cuda(cudaMemcpyAsync(o, dout, sizeof(float) * n, cudaMemcpyDeviceToHost, s), "D2H o");
  if (lse) check_cuda(cudaMemcpyAsync(lse, dlse, sizeof(float) * seq, cudaMemcpyDeviceToHost, s), "D2H lse");
  check_cuda(cudaStreamSynchronize(s), "attention f32 execution");
}

// oracle_attention (oracles.cpp:119-145) at MIMW_PREC_F32_BF16X3: split-bf16 x3
// on the tcgen05 GEMM (attention_x3.cu), one head at a time.
void host_attention_x3(const float *q, const float *k, const float *v, float *o, float *lse, int64_t heads,
                       int64_t seq, int64_t d, int64_t w, double scale) {
  cudaStream_t s = cudaStreamPerThread;
  const int64_t n = seq * d;
  DevBuf din(sizeof(float) * (4 * n + seq), s);
  DevBuf dws(mimw::attention_x3_workspace_bytes(seq, d), s);
  float *f = din.as<float>();
  for (int64_t h = 0; h < heads; ++h) {
    const float *src[3] = {q + h * n, k + h * n, v + h * n};
    for (int t = 0; t < 3; ++t)
      check_cuda(cudaMemcpyAsync(f + t * n, src[t], sizeof(float) * n, cudaMemcpyHostToDevice, s), "H2D");
    mimw::AttnX3Args a{};
    a.q = f;
    a.k = f + n;
    a.v = f + 2 * n;
    a.o = f + 3 * n;
    a.lse = f + 4 * n;
    a.seq = seq;
    a.d = d;
    a.w = w;
    a.scale = scale;
    a.workspace = dws.p;
    check_cuda(mimw::attention_x3_launch(a, s), "attention x3 launch");
    check_cuda(cudaMemcpyAsync(o + h * n, a.o, sizeof(float) * n, cudaMemcpyDeviceToHost, s), "D2H o");
    if (lse)
      check_cuda(cudaMemcpyAsync(lse + h * seq, a.lse, sizeof(float) * seq, cudaMemcpyDeviceToHost, s), "D2H lse");
    check_cuda(cudaStreamSynchronize(s), "attention x3 execution");  // the next head reuses f
  }
}

// oracle_attention (oracles.cpp:119-145) for `heads` independent [seq, d]
// heads of host f32 Tiles stored back to back ([heads, seq, d]); heads == 1
// is exactly the reference signature.  Head dim zero-padded to 128 (exact:
// padded q/k columns add 0 to every score, padded v columns give 0 outputs).
// Pipelined over chunks of heads on three streams, with the f32 <-> bf16
// conversions on the host threads into pinned slots, so PCIe carries 2 bytes
// per element in both directions and pageable caller buffers (the reference's
// Tile is a std::vector, sim.hpp:13-26) are read and written by the host
// threads at memory speed instead of through the driver's pageable staging:
//   host: round chunk c -> slot   cs: H2D c   s: FA c   ds: D2H O_c (bf16), lse_c
//   host: widen O_(c-1) -> o (exact)
void host_attention_heads(const float *q, const float *k, const float *v, float *o, float *lse,
                          int64_t heads, int64_t seq, int64_t d, int64_t w, double scale,
                          int precision = MIMW_PREC_BF16) {
  require(precision == MIMW_PREC_BF16 || precision == MIMW_PREC_F32 || precision == MIMW_PREC_F32_BF16X3,
          MIMW_ERR_ARG, "precision must be MIMW_PREC_BF16, MIMW_PREC_F32 or MIMW_PREC_F32_BF16X3");
  require(heads >= 0 && seq >= 0 && d >= 0, MIMW_ERR_SHAPE, "negative extent");
  require(d <= 128, MIMW_ERR_UNSUPPORTED, "head dim > 128 not supported");
  require(w >= 1 || seq == 0 || heads == 0, MIMW_ERR_ARG, "window must be >= 1");
  require(seq < (1ll << 31) && heads * ((seq + 255) / 256) < (1ll << 31), MIMW_ERR_UNSUPPORTED,
          "extent too large");
  if (heads == 0 || seq == 0) return;
  if (d == 0) {
    if (lse)
      for (int64_t h = 0; h < heads; ++h)
        for (int64_t i = 0; i < seq; ++i) lse[h * seq + i] = std::log((float)std::min<int64_t>(w, i + 1));
    return;
  }
  require(q && k && v && o, MIMW_ERR_ARG, "null pointer");
  require_sm100();
  if (precision == MIMW_PREC_F32) {
    for (int64_t h = 0; h < heads; ++h) {
      const float *in[3] = {q + h * seq * d, k + h * seq * d, v + h * seq * d};
      host_attention_f32(in, 3, o + h * seq * d, lse ? lse + h * seq : nullptr, seq, d, w, 1, false, scale);
    }
    return;
  }
  if (precision == MIMW_PREC_F32_BF16X3) {
    host_attention_x3(q, k, v, o, lse, heads, seq, d, w, scale);
    return;
  }
  cudaStream_t s = cudaStreamPerThread, cs = side_stream(0), ds = side_stream(1);
  const int64_t he = seq * 128;  // padded elements per head and tensor
  const int64_t ch = std::max<int64_t>(1, std::min<int64_t>(heads, (32ll << 20) / (3 * he * 2)));
  const int64_t nchunks = (heads + ch - 1) / ch;
  const size_t in_bytes = (size_t)3 * ch * he * 2, o_bytes = (size_t)ch * he * 2;
  const size_t out_bytes = o_bytes + (size_t)ch * seq * 4;
  DevBuf din(2 * in_bytes, s), dout(2 * out_bytes, s);
  UnwindSync guard(s, cs, ds);
  Event ev_alloc, ev_in[2], ev_fa[2], ev_out[2];
  bool used[2] = {false, false};
  check_cuda(cudaEventRecord(ev_alloc.e, s), "event");
  check_cuda(cudaStreamWaitEvent(cs, ev_alloc.e, 0), "wait");
  check_cuda(cudaStreamWaitEvent(ds, ev_alloc.e, 0), "wait");
  auto widen = [&](int64_t c) {
    const int b = (int)(c & 1);
    const int64_t h0 = c * ch, nh = std::min(ch, heads - h0);
    check_cuda(cudaEventSynchronize(ev_out[b].e), "attention execution");
    const uint16_t *ho = static_cast<const uint16_t *>(mimw::pinned_slot(5 + b, out_bytes));
    mimw::host_parallel_for(nh * seq, [&](int64_t lo, int64_t hi) {
      mimw::host_rows_bf16_to_f32(ho + lo * 128, 128, hi - lo, d, o + (h0 * seq + lo) * d, d);
    });
    if (lse) std::memcpy(lse + h0 * seq, reinterpret_cast<const char *>(ho) + o_bytes, (size_t)nh * seq * 4);
  };
  for (int64_t c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    const int64_t h0 = c * ch, nh = std::min(ch, heads - h0);
    if (used[b]) check_cuda(cudaEventSynchronize(ev_in[b].e), "pinned slot reuse");  // H2D of c-2 done
    uint16_t *hin = static_cast<uint16_t *>(mimw::pinned_slot(3 + b, in_bytes));
    uint16_t *hout = static_cast<uint16_t *>(mimw::pinned_slot(5 + b, out_bytes));
    require(hin != nullptr && hout != nullptr, MIMW_ERR_CUDA, "cudaHostAlloc failed");
    const float *src3[3] = {q, k, v};
    mimw::host_parallel_for(3 * nh * seq, [&](int64_t lo, int64_t hi) {
      for (int64_t r = lo; r < hi; ++r) {
        const int64_t t = r / (nh * seq), rr = r - t * nh * seq;
        uint16_t *dst = hin + t * ch * he + rr * 128;
        mimw::host_rows_to_bf16(src3[t] + (h0 * seq + rr) * d, d, 1, d, dst, 128, 0);
        if (d < 128) std::memset(dst + d, 0, (size_t)(128 - d) * 2);
      }
    });
    uint16_t *dq = din.as<uint16_t>() + (size_t)b * 3 * ch * he;
    if (used[b]) check_cuda(cudaStreamWaitEvent(cs, ev_fa[b].e, 0), "wait");  // FA of c-2 read its inputs
    for (int t = 0; t < 3; ++t)
      check_cuda(cudaMemcpyAsync(dq + t * ch * he, hin + t * ch * he, (size_t)nh * he * 2, cudaMemcpyHostToDevice, cs),
                 "H2D q/k/v");
    check_cuda(cudaEventRecord(ev_in[b].e, cs), "event");
    check_cuda(cudaStreamWaitEvent(s, ev_in[b].e, 0), "wait");
    char *dob = static_cast<char *>(dout.p) + (size_t)b * out_bytes;
    if (used[b]) check_cuda(cudaStreamWaitEvent(s, ev_out[b].e, 0), "wait");  // D2H of c-2 read its outputs
    mimw::AttnArgs a{};
    a.q = dq;
    a.k = dq + ch * he;
    a.v = dq + 2 * ch * he;
    a.o = dob;
    a.lse = reinterpret_cast<float *>(dob + o_bytes);
    a.batch = 1;
    a.heads = nh;
    a.seq = seq;
    a.window = w;
    a.scale = scale;
    check_cuda(mimw::attention_fwd_launch(a, s), "attention launch");
    check_cuda(cudaEventRecord(ev_fa[b].e, s), "event");
    check_cuda(cudaStreamWaitEvent(ds, ev_fa[b].e, 0), "wait");
    check_cuda(cudaMemcpyAsync(hout, dob, (size_t)nh * he * 2, cudaMemcpyDeviceToHost, ds), "D2H o");
    if (lse)
      check_cuda(cudaMemcpyAsync(reinterpret_cast<char *>(hout) + o_bytes, dob + o_bytes, (size_t)nh * seq * 4,
                                 cudaMemcpyDeviceToHost, ds), "D2H lse");
    check_cuda(cudaEventRecord(ev_out[b].e, ds), "event");
    used[b] = true;
    if (c >= 1) widen(c - 1);
  }
  widen(nchunks - 1);
  check_cuda(cudaStreamSynchronize(cs), "attention execution");
  check_cuda(cudaStreamSynchronize(s), "attention execution");
}

void host_attention(const float *q, const float *k, const float *v, float *o, float *lse,
                    int64_t seq, int64_t d, int64_t w, double scale, int precision = MIMW_PREC_BF16) {
  host_attention_heads(q, k, v, o, lse, 1, seq, d, w, scale, precision);
}

void grouped_gemm(const void *x, const int64_t *m_offsets, const void *w, void *y, int64_t n_groups,
                  int64_t n, int64_t k, int32_t w_layout, int cta_group, int max_clusters,
                  int swap_tails, int tile_n, cudaStream_t stream) {
  require(w_layout == MIMW_B_KN || w_layout == MIMW_B_NK, MIMW_ERR_ARG, "bad w_layout");
  require(cta_group == 1 || cta_group == 2, MIMW_ERR_ARG, "cta_group must be 1 or 2");
  require(tile_n == 0 || tile_n == 256 || (tile_n == 512 && cta_group == 2), MIMW_ERR_ARG,
          "tile_n must be 0 (auto), 256, or 512 (cta_group 2)");
  require(n_groups >= 0 && n >= 0 && k >= 0, MIMW_ERR_SHAPE, "negative extent");
  if (n_groups == 0 || n == 0) return;
  require(m_offsets != nullptr, MIMW_ERR_ARG, "null m_offsets");
  require(m_offsets[0] >= 0, MIMW_ERR_SHAPE, "m_offsets[0] < 0");
  for (int64_t e = 0; e < n_groups; ++e)
    require(m_offsets[e + 1] >= m_offsets[e], MIMW_ERR_SHAPE, "m_offsets must be non-decreasing");
  require(m_offsets[n_groups] < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31),
          MIMW_ERR_UNSUPPORTED, "extent >= 2^31");
  if (m_offsets[n_groups] == m_offsets[0]) return;
  require(y != nullptr && (k == 0 || (x && w)), MIMW_ERR_ARG, "null pointer");
  require(n % 8 == 0 && k % 8 == 0, MIMW_ERR_UNSUPPORTED,
          "grouped GEMM needs n and k multiples of 8 (16-byte TMA row pitch)");
  require((((uintptr_t)x | (uintptr_t)w | (uintptr_t)y) & 15) == 0, MIMW_ERR_UNSUPPORTED,
          "tensors must be 16-byte aligned");
  require_sm100();
  mimw::GroupedGemmArgs g{};
  g.x = x;
  g.m_offsets = m_offsets;
  g.w = w;
  g.y = y;
  g.n_groups = n_groups;
  g.n = n;
  g.k = k;
  g.w_kn = w_layout == MIMW_B_KN;
  g.cta_group = cta_group;
  g.max_clusters = max_clusters;
  g.swap_tails = swap_tails;
  g.tile_n = tile_n;
  check_cuda(mimw::grouped_gemm_bf16_launch(g, stream), "grouped gemm launch");
}

void layernorm_checks(const void *x, const void *w, const void *b, const void *y, int64_t rows,
                      int64_t n) {
  require(rows >= 0 && n >= 0, MIMW_ERR_SHAPE, "negative extent");
  require(n <= 16 * 16 * 1024, MIMW_ERR_UNSUPPORTED, "row length > 262144 not supported");
  require(rows < (1ll << 31), MIMW_ERR_UNSUPPORTED, "rows >= 2^31");
  if (rows == 0 || n == 0) return;
  require(x && w && b && y, MIMW_ERR_ARG, "null pointer");
}

// oracle_simplicial_attention (oracles.cpp:82-117) for one [seq, d] head of
// host f32 Tiles; d <= 128 zero-padded to 128 (exact, as host_attention).
void host_simplicial(const float *q, const float *k1, const float *v1, const float *k2,
                     const float *v2, float *o, float *lse, int64_t seq, int64_t d, int64_t w1,
                     int64_t w2, double scale, int precision = MIMW_PREC_BF16) {
  require(precision == MIMW_PREC_BF16 || precision == MIMW_PREC_F32, MIMW_ERR_ARG,
          "precision must be MIMW_PREC_BF16 or MIMW_PREC_F32");
  require(seq >= 0 && d >= 0, MIMW_ERR_SHAPE, "negative extent");
  require(d <= 128, MIMW_ERR_UNSUPPORTED, "head dim > 128 not supported");
  require((w1 >= 1 && w2 >= 1) || seq == 0, MIMW_ERR_ARG, "windows must be >= 1");
  if (seq == 0) return;
  require(q && k1 && v1 && k2 && v2 && o, MIMW_ERR_ARG, "null pointer");
  require_sm100();
  if (precision == MIMW_PREC_F32) {
    const float *in[5] = {q, k1, v1, k2, v2};
    host_attention_f32(in, 5, o, lse, seq, d, w1, w2, true, scale);
    return;
  }
  cudaStream_t s = cudaStreamPerThread;
  const int64_t n = seq * d;
  DevBuf din(sizeof(float) * 5 * n, s);
  DevBuf dx(2 * 5 * seq * 128, s), dout(2 * seq * 128, s), dlse(sizeof(float) * seq, s),
      dof(sizeof(float) * (n ? n : 1), s);
  const float *src[5] = {q, k1, v1, k2, v2};
  void *dst[5];
  for (int t = 0; t < 5; ++t) {
    float *f = din.as<float>() + t * n;
    dst[t] = static_cast<char *>(dx.p) + (size_t)t * seq * 128 * 2;
    if (n) check_cuda(cudaMemcpyAsync(f, src[t], sizeof(float) * n, cudaMemcpyHostToDevice, s), "H2D");
    mimw::stage_cols_bf16(f, seq, d, 128, dst[t], 128, 0, 0, s);
  }
  check_cuda(cudaGetLastError(), "staging kernels");
  mimw::SimplicialArgs a{dst[0], dst[1], dst[2], dst[3], dst[4], dout.p, dlse.as<float>(),
                         1, seq, w1, w2, scale};
  check_cuda(mimw::simplicial_fwd_launch(a, s), "simplicial launch");
  if (n) {
    mimw::unpad_bf16_to_f32(dout.p, 128, dof.as<float>(), seq, d, s);
    check_cuda(cudaGetLastError(), "unpad");
    check_cuda(cudaMemcpyAsync(o, dof.p, sizeof(float) * n, cudaMemcpyDeviceToHost, s), "D2H o");
  }
  if (lse) check_cuda(cudaMemcpyAsync(lse, dlse.p, sizeof(float) * seq, cudaMemcpyDeviceToHost, s), "D2H lse");
  check_cuda(cudaStreamSynchronize(s), "simplicial execution");
}

// Argument checks shared by the public device GEMM entry and its tuning hook.
// Returns false when there is nothing to launch (empty output, or K == 0,
// for which C has been zero-filled: oracles.cpp:19).
bool gemm_device_checks(const void *a, const void *b, void *c, int64_t m, int64_t n, int64_t k, int64_t lda,
                        int64_t ldb, int64_t ldc, int32_t b_layout, int32_t c_dtype, void *stream) {
  require(b_layout == MIMW_B_KN || b_layout == MIMW_B_NK, MIMW_ERR_ARG, "bad b_layout");
  require(c_dtype == MIMW_F32 || c_dtype == MIMW_BF16, MIMW_ERR_ARG, "bad c_dtype");
  require(m >= 0 && n >= 0 && k >= 0, MIMW_ERR_SHAPE, "negative extent");
  require(m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31), MIMW_ERR_UNSUPPORTED, "extent >= 2^31");
  if (m == 0 || n == 0) return false;
  const int64_t es = c_dtype == MIMW_F32 ? 4 : 2;
  if (k == 0) {  // C = 0 (oracles.cpp:19)
    require(c != nullptr, MIMW_ERR_ARG, "null pointer");
    require(ldc >= n, MIMW_ERR_SHAPE, "leading dimension smaller than the row");
    require_sm100();
    check_cuda(cudaMemset2DAsync(c, ldc * es, 0, n * es, m, static_cast<cudaStream_t>(stream)), "memset");
    return false;
  }
  require(a && b && c, MIMW_ERR_ARG, "null pointer");
  require(lda >= k && ldc >= n && ldb >= (b_layout == MIMW_B_KN ? n : k), MIMW_ERR_SHAPE,
          "leading dimension smaller than the row");
  require_pitch(a, lda, 2, "a");
  require_pitch(b, ldb, 2, "b");
  require_pitch(c, ldc, es, "c");
  require_sm100();
  return true;
}

// Argument checks shared by the public device attention entry and its hook.
bool attention_device_checks(const void *q, const void *k, const void *v, const void *o, int64_t batch,
                             int64_t heads, int64_t seq, int64_t head_dim, int64_t window) {
  require(batch >= 0 && heads >= 0 && seq >= 0, MIMW_ERR_SHAPE, "negative extent");
  require(head_dim == 128, MIMW_ERR_UNSUPPORTED, "device attention supports head_dim == 128");
  require(window >= 1 || window == MIMW_WINDOW_NONCAUSAL, MIMW_ERR_ARG,
          "window must be >= 1 (or MIMW_WINDOW_NONCAUSAL)");
  require(seq < (1ll << 31) && batch * heads * ((seq + 255) / 256) < (1ll << 31), MIMW_ERR_UNSUPPORTED,
          "extent too large");
  if (batch == 0 || heads == 0 || seq == 0) return false;
  require(q && k && v && o, MIMW_ERR_ARG, "null pointer");
  require(((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o) % 16 == 0, MIMW_ERR_UNSUPPORTED,
          "tensors must be 16-byte aligned");
  require_sm100();
  return true;
}

}  // namespace

extern "C" {

int mimw_b200_version(void) { return 1; }

const char *mimw_b200_last_error(void) { return g_last_error.c_str(); }

int mimw_b200_trim_pool(void) {
  return guarded([&] {
    cudaMemPool_t pool = mimw::scratch_pool();
    if (pool) check_cuda(cudaMemPoolTrimTo(pool, 0), "cudaMemPoolTrimTo");
  });
}

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
    if (!gemm_device_checks(a, b, c, m, n, k, lda, ldb, ldc, b_layout, c_dtype, stream)) return;
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

int mimw_b200_oracle_attention(const float *q, const float *k, const float *v, float *o, float *lse,
                               int64_t seq, int64_t d, int64_t w, double scale) {
  return guarded([&] { host_attention(q, k, v, o, lse, seq, d, w, scale); });
}

int mimw_b200_oracle_attention_ex(const float *q, const float *k, const float *v, float *o, float *lse,
                                  int64_t seq, int64_t d, int64_t w, double scale, int32_t precision) {
  return guarded([&] { host_attention(q, k, v, o, lse, seq, d, w, scale, precision); });
}

int mimw_b200_oracle_attention_heads(const float *q, const float *k, const float *v, float *o, float *lse,
                                     int64_t heads, int64_t seq, int64_t d, int64_t w, double scale,
                                     int32_t precision) {
  return guarded([&] { host_attention_heads(q, k, v, o, lse, heads, seq, d, w, scale, precision); });
}

int mimw_b200_attention_fwd(const void *q, const void *k, const void *v, void *o, float *lse,
                            int64_t batch, int64_t heads, int64_t seq, int64_t head_dim,
                            int64_t window, double scale, void *stream) {
  return guarded([&] {
    if (!attention_device_checks(q, k, v, o, batch, heads, seq, head_dim, window)) return;
    mimw::AttnArgs a{};
    a.q = q;
    a.k = k;
    a.v = v;
    a.o = o;
    a.lse = lse;
    a.batch = batch;
    a.heads = heads;
    a.seq = seq;
    a.window = window;
    a.scale = scale;
    check_cuda(mimw::attention_fwd_launch(a, static_cast<cudaStream_t>(stream)), "attention launch");
  });
}

// ---- attention backward ---------------------------------
int mimw_b200_attention_bwd(const void *q, const void *k, const void *v, const void *o,
                            const void *dout, const float *lse, void *dq, void *dk, void *dv,
                            int64_t batch, int64_t heads, int64_t seq, int64_t head_dim,
                            int64_t window, double scale, void *stream) {
  return guarded([&] {
    require(batch >= 0 && heads >= 0 && seq >= 0, MIMW_ERR_SHAPE, "negative extent");
    require(head_dim == 128, MIMW_ERR_UNSUPPORTED, "device attention supports head_dim == 128");
    require(window >= 1 || window == MIMW_WINDOW_NONCAUSAL, MIMW_ERR_ARG,
            "window must be >= 1 (or MIMW_WINDOW_NONCAUSAL)");
    require(seq < (1ll << 31) && batch * heads < (1ll << 31), MIMW_ERR_UNSUPPORTED, "extent >= 2^31");
    if (batch == 0 || heads == 0 || seq == 0) return;
    require(q && k && v && o && dout && lse && dq && dk && dv, MIMW_ERR_ARG, "null pointer");
    require(((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)o | (uintptr_t)dout | (uintptr_t)dq |
             (uintptr_t)dk | (uintptr_t)dv) % 16 == 0,
            MIMW_ERR_UNSUPPORTED, "tensors must be 16-byte aligned");
    require_sm100();
    mimw::AttnBwdArgs a{};
    a.q = q;
    a.k = k;
    a.v = v;
    a.o = o;
    a.dout = dout;
    a.lse = lse;
    a.dq = dq;
    a.dk = dk;
    a.dv = dv;
    a.batch = batch;
    a.heads = heads;
    a.seq = seq;
    a.window = window;
    a.scale = scale;
    check_cuda(mimw::attention_bwd_launch(a, static_cast<cudaStream_t>(stream)), "attention bwd launch");
  });
}

static void gemm_mxfp8(const void *a, const void *sfa, const void *b, const void *sfb, void *c,
                       int64_t m, int64_t n, int64_t k, int cta_group, void *stream) {
  {
    require(m >= 0 && n >= 0 && k >= 0, MIMW_ERR_SHAPE, "negative extent");
    require(k % 32 == 0, MIMW_ERR_SHAPE, "k must be a multiple of the 32-element scale block");
    require(m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31), MIMW_ERR_UNSUPPORTED, "extent >= 2^31");
    if (m == 0 || n == 0) return;
    require(c != nullptr, MIMW_ERR_ARG, "null pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (k == 0) {
      require_sm100();
      check_cuda(cudaMemsetAsync(c, 0, (size_t)m * n * 2, s), "memset");
      return;
    }
    require(a && b && sfa && sfb, MIMW_ERR_ARG, "null pointer");
    require_pitch(a, k, 1, "a");
    require_pitch(b, k, 1, "b");
    require_pitch(c, n, 2, "c");
    require_sm100();
    DevBuf ws(mimw::gemm_mxfp8_workspace(m, n, k), s);
    mimw::Mxfp8Args g{};
    g.a = a;
    g.sfa = sfa;
    g.b = b;
    g.sfb = sfb;
    g.c = c;
    g.m = m;
    g.n = n;
    g.k = k;
    g.lda = k;
    g.ldb = k;
    g.ldc = n;
    g.workspace = ws.p;
    g.cta_group = cta_group;
    check_cuda(mimw::gemm_mxfp8_launch(g, s), "mxfp8 gemm launch");
  }
}

int mimw_b200_gemm_mxfp8(const void *a, const void *sfa, const void *b, const void *sfb, void *c,
                         int64_t m, int64_t n, int64_t k, void *stream) {
  return guarded([&] { gemm_mxfp8(a, sfa, b, sfb, c, m, n, k, 2, stream); });
}

// Test hook (not part of the public header): MXFP8 GEMM with forced cta_group
// (3: the 2-CTA kernel with 256 x 448 tiles, gemm_mxfp8_wide.cuh).
int mimw_b200_gemm_mxfp8_ex(const void *a, const void *sfa, const void *b, const void *sfb, void *c,
                            int64_t m, int64_t n, int64_t k, int32_t cta_group, void *stream) {
  return guarded([&] {
    require(cta_group >= 1 && cta_group <= 3, MIMW_ERR_ARG, "cta_group must be 1, 2 or 3 (2-CTA, 448-wide tiles)");
    gemm_mxfp8(a, sfa, b, sfb, c, m, n, k, cta_group, stream);
  });
}

int mimw_b200_grouped_gemm_bf16(const void *x, const int64_t *m_offsets, const void *w, void *y,
                                int64_t n_groups, int64_t n, int64_t k, int32_t w_layout,
                                void *stream) {
  return guarded([&] {
    grouped_gemm(x, m_offsets, w, y, n_groups, n, k, w_layout, 2, 0, -1, 0,
                 static_cast<cudaStream_t>(stream));
  });
}

int mimw_b200_oracle_simplicial_attention(const float *q, const float *k1, const float *v1,
                                           const float *k2, const float *v2, float *o, float *lse,
                                           int64_t seq, int64_t d, int64_t w1, int64_t w2,
                                           double scale) {
  return guarded([&] { host_simplicial(q, k1, v1, k2, v2, o, lse, seq, d, w1, w2, scale); });
}

int mimw_b200_oracle_simplicial_attention_ex(const float *q, const float *k1, const float *v1,
                                              const float *k2, const float *v2, float *o, float *lse,
                                              int64_t seq, int64_t d, int64_t w1, int64_t w2,
                                              double scale, int32_t precision) {
  return guarded([&] { host_simplicial(q, k1, v1, k2, v2, o, lse, seq, d, w1, w2, scale, precision); });
}

int mimw_b200_simplicial_attention_fwd(const void *q, const void *k1, const void *v1, const void *k2,
                                       const void *v2, void *o, float *lse, int64_t bh, int64_t seq,
                                       int64_t head_dim, int64_t w1, int64_t w2, double scale,
                                       void *stream) {
  return guarded([&] {
    require(bh >= 0 && seq >= 0, MIMW_ERR_SHAPE, "negative extent");
    require(head_dim == 128, MIMW_ERR_UNSUPPORTED, "device simplicial attention supports head_dim == 128");
    require(w1 >= 1 && w2 >= 1, MIMW_ERR_ARG, "windows must be >= 1");
    require(seq < (1ll << 31) && bh * ((seq + 127) / 128) < (1ll << 31), MIMW_ERR_UNSUPPORTED, "extent too large");
    if (bh == 0 || seq == 0) return;
    require(q && k1 && v1 && k2 && v2 && o, MIMW_ERR_ARG, "null pointer");
    require((((uintptr_t)q | (uintptr_t)k1 | (uintptr_t)v1 | (uintptr_t)k2 | (uintptr_t)v2 | (uintptr_t)o) & 15) == 0,
            MIMW_ERR_UNSUPPORTED, "tensors must be 16-byte aligned");
    require_sm100();
    mimw::SimplicialArgs a{q, k1, v1, k2, v2, o, lse, bh, seq, w1, w2, scale};
    check_cuda(mimw::simplicial_fwd_launch(a, static_cast<cudaStream_t>(stream)), "simplicial launch");
  });
}

int mimw_b200_layernorm(const float *x, const float *w, const float *b, float *y, float *mean,
                        float *rstd, int64_t rows, int64_t n, double eps, void *stream) {
  return guarded([&] {
    layernorm_checks(x, w, b, y, rows, n);
    if (rows == 0 || n == 0) return;
    require_sm100();
    mimw::LayerNormArgs a{x, w, b, y, mean, rstd, rows, n, eps, 0};
    check_cuda(mimw::layernorm_cluster_launch(a, static_cast<cudaStream_t>(stream)), "layernorm launch");
  });
}

// Test hook (not part of the public header): LayerNorm with a forced cluster size.
int mimw_b200_layernorm_ex(const float *x, const float *w, const float *b, float *y, float *mean,
                           float *rstd, int64_t rows, int64_t n, double eps, int32_t cluster,
                           void *stream) {
  return guarded([&] {
    layernorm_checks(x, w, b, y, rows, n);
    require(cluster >= 0 && cluster <= 16, MIMW_ERR_ARG, "cluster must be 0..16");
    if (rows == 0 || n == 0) return;
    require_sm100();
    mimw::LayerNormArgs a{x, w, b, y, mean, rstd, rows, n, eps, cluster};
    check_cuda(mimw::layernorm_cluster_launch(a, static_cast<cudaStream_t>(stream)), "layernorm launch");
  });
}

int mimw_b200_oracle_layernorm(const float *x, const float *w, const float *b, double eps, float *y,
                               float *mean, float *rstd, int64_t rows, int64_t n) {
  return guarded([&] {
    layernorm_checks(x, w, b, y, rows, n);
    if (rows == 0 || n == 0) return;
    require_sm100();
    cudaStream_t s = cudaStreamPerThread;
    const size_t xn = (size_t)rows * n;
    DevBuf dx(4 * xn, s), dw(4 * n, s), db(4 * n, s), dy(4 * xn, s), dm(4 * rows, s), dr(4 * rows, s);
    check_cuda(cudaMemcpyAsync(dx.p, x, 4 * xn, cudaMemcpyHostToDevice, s), "H2D x");
    check_cuda(cudaMemcpyAsync(dw.p, w, 4 * n, cudaMemcpyHostToDevice, s), "H2D w");
    check_cuda(cudaMemcpyAsync(db.p, b, 4 * n, cudaMemcpyHostToDevice, s), "H2D b");
    mimw::LayerNormArgs a{dx.as<float>(), dw.as<float>(), db.as<float>(), dy.as<float>(),
                          dm.as<float>(), dr.as<float>(), rows, n, eps, 0};
    check_cuda(mimw::layernorm_cluster_launch(a, s), "layernorm launch");
    check_cuda(cudaMemcpyAsync(y, dy.p, 4 * xn, cudaMemcpyDeviceToHost, s), "D2H y");
    if (mean) check_cuda(cudaMemcpyAsync(mean, dm.p, 4 * rows, cudaMemcpyDeviceToHost, s), "D2H mean");
    if (rstd) check_cuda(cudaMemcpyAsync(rstd, dr.p, 4 * rows, cudaMemcpyDeviceToHost, s), "D2H rstd");
    check_cuda(cudaStreamSynchronize(s), "layernorm execution");
  });
}

// Test hook (not part of the public header): grouped GEMM with forced
// cta_group / cluster cap.
int mimw_b200_grouped_gemm_bf16_ex(const void *x, const int64_t *m_offsets, const void *w, void *y,
                                   int64_t n_groups, int64_t n, int64_t k, int32_t w_layout,
                                   int32_t cta_group, int32_t max_clusters, int32_t swap_tails,
                                   int32_t tile_n, void *stream) {
  return guarded([&] {
    require(swap_tails >= -1 && swap_tails <= 1, MIMW_ERR_ARG, "swap_tails must be -1, 0 or 1");
    grouped_gemm(x, m_offsets, w, y, n_groups, n, k, w_layout, cta_group, max_clusters, swap_tails, tile_n,
                 static_cast<cudaStream_t>(stream));
  });
}

// Tuning hook (not part of the public header): attention with an explicit
// exp2-emulation split and CTA cap.
int mimw_b200_attention_fwd_ex(const void *q, const void *k, const void *v, void *o, float *lse,
                               int64_t batch, int64_t heads, int64_t seq, int64_t window,
                               double scale, int32_t emu, int32_t max_ctas, void *trace,
                               int32_t cta_group, void *stream) {
  return guarded([&] {
    if (!attention_device_checks(q, k, v, o, batch, heads, seq, 128, window)) return;
    require(emu >= -1 && emu <= 4 && max_ctas >= 0, MIMW_ERR_ARG, "bad emu / max_ctas");
    require(cta_group == 1 || cta_group == 2, MIMW_ERR_ARG, "cta_group must be 1 or 2");
    mimw::AttnArgs a{};
    a.q = q;
    a.k = k;
    a.v = v;
    a.o = o;
    a.lse = lse;
    a.batch = batch;
    a.heads = heads;
    a.seq = seq;
    a.window = window;
    a.scale = scale;
    a.emu = emu;
    a.max_ctas = max_ctas;
    a.trace = static_cast<unsigned long long *>(trace);
    a.cta_group = cta_group;
    check_cuda(mimw::attention_fwd_launch(a, static_cast<cudaStream_t>(stream)), "attention launch");
  });
}

#ifdef MIMW_TILE_TRACE
// trace builds only (tools/moe_trace.py): per-tile timeline buffer, 4 u64 per tile
int mimw_b200_debug_tile_trace(void *buf) {
  return guarded([&] { check_cuda(mimw::set_tile_trace(buf), "tile trace"); });
}
#endif

// Tuning / test hook (not part of the public header): force cta_group and
// raster group.  Used by the parity tests to cover the 1-CTA variant.
int mimw_b200_gemm_bf16_ex(const void *a, const void *b, void *c, int64_t m, int64_t n, int64_t k,
                           int64_t lda, int64_t ldb, int64_t ldc, int32_t b_layout, int32_t c_dtype,
                           int32_t cta_group, int32_t raster_group, int32_t max_clusters,
                           int32_t tile_n, void *stream) {
  return guarded([&] {
    require(cta_group == 1 || cta_group == 2 || cta_group == 4, MIMW_ERR_ARG,
            "cta_group must be 1, 2 or 4 (two CTA pairs sharing B by multicast)");
    require(tile_n == 0 || tile_n == 256 || (tile_n == 512 && cta_group == 2 && c_dtype == MIMW_BF16),
            MIMW_ERR_ARG, "tile_n must be 0 (auto), 256, or 512 (cta_group 2, bf16 out)");
    require(max_clusters >= 0, MIMW_ERR_ARG, "bad max_clusters");
    if (!gemm_device_checks(a, b, c, m, n, k, lda, ldb, ldc, b_layout, c_dtype, stream)) return;
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
    g.cta_group = cta_group == 4 ? 2 : cta_group;
    g.cluster_pairs = cta_group == 4 ? 2 : 1;
    g.raster_group = raster_group;
    g.max_clusters = max_clusters;
    g.tile_n = tile_n;
    check_cuda(mimw::gemm_bf16_launch(g, static_cast<cudaStream_t>(stream)), "gemm launch");
  });
}

// ---- all-gather multi-device GEMM ------------------------
int64_t mimw_b200_multi_device_gemm_workspace_bytes(int32_t rank, int32_t world,
                                                    const int64_t *k_splits, int64_t rows,
                                                    int64_t n) {
  if (world < 1 || world > MIMW_MAX_DEVICES || rank < 0 || rank >= world || !k_splits || rows < 0 ||
      n < 0)
    return -1;
  return (int64_t)mimw::multi_device_gemm_workspace_bytes(rank, world, k_splits, rows, n);
}

int mimw_b200_multi_device_gemm_ex(int32_t rank, int32_t world, const void *const *a_splits,
                                   const void *const *b_splits, const int64_t *k_splits, int64_t m,
                                   int64_t n, int64_t row0, int64_t rows, void *c, int64_t ldc,
                                   void *workspace, int64_t workspace_bytes, uint32_t *const *pads,
                                   uint32_t epoch, int32_t comm_pairs, int32_t max_pairs,
                                   int32_t comm_box, int32_t comm_agents, int32_t comm_lag,
                                   void *stream) {
  return guarded([&] {
    require(world >= 1 && world <= MIMW_MAX_DEVICES && rank >= 0 && rank < world, MIMW_ERR_ARG,
            "rank/world out of range (world <= MIMW_MAX_DEVICES)");
    require(a_splits && b_splits && k_splits, MIMW_ERR_ARG, "null split arrays");
    require(m >= 0 && n >= 0 && row0 >= 0 && rows >= 0 && row0 + rows <= m, MIMW_ERR_SHAPE,
            "row range [row0, row0 + rows) outside [0, m)");
    require(n % 8 == 0, MIMW_ERR_UNSUPPORTED, "n must be a multiple of 8 (16-byte TMA rows)");
    mimw::MultiDeviceGemmArgs g{};
    g.rank = rank;
    g.world = world;
    bool any_pad = false, all_pad = true;
    for (int s = 0; s < world; ++s) {
      require(k_splits[s] >= 0, MIMW_ERR_SHAPE, "negative K split");
      require(k_splits[s] % 8 == 0, MIMW_ERR_UNSUPPORTED,
              "every K split must be a multiple of 8 (16-byte TMA rows)");
      if (k_splits[s] && rows && n) {
        require(a_splits[s] && b_splits[s], MIMW_ERR_ARG, "null split pointer");
        require_pitch(a_splits[s], k_splits[s], 2, "a split");
        require_pitch(b_splits[s], n, 2, "b split");
      }
      g.a[s] = a_splits[s];
      g.b[s] = b_splits[s];
      g.k[s] = k_splits[s];
      const bool has = pads && pads[s];
      any_pad |= has;
      all_pad &= has;
      g.pads[s] = has ? pads[s] : nullptr;
    }
    require(!any_pad || all_pad, MIMW_ERR_ARG, "pads: give every device's signal pad or none");
    require(!any_pad || epoch != 0, MIMW_ERR_ARG, "epoch must be >= 1 with a device barrier");
    const bool work = rows > 0 && n > 0;
    if (!work && !any_pad) return;  // nothing to compute, no peers to meet
    require(workspace != nullptr, MIMW_ERR_ARG, "null workspace");
    if (work) {
      require(c != nullptr, MIMW_ERR_ARG, "null output");
      require_pitch(c, ldc, 2, "c");
    }
    require(((uintptr_t)workspace & 1023) == 0, MIMW_ERR_UNSUPPORTED, "workspace not 1 KiB aligned");
    const int64_t need = (int64_t)mimw::multi_device_gemm_workspace_bytes(rank, world, k_splits, rows, n);
    require(workspace_bytes >= need, MIMW_ERR_ARG,
            "workspace too small: need " + std::to_string(need) + " bytes");
    require_sm100();
    g.n = n;
    g.row0 = row0;
    g.rows = rows;
    g.c = c;
    g.ldc = ldc;
    g.ws = workspace;
    g.ws_bytes = (size_t)workspace_bytes;
    g.epoch = epoch;
    g.comm_clusters = comm_pairs;  // 0 default, > 0 dedicated comm pairs, < 0 distributed comm warps
    g.max_clusters = max_pairs;
    g.comm_box = comm_box;
    g.comm_agents = comm_agents;
    g.comm_lag = comm_lag;
    check_cuda(mimw::multi_device_gemm_launch(g, static_cast<cudaStream_t>(stream)),
               "multi-device gemm launch");
  });
}

int mimw_b200_multi_device_gemm(int32_t rank, int32_t world, const void *const *a_splits,
                                const void *const *b_splits, const int64_t *k_splits, int64_t m,
                                int64_t n, int64_t row0, int64_t rows, void *c, int64_t ldc,
                                void *workspace, int64_t workspace_bytes, uint32_t *const *pads,
                                uint32_t epoch, int32_t comm_pairs, int32_t max_pairs,
                                void *stream) {
  return mimw_b200_multi_device_gemm_ex(rank, world, a_splits, b_splits, k_splits, m, n, row0, rows,
                                        c, ldc, workspace, workspace_bytes, pads, epoch, comm_pairs,
                                        max_pairs, 0, 0, 0, stream);
}

// ---- CUDA IPC plumbing for the peer mappings ----------------------------------
int mimw_b200_ipc_alloc(int64_t bytes, void **ptr, void *handle) {
  return guarded([&] {
    require(bytes > 0 && ptr && handle, MIMW_ERR_ARG, "bad ipc_alloc arguments");
    require_sm100();
    check_cuda(cudaMalloc(ptr, (size_t)bytes), "cudaMalloc");
    check_cuda(cudaMemset(*ptr, 0, (size_t)bytes), "cudaMemset");
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, *ptr), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == MIMW_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
  });
}

int mimw_b200_ipc_open(const void *handle, void **ptr) {
  return guarded([&] {
    require(handle && ptr, MIMW_ERR_ARG, "bad ipc_open arguments");
    require_sm100();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    check_cuda(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int mimw_b200_ipc_close(void *ptr) {
  return guarded([&] { check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); });
}

int mimw_b200_ipc_free(void *ptr) {
  return guarded([&] { check_cuda(cudaFree(ptr), "cudaFree"); });
}

}  // extern "C"
