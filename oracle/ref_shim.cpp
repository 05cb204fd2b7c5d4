// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference oracles, compiled together
// with /root/reference/proj/core/src/{oracles,case,tensor_io}.cpp by
// oracle/Makefile into oracle/_ref/libmimw_ref.so.  It exists so that the
// Python tests and bench.py's CPU leg can call the reference's own code:
//
//   mimw::oracle_gemm                 proj/core/src/oracles.cpp:14-26
//   mimw::oracle_attention            proj/core/src/oracles.cpp:119-145
//   mimw::oracle_simplicial_attention proj/core/src/oracles.cpp:82-117
//   mimw::oracle_multi_device_gemm    proj/core/src/oracles.cpp:57-80
//   mimw::oracle_layernorm            proj/core/src/oracles.cpp:28-55
//   mimw::random_tile                 proj/core/src/tensor_io.cpp:80-88
//   mimw::rel_error                   proj/core/src/case.cpp:94-104
//   mimw::write_tensor / read_tensor  proj/core/src/tensor_io.cpp:30-78
//
// The *_mt entry points are the "N-core" CPU baseline from BASELINE.md §4:
// the same single-threaded reference oracle called on independent GEMM row
// blocks / attention heads from N std::threads (SPEC.md:505-506 allows
// parallelising pure oracle calls).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "mimw/case.hpp"
#include "mimw/oracles.hpp"
#include "mimw/tensor_io.hpp"

using mimw::Tile;

namespace {
Tile make_tile(const float *p, std::vector<std::int64_t> shape) {
  Tile t(std::move(shape));
  std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
  return t;
}
void put(const Tile &t, float *out) {
  std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}
}  // namespace

extern "C" {

void ref_random_tile(const std::int64_t *shape, int rank, std::uint64_t seed,
                     float *out) {
  std::vector<std::int64_t> s(shape, shape + rank);
  put(mimw::random_tile(s, seed), out);
}

double ref_rel_error(const float *a, const float *b, std::int64_t n) {
  Tile ta = make_tile(a, {n}), tb = make_tile(b, {n});
  return mimw::rel_error(ta, tb);
}

void ref_oracle_gemm(const float *a, const float *b, float *c, std::int64_t m,
                     std::int64_t n, std::int64_t k) {
  put(mimw::oracle_gemm(make_tile(a, {m, k}), make_tile(b, {k, n})), c);
}

// Rows [r0, r1) of C = A.B through the unmodified oracle on A[r0:r1, :].
// Exact: c[i, j] depends only on A[i, :] and B[:, j] (oracles.cpp:17-23).
void ref_oracle_gemm_rows(const float *a, const float *b, float *c,
                          std::int64_t m, std::int64_t n, std::int64_t k,
                          std::int64_t r0, std::int64_t r1) {
  (void)m;
  Tile tb = make_tile(b, {k, n});
  put(mimw::oracle_gemm(make_tile(a + r0 * k, {r1 - r0, k}), tb), c + r0 * n);
}

void ref_oracle_gemm_mt(const float *a, const float *b, float *c,
                        std::int64_t m, std::int64_t n, std::int64_t k,
                        int threads) {
  threads = std::max(1, threads);
  Tile tb = make_tile(b, {k, n});
  std::vector<std::thread> pool;
  std::int64_t per = (m + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    std::int64_t r0 = t * per, r1 = std::min(m, r0 + per);
    if (r0 >= r1) break;
    pool.emplace_back([&, r0, r1] {
      put(mimw::oracle_gemm(make_tile(a + r0 * k, {r1 - r0, k}), tb),
          c + r0 * n);
    });
  }
  for (auto &th : pool) th.join();
}

void ref_oracle_attention(const float *q, const float *k, const float *v,
                          float *o, std::int64_t seq, std::int64_t d, int w,
                          double scale) {
  Tile to;
  mimw::oracle_attention(make_tile(q, {seq, d}), make_tile(k, {seq, d}),
                         make_tile(v, {seq, d}), w, scale, &to);
  put(to, o);
}

// heads independent [seq, d] problems laid out back to back ([B*H, S, D]).
void ref_oracle_attention_heads_mt(const float *q, const float *k,
                                   const float *v, float *o,
                                   std::int64_t heads, std::int64_t seq,
                                   std::int64_t d, int w, double scale,
                                   int threads) {
  threads = std::max(1, threads);
  std::vector<std::thread> pool;
  std::int64_t hs = seq * d;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (std::int64_t h = t; h < heads; h += threads) {
        Tile to;
        mimw::oracle_attention(make_tile(q + h * hs, {seq, d}),
                               make_tile(k + h * hs, {seq, d}),
                               make_tile(v + h * hs, {seq, d}), w, scale, &to);
        put(to, o + h * hs);
      }
    });
  }
  for (auto &th : pool) th.join();
}

void ref_oracle_simplicial_attention(const float *q, const float *k1,
                                     const float *v1, const float *k2,
                                     const float *v2, float *o, float *lse,
                                     std::int64_t seq, std::int64_t d, int w1,
                                     int w2, double scale) {
  Tile to, tl;
  std::vector<std::int64_t> s{seq, d};
  mimw::oracle_simplicial_attention(make_tile(q, s), make_tile(k1, s),
                                    make_tile(v1, s), make_tile(k2, s),
                                    make_tile(v2, s), w1, w2, scale, &to, &tl);
  put(to, o);
  put(tl, lse);
}

void ref_oracle_multi_device_gemm(const float *a0, const float *a1,
                                  const float *b0, const float *b1, float *c,
                                  std::int64_t m, std::int64_t k0,
                                  std::int64_t k1, std::int64_t n) {
  put(mimw::oracle_multi_device_gemm(make_tile(a0, {m, k0}),
                                     make_tile(a1, {m, k1}),
                                     make_tile(b0, {k0, n}),
                                     make_tile(b1, {k1, n})),
      c);
}

void ref_oracle_layernorm(const float *x, const float *w, const float *b,
                          double eps, float *y, float *mean, float *rstd,
                          std::int64_t rows, std::int64_t n) {
  Tile ty, tm, tr;
  mimw::oracle_layernorm(make_tile(x, {rows, n}), make_tile(w, {n}),
                         make_tile(b, {n}), eps, &ty, &tm, &tr);
  put(ty, y);
  put(tm, mean);
  put(tr, rstd);
}

int ref_write_tensor(const char *path, const float *data,
                     const std::int64_t *shape, int rank) {
  Tile t = make_tile(data, std::vector<std::int64_t>(shape, shape + rank));
  return mimw::write_tensor(path, t) ? 0 : 1;
}

}  // extern "C"
