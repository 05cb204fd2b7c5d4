// Drop-in check of the reference-side binding (integration/oracles_b200.cpp).
// TEST INFRASTRUCTURE: compiled against the reference's UNMODIFIED headers
// and its tensor_io.cpp / case.cpp (seeded random_tile, MIMWTNSR read_tensor,
// rel_error), with the shim standing in for the oracle bodies of
// proj/core/src/oracles.cpp.  Every reference case (the *.case sidecars and
// the acceptance cases the golden fixtures pin) is regenerated exactly as the
// reference does (make_inputs seed rule, case.cpp:82-92), run through the
// reference's own function signatures -> libmimw_b200 -> B200, and compared
// with the reference's output by the reference's rel_error at the case's own
// tolerance.
//   dropin_check <golden dir>
#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "mimw/case.hpp"
#include "mimw/oracles.hpp"
#include "mimw/tensor_io.hpp"

using namespace mimw;

namespace {
std::string g_dir;
int g_fail = 0;

Tile input(std::uint64_t seed, int k, std::vector<std::int64_t> shape) {
  return random_tile(shape, seed * 1000003ull + (std::uint64_t)k);  // case.cpp:88
}
Tile golden(const std::string &file) {
  auto t = read_tensor(g_dir + "/" + file);
  if (!t) {
    std::fprintf(stderr, "missing fixture %s\n", file.c_str());
    ++g_fail;
    return Tile();
  }
  return *t;
}
void check(const char *name, const Tile &got, const Tile &want, double tol) {
  const double e = rel_error(got, want);
  const bool pass = got.shape == want.shape && e <= tol;
  std::printf("%-28s rel_error %.3e  tol %.0e  %s\n", name, e, tol, pass ? "ok" : "FAIL");
  if (!pass) ++g_fail;
}
}  // namespace

int main(int argc, char **argv) {
  g_dir = argc > 1 ? argv[1] : "tests/golden";
  try {
    {  // kernels/gemm_pipeline.case: seed 7, tol 1e-4
      Tile a = input(7, 0, {64, 64}), b = input(7, 1, {64, 64});
      check("gemm_pipeline", oracle_gemm(a, b), golden("gemm_pipeline.c.tnsr"), 1e-4);
    }
    {  // kernels/gemm_clc.case: seed 19
      Tile a = input(19, 0, {64, 128}), b = input(19, 1, {128, 64});
      check("gemm_clc", oracle_gemm(a, b), golden("gemm_clc.c.tnsr"), 1e-4);
    }
    {  // tests/acceptance.cpp:392-421 collective_dot: seeds 41 / 42
      Tile a = random_tile({32, 16}, 41), b = random_tile({16, 24}, 42);
      check("collective_dot", oracle_gemm(a, b), golden("collective_dot.c.tnsr"), 1e-4);
    }
    {  // kernels/multi_device_gemm.case: seed 23
      Tile a0 = input(23, 0, {64, 64}), a1 = input(23, 1, {64, 64});
      Tile b0 = input(23, 2, {64, 32}), b1 = input(23, 3, {64, 32});
      check("multi_device_gemm", oracle_multi_device_gemm(a0, a1, b0, b1), golden("multi_device_gemm.c.tnsr"),
            1e-4);
    }
    {  // kernels/simplicial_attention.case: seed 31, w1 2, w2 16, scale 0.25, tol 1e-3
      Tile q = input(31, 0, {32, 16}), k1 = input(31, 1, {32, 16}), v1 = input(31, 2, {32, 16});
      Tile k2 = input(31, 3, {32, 16}), v2 = input(31, 4, {32, 16});
      Tile o, lse;
      oracle_simplicial_attention(q, k1, v1, k2, v2, 2, 16, 0.25, &o, &lse);
      check("simplicial_attention.o", o, golden("simplicial_attention.o.tnsr"), 1e-3);
      check("simplicial_attention.lse", lse, golden("simplicial_attention.lse.tnsr"), 1e-3);
      // tests/acceptance.cpp:333-355: attention on (q, k2, v2), w 16, scale 0.25, tol 1e-4
      Tile oa;
      oracle_attention(q, k2, v2, 16, 0.25, &oa);
      check("attention_degeneration", oa, golden("attention_degeneration.o.tnsr"), 1e-4);
    }
    {  // kernels/layernorm_cluster.case: seed 5, eps 1e-5, tol 1e-5
      Tile x = input(5, 0, {4, 1024}), w = input(5, 1, {1024}), b = input(5, 2, {1024});
      Tile y;
      oracle_layernorm(x, w, b, 1e-5, &y);
      check("layernorm_cluster", y, golden("layernorm_cluster.y.tnsr"), 1e-5);
    }
  } catch (const std::exception &e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s\n", g_fail ? "dropin FAILED" : "dropin ok");
  return g_fail ? 1 : 0;
}
