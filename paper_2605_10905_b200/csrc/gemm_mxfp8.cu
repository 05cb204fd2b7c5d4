// Block-scaled FP8 (MXFP8: e4m3 values, one UE8M0 scale per 32 K-elements)
// persistent warp-specialized GEMM for sm_100a:
//     C[M,N] (bf16) = sum_k  A[m,k] * 2^(sfa[m,k/32]-127) * B[n,k] * 2^(sfb[n,k/32]-127)
//
// The reference has no FP8; the oracle for this path is
// oracle_gemm (proj/core/src/oracles.cpp:14-26) on the dequantised f32 Tiles
// (oracle/oracle.c orc_mx_dequant).  Same MIMW roles as gemm_bf16.cu:
//   warp 0      TMA producer: A/B tiles and the stage's scale-factor atoms
//               (all cp.async.bulk.tensor, 128-B swizzle for A/B), completing
//               on the pair leader's `full[s]` with the stage's byte count
//   warp 1      TMEM allocator + MMA issuer (pair leader): tcgen05.cp moves the
//               stage's scale factors smem -> TMEM (32x128b.warpx4), then
//               4 x tcgen05.mma.kind::mxf8f6f4.block_scale (K = 32 each, sf_id
//               selects the k-block byte); the commit frees both CTAs' slots
//   warps 2..5  epilogue: TMEM -> bf16 -> swizzled smem -> TMA store
// Scale factors in TMEM (found with tools/sf_probe.cu): row m of A reads lane
// m, column (m >> 5), byte sf_id; column n of B reads lane (n & 31), column
// (n >> 5), byte sf_id.  The 512-byte "atom" [r*16 + c*4 + y] = sf(row 32c+r,
// kblock y) is exactly what one tcgen05.cp.32x128b.warpx4 consumes; a small
// pre-pass (sf_tile_kernel) reorders the natural [rows, K/32] scale arrays
// into per-tile atoms.
//
// CG = 2 (default): a CTA pair runs M=256 x N=224 cta_group::2 MMAs.  Each
// CTA stages its own 128 A rows and 112 of the 224 B rows (halving the
// L2->smem traffic and the smem write bandwidth of the 1-CTA tile, the limit
// of the FP8 rate), its own rows' SFA atom and the FULL tile's SFB atoms
// (every CTA's D rows see all N columns).  The leader's tcgen05.cp.cta_group::2
// copies each CTA's smem into that CTA's TMEM.  Two fp32 accumulators
// (2 x 224 columns) + double-buffered scale factors fill the 512 TMEM columns.
#include "gemm_mxfp8.h"
#include "ptx.cuh"
#include "tma_host.h"

#include <algorithm>

namespace mimw {

namespace {

constexpr int BM_CTA = 128;      // A rows per CTA
constexpr int BN = 224;          // N per MMA / cluster tile (7 x 32 columns)
constexpr int BK = 128;          // fp8 bytes per 128-B swizzle row = 4 scale blocks
constexpr int UMMA_K = 32;
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_COLS = 32;
constexpr int SFA_BYTES = 512;                   // one atom: 128 rows x 4 k-blocks
constexpr int SFB_BYTES = 1024;                  // two atoms: 256 (>= 224) columns
constexpr int SF_STAGE = SFA_BYTES + SFB_BYTES;
constexpr int EPI_BUF = 32 * EPI_COLS * 2;       // bf16
constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_BUF;
constexpr uint32_t TM_ACC = 0;                   // 2 x 224 columns
constexpr uint32_t TM_SF = 448;                  // per SF buffer: SFA 4 cols + SFB 8 cols
constexpr uint32_t SF_STRIDE = 16;

template <int CG>
struct Cfg {
  static constexpr int NB_CTA = BN / CG;                        // B rows staged per CTA
  static constexpr int A_BYTES = BM_CTA * BK;                   // 16 KiB
  static constexpr int B_BYTES = NB_CTA * BK;                   // 14 / 28 KiB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 2 ? 6 : 4;
  static constexpr int SF_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = SF_OFF + STAGES * SF_STAGE;
  static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int TX = CG * (STAGE_BYTES + SF_STAGE);      // bytes landing per stage (pair)
  static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1024-B aligned for SWIZZLE_128B");
  static_assert(SMEM <= 232448, "smem budget");
};

struct Sched {
  int num_m, num_n, group;  // num_m in cluster tiles (128 * CG rows)
  __device__ __forceinline__ void tile(int t, int &mt, int &nt) const {
    int per_group = group * num_n;
    int g = t / per_group;
    int first_m = g * group;
    int gsize = min(num_m - first_m, group);
    int r = t - g * per_group;
    mt = first_m + r % gsize;
    nt = r / gsize;
  }
};

// tmSFA / tmSFB: the atom workspace viewed as [atoms * 2, 256] bytes
// (TMA boxes of 256 x 2 = one SFA atom, 256 x 4 = the two SFB atoms of a tile).
template <int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_mxfp8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmSFA,
                  const __grid_constant__ CUtensorMap tmSFB, int M, int N, int K, int KG, Sched sched) {
  using C = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + C::BAR_OFF;
  auto full_bar = [&](int s) { return bar_base + 8 * s; };
  auto empty_bar = [&](int s) { return bar_base + 8 * (C::STAGES + s); };
  auto tfull_bar = [&](int a) { return bar_base + 8 * (2 * C::STAGES + a); };
  auto tempty_bar = [&](int a) { return bar_base + 8 * (2 * C::STAGES + 2 + a); };
  const uint32_t tmem_slot = bar_base + 8 * (2 * C::STAGES + 4);
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + C::BAR_OFF + 8 * (2 * C::STAGES + 4));

  const int warp = threadIdx.x / 32;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0;
  const bool leader = (rank == 0);
  const int cluster = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
  const int nclusters = (CG == 2) ? (int)nclusters_x() : (int)gridDim.x;
  const int num_tiles = sched.num_m * sched.num_n;
  const int num_k = (K + BK - 1) / BK;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    tma_prefetch_desc(&tmSFA);
    tma_prefetch_desc(&tmSFB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), EPI_WARPS * CG);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<CG>(tmem_slot, 512);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = (CG == 2) ? map_to_rank(full_bar(0), 0) : full_bar(0);
      for (int t = cluster; t < num_tiles; t += nclusters) {
        int mt, nt;
        sched.tile(t, mt, nt);
        const int m128 = mt * CG + (int)rank;   // this CTA's 128-row block
        for (int kb = 0; kb < num_k; ++kb) {
          if constexpr (CG == 2) mbar_wait_cluster(empty_bar(stage), phase ^ 1, 1);
          else mbar_wait(empty_bar(stage), phase ^ 1, 1);
          const uint32_t fb = full0 + 8 * stage;
          if (leader) mbar_arrive_expect_tx(full_bar(stage), C::TX);
          const uint32_t sa = sbase + stage * C::STAGE_BYTES;
          const uint32_t sb = sa + C::A_BYTES;
          const uint32_t ssf = sbase + C::SF_OFF + stage * SF_STAGE;
          const int sfa_row = (m128 * KG + kb) * 2;
          const int sfb_row = (nt * KG + kb) * 4;
          if constexpr (CG == 2) {
            tma_load_2d_cg2(sa, &tmA, fb, kb * BK, m128 * BM_CTA);
            tma_load_2d_cg2(sb, &tmB, fb, kb * BK, nt * BN + (int)rank * C::NB_CTA);
            tma_load_2d_cg2(ssf, &tmSFA, fb, 0, sfa_row);
            tma_load_2d_cg2(ssf + SFA_BYTES, &tmSFB, fb, 0, sfb_row);
          } else {
            tma_load_2d(sa, &tmA, fb, kb * BK, m128 * BM_CTA);
            tma_load_2d(sb, &tmB, fb, kb * BK, nt * BN);
            tma_load_2d(ssf, &tmSFA, fb, 0, sfa_row);
            tma_load_2d(ssf + SFA_BYTES, &tmSFB, fb, 0, sfb_row);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      uint32_t sf_buf = 0;  // TMEM scale-factor double buffer (runs across tiles)
      constexpr uint32_t HI_SW128 = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        mbar_wait_cluster(tempty_bar(acc), acc_phase ^ 1, 2);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + TM_ACC + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(full_bar(stage), phase, 3);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = sbase + stage * C::STAGE_BYTES;
            const uint32_t sb = sa + C::A_BYTES;
            const uint32_t ssf = sbase + C::SF_OFF + stage * SF_STAGE;
            const uint32_t tsf = tmem_base + TM_SF + sf_buf * SF_STRIDE;
            // scale factors smem -> TMEM (ordered before the MMAs in the tensor pipe)
            tmem_cp_32x128b_warpx4<CG>(tsf, smem_desc_noswz(ssf, 128, 128));
            tmem_cp_32x128b_warpx4<CG>(tsf + 4, smem_desc_noswz(ssf + SFA_BYTES, 128, 128));
            tmem_cp_32x128b_warpx4<CG>(tsf + 8, smem_desc_noswz(ssf + SFA_BYTES + 512, 128, 128));
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              uint64_t ad, bd;
              asm volatile("mov.b64 %0, {%1, %2};" : "=l"(ad) : "r"(LO_KMAJ | ((sa + k * 32) >> 4)), "r"(HI_SW128));
              asm volatile("mov.b64 %0, {%1, %2};" : "=l"(bd) : "r"(LO_KMAJ | ((sb + k * 32) >> 4)), "r"(HI_SW128));
              mma_mxf8_ss<CG>(d_tmem, ad, bd, idesc_mxf8(BM_CTA * CG, BN, k, k), tsf, tsf + 4,
                              (kb | k) != 0);
            }
            if constexpr (CG == 2) {
              mma_commit_cg2_mc(empty_bar(stage), 0x3);
              if (kb == num_k - 1) mma_commit_cg2_mc(tfull_bar(acc), 0x3);
            } else {
              mma_commit(empty_bar(stage));
              if (kb == num_k - 1) mma_commit(tfull_bar(acc));
            }
          }
          __syncwarp();
          sf_buf ^= 1;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const int ew = warp - 2;
    const uint32_t lane = lane_id();
    const uint32_t stage_base = sbase + C::EPI_OFF + ew * 2 * EPI_BUF;
    const uint32_t tempty_leader0 = (CG == 2) ? map_to_rank(tempty_bar(0), 0) : tempty_bar(0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = cluster; t < num_tiles; t += nclusters) {
      int mt, nt;
      sched.tile(t, mt, nt);
      const int row0 = (mt * CG + (int)rank) * BM_CTA + q * 32;
      const int col0 = nt * BN;
      mbar_wait(tfull_bar(acc), acc_phase, 4);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + TM_ACC + acc * BN;
#pragma unroll 1
      for (int ch = 0; ch < BN / EPI_COLS; ++ch) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + ch * EPI_COLS, v);
        tmem_ld_wait();
        if (ch == BN / EPI_COLS - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + 8 * acc);
            else mbar_arrive(tempty_bar(acc));
          }
        }
        if (row0 < M && col0 + ch * EPI_COLS < N) {
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const uint32_t sbuf = stage_base + buf * EPI_BUF;
          const uint32_t rbase = sbuf + lane * 64;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t pc = (uint32_t)c ^ ((lane >> 1) & 3);
            st_shared_v4(rbase + pc * 16,
                         pack_bf16(__uint_as_float(v[8 * c + 0]), __uint_as_float(v[8 * c + 1])),
                         pack_bf16(__uint_as_float(v[8 * c + 2]), __uint_as_float(v[8 * c + 3])),
                         pack_bf16(__uint_as_float(v[8 * c + 4]), __uint_as_float(v[8 * c + 5])),
                         pack_bf16(__uint_as_float(v[8 * c + 6]), __uint_as_float(v[8 * c + 7])));
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, sbuf, col0 + ch * EPI_COLS, row0);
            bulk_commit();
          }
          buf ^= 1;
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, 512);
  }
}

// Reorder natural [rows, kb] UE8M0 scales into per-tile atoms:
//   atom(tile, g, half)[r*16 + c*4 + y] = sf[tile*rows_per_tile + half*128 + 32c + r, 4g + y]
// (127 = 1.0 outside the matrix), for SFA (128-row tiles, 1 half) and SFB
// (224-row tiles, 2 halves) in ONE launch.  A CTA owns one 128-row group and
// 32 k-groups: it reads the 128 x 128-byte block row-wise (coalesced) into
// padded smem, then writes the 32 atoms as whole 512-byte lines.
__global__ void __launch_bounds__(256) sf_tile_kernel(const uint8_t *__restrict__ sfa, int m,
                                                      const uint8_t *__restrict__ sfb, int n, int kb,
                                                      int kg, int m128, uint8_t *__restrict__ out_a,
                                                      uint8_t *__restrict__ out_b) {
  constexpr int PITCH = 33;  // words per smem row (+1: conflict-free column reads)
  __shared__ uint32_t blk[128 * PITCH];
  const int grp = blockIdx.x;
  const bool is_a = grp < m128;
  const uint8_t *sf = is_a ? sfa : sfb;
  const int rows = is_a ? m : n;
  int row0, valid;  // first row of the group, rows of the group inside its tile
  uint8_t *out;
  int halves, tile, half;
  if (is_a) {
    tile = grp; half = 0; halves = 1; row0 = grp * 128; valid = 128; out = out_a;
  } else {
    const int gg = grp - m128;
    tile = gg >> 1; half = gg & 1; halves = 2;
    row0 = tile * BN + half * 128; valid = min(128, BN - half * 128); out = out_b;
  }
  const int g0 = blockIdx.y * 32;
  const int k0 = g0 * 4;  // first byte (k-block) of this chunk in a row
  // load: 128 rows x 128 bytes, one byte-quad (4 k-blocks = one word) per load
  for (int i = threadIdx.x; i < 128 * 32; i += 256) {
    const int r = i >> 5, wq = i & 31;
    const int row = row0 + r, k = k0 + wq * 4;
    uint32_t v = 0x7F7F7F7Fu;
    if (r < valid && row < rows) {
      const uint8_t *src = sf + (size_t)row * kb + k;
      if (k + 3 < kb && ((reinterpret_cast<uintptr_t>(src) & 3) == 0)) {
        v = __ldg(reinterpret_cast<const uint32_t *>(src));
      } else {
        v = 0;
        for (int y = 0; y < 4; ++y) v |= (uint32_t)(k + y < kb ? __ldg(src + y) : 127) << (8 * y);
      }
    }
    blk[r * PITCH + wq] = v;
  }
  __syncthreads();
  // write: atom (g0 + a) line r = words {blk[32c + r][a]}, c = 0..3
  for (int i = threadIdx.x; i < 32 * 32; i += 256) {
    const int a = i >> 5, r = i & 31;
    const int g = g0 + a;
    if (g >= kg) continue;
    uint4 w;
    w.x = blk[(r) * PITCH + a];
    w.y = blk[(32 + r) * PITCH + a];
    w.z = blk[(64 + r) * PITCH + a];
    w.w = blk[(96 + r) * PITCH + a];
    uint8_t *dst = out + ((size_t)((size_t)tile * kg + g) * halves + half) * 512 + r * 16;
    *reinterpret_cast<uint4 *>(dst) = w;
  }
}

#include "gemm_mxfp8_wide.cuh"

}  // namespace

// Workspace: SFA atoms [ceil(m/128)][KG] x 512 B, then SFB atoms
// [ceil(n/224)][KG][2] x 512 B (KG = ceil(k/128)).
size_t gemm_mxfp8_workspace(int64_t m, int64_t n, int64_t k) {
  const int64_t kg = (k + BK - 1) / BK;
  const int64_t m128 = (m + BM_CTA - 1) / BM_CTA + 1;  // +1: a pair's odd tail block
  const int64_t nt = (n + BN - 1) / BN;
  return (size_t)(m128 * kg * SFA_BYTES + nt * kg * SFB_BYTES);
}

template <int CG>
cudaError_t launch_cg(const Mxfp8Args &g, cudaStream_t stream) {
  using Cf = Cfg<CG>;
  const int kg = (int)((g.k + BK - 1) / BK);
  const int num_m = (int)((g.m + BM_CTA * CG - 1) / (BM_CTA * CG));
  const int num_n = (int)((g.n + BN - 1) / BN);
  const int m128 = num_m * CG;
  uint8_t *sfa_t = static_cast<uint8_t *>(g.workspace);
  uint8_t *sfb_t = sfa_t + (size_t)m128 * kg * SFA_BYTES;
  const int kb = (int)(g.k / 32);
  sf_tile_kernel<<<dim3(m128 + 2 * num_n, (kg + 31) / 32), 256, 0, stream>>>(
      static_cast<const uint8_t *>(g.sfa), (int)g.m, static_cast<const uint8_t *>(g.sfb), (int)g.n, kb,
      kg, m128, sfa_t, sfb_t);
  CUtensorMap tA = make_tmap_2d(g.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.m, g.k, g.lda, BK, BM_CTA,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.n, g.k, g.ldb, BK, Cf::NB_CTA,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tC = make_tmap_2d(g.c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.m, g.n, g.ldc, EPI_COLS,
                                32, CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap tSFA = make_tmap_2d(sfa_t, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)m128 * kg * 2,
                                  256, 256, 256, 2, CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap tSFB = make_tmap_2d(sfb_t, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)num_n * kg * 4,
                                  256, 256, 256, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
  Sched s;
  s.num_m = num_m;
  s.num_n = num_n;
  s.group = CG == 2 ? 8 : 16;
  const int tiles = num_m * num_n;
  int clusters = sm_count() / CG;
  if (clusters > tiles) clusters = tiles;
  auto kern = gemm_mxfp8_kernel<CG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG, 1, 1);
  cfg.blockDim = dim3(NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, tSFA, tSFB, (int)g.m, (int)g.n, (int)g.k, kg, s);
}

// 256 x 448 pair tiles (gemm_mxfp8_wide.cuh): same scale-atom pre-pass and
// workspace as the 256 x 224 kernel.
cudaError_t launch_wide(const Mxfp8Args &g, cudaStream_t stream) {
  const int kg = (int)((g.k + BK - 1) / BK);
  const int num_m = (int)((g.m + 255) / 256);
  const int num_n224 = (int)((g.n + BN - 1) / BN);
  const int m128 = num_m * 2;
  uint8_t *sfa_t = static_cast<uint8_t *>(g.workspace);
  uint8_t *sfb_t = sfa_t + (size_t)m128 * kg * SFA_BYTES;
  const int kb = (int)(g.k / 32);
  sf_tile_kernel<<<dim3(m128 + 2 * num_n224, (kg + 31) / 32), 256, 0, stream>>>(
      static_cast<const uint8_t *>(g.sfa), (int)g.m, static_cast<const uint8_t *>(g.sfb), (int)g.n, kb, kg, m128,
      sfa_t, sfb_t);
  CUtensorMap tA = make_tmap_2d(g.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.m, g.k, g.lda, BK, BM_CTA,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.n, g.k, g.ldb, BK, BN / 2,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tC = make_tmap_2d(g.c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.m, g.n, g.ldc, EPI_COLS, 32,
                                CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap tSFA = make_tmap_2d(sfa_t, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)m128 * kg * 2, 256, 256,
                                  256, 2, CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap tSFB = make_tmap_2d(sfb_t, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)num_n224 * kg * 4, 256, 256,
                                  256, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
  WideSched s;
  s.num_m = num_m;
  s.num_n = (int)((g.n + MW_BN - 1) / MW_BN);
  s.group = 8;
  s.clc = 1;
  s.last_partial = (g.n % MW_BN) != 0 ? 1 : 0;
  const int tiles = s.num_m * s.num_n;
  auto kern = gemm_mxfp8_wide_kernel;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, MW_SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * 2, 1, 1);  // one cluster per tile; running clusters cancel the rest (CLC)
  cfg.blockDim = dim3(MW_THREADS, 1, 1);
  cfg.dynamicSmemBytes = MW_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, tSFA, tSFB, (int)g.m, (int)g.n, (int)g.k, kg, s);
}

cudaError_t gemm_mxfp8_launch(const Mxfp8Args &g, cudaStream_t stream) {
  static const int wide_env = getenv("MIMW_FP8_WIDE") ? atoi(getenv("MIMW_FP8_WIDE")) : 0;  // A/B knob
  if (g.cta_group == 3 || (g.cta_group == 2 && wide_env != 0)) return launch_wide(g, stream);
  return g.cta_group == 1 ? launch_cg<1>(g, stream) : launch_cg<2>(g, stream);
}

}  // namespace mimw
