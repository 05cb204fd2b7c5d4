// Block-scaled FP8 (MXFP8: e4m3 values, one UE8M0 scale per 32 K-elements)
// persistent warp-specialized GEMM for sm_100a:
//     C[M,N] (bf16) = sum_k  A[m,k] * 2^(sfa[m,k/32]-127) * B[n,k] * 2^(sfb[n,k/32]-127)
//
// The reference has no FP8; the oracle for this path is
// oracle_gemm (proj/core/src/oracles.cpp:14-26) on the dequantised f32 Tiles
// (oracle/oracle.c orc_mx_dequant).  Same MIMW roles as gemm_bf16.cu:
//   warp 0      TMA producer: A/B tiles (cp.async.bulk.tensor, 128-B swizzle)
//               and the stage's scale-factor atoms (cp.async.bulk), one
//               mbarrier per stage with the total byte count
//   warp 1      TMEM allocator + MMA issuer: tcgen05.cp moves the stage's
//               scale factors smem -> TMEM (32x128b.warpx4), then 4 x
//               tcgen05.mma.kind::mxf8f6f4.block_scale (K = 32 each, sf_id
//               selects the k-block byte), commit frees the smem slot
//   warps 2..5  epilogue: TMEM -> bf16 -> swizzled smem -> TMA store
// Scale factors in TMEM (found with tools/sf_probe.cu): row m of A reads lane
// m, column (m >> 5), byte sf_id; column n of B reads lane (n & 31), column
// (n >> 5), byte sf_id.  The 512-byte "atom" [r*16 + c*4 + y] = sf(row 32c+r,
// kblock y) is exactly what one tcgen05.cp.32x128b.warpx4 consumes; a small
// pre-pass (sf_tile_kernel) reorders the natural [rows, K/32] scale arrays
// into per-tile atoms.
//
// Tile 128 x 224 x 128 (cta_group::1): two fp32 accumulators (2 x 224
// columns) + double-buffered scale factors fit the 512 TMEM columns.
#include "gemm_mxfp8.h"
#include "ptx.cuh"
#include "tma_host.h"

#include <algorithm>

namespace mimw {

namespace {

constexpr int BM = 128;
constexpr int BN = 224;          // 7 x 32 columns
constexpr int BK = 128;          // fp8 bytes per 128-B swizzle row = 4 scale blocks
constexpr int UMMA_K = 32;
constexpr int STAGES = 4;
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_COLS = 32;
constexpr int A_BYTES = BM * BK;                 // 16 KiB
constexpr int B_BYTES = BN * BK;                 // 28 KiB
constexpr int SFA_BYTES = 512;                   // one atom: 128 rows x 4 k-blocks
constexpr int SFB_BYTES = 1024;                  // two atoms: 256 (>= 224) columns
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 44 KiB, 1024-B aligned
constexpr int SF_STAGE = SFA_BYTES + SFB_BYTES;  // scale-factor atoms of one stage
constexpr int SF_OFF = STAGES * STAGE_BYTES;
constexpr int EPI_BUF = 32 * EPI_COLS * 2;       // bf16
constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_BUF;
constexpr int EPI_OFF = SF_OFF + STAGES * SF_STAGE;
constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
constexpr int SMEM = BAR_OFF + 256 + 1024;
constexpr uint32_t TM_ACC = 0;                   // 2 x 224 columns
constexpr uint32_t TM_SF = 448;                  // per SF buffer: SFA 4 cols + SFB 8 cols
constexpr uint32_t SF_STRIDE = 16;

static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1024-B aligned for SWIZZLE_128B");

struct Sched {
  int num_m, num_n, group, kg;  // kg = K / 128 (scale-factor atoms per tile row)
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

__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_mxfp8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const uint8_t *__restrict__ sfa_t,
                  const uint8_t *__restrict__ sfb_t, int M, int N, int K, Sched sched) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + BAR_OFF;
  auto full_bar = [&](int s) { return bar_base + 8 * s; };
  auto empty_bar = [&](int s) { return bar_base + 8 * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar_base + 8 * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar_base + 8 * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bar_base + 8 * (2 * STAGES + 4);
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + BAR_OFF + 8 * (2 * STAGES + 4));

  const int warp = threadIdx.x / 32;
  const int num_tiles = sched.num_m * sched.num_n;
  const int num_k = (K + BK - 1) / BK;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mt, nt;
        sched.tile(t, mt, nt);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1, 1);
          mbar_arrive_expect_tx(full_bar(stage), STAGE_BYTES + SF_STAGE);
          const uint32_t sa = sbase + stage * STAGE_BYTES;
          const uint32_t sb = sa + A_BYTES;
          const uint32_t ssf = sbase + SF_OFF + stage * SF_STAGE;
          tma_load_2d(sa, &tmA, full_bar(stage), kb * BK, mt * BM);
          tma_load_2d(sb, &tmB, full_bar(stage), kb * BK, nt * BN);
          bulk_load(ssf, sfa_t + ((size_t)mt * sched.kg + kb) * SFA_BYTES, SFA_BYTES, full_bar(stage));
          bulk_load(ssf + SFA_BYTES, sfb_t + ((size_t)nt * sched.kg + kb) * SFB_BYTES, SFB_BYTES,
                    full_bar(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t sf_buf = 0;  // TMEM scale-factor double buffer (runs across tiles)
    constexpr uint32_t HI_SW128 = (1024u >> 4) | (1u << 14) | (2u << 29);
    constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      mbar_wait(tempty_bar(acc), acc_phase ^ 1, 2);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + TM_ACC + acc * BN;
      for (int kb = 0; kb < num_k; ++kb) {
        mbar_wait(full_bar(stage), phase, 3);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = sbase + stage * STAGE_BYTES;
          const uint32_t sb = sa + A_BYTES;
          const uint32_t ssf = sbase + SF_OFF + stage * SF_STAGE;
          const uint32_t tsf = tmem_base + TM_SF + sf_buf * SF_STRIDE;
          // scale factors smem -> TMEM (ordered before the MMAs in the tensor pipe)
          tmem_cp_32x128b_warpx4(tsf, smem_desc_noswz(ssf, 128, 128));
          tmem_cp_32x128b_warpx4(tsf + 4, smem_desc_noswz(ssf + SFA_BYTES, 128, 128));
          tmem_cp_32x128b_warpx4(tsf + 8, smem_desc_noswz(ssf + SFA_BYTES + 512, 128, 128));
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            uint64_t ad, bd;
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(ad) : "r"(LO_KMAJ | ((sa + k * 32) >> 4)), "r"(HI_SW128));
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(bd) : "r"(LO_KMAJ | ((sb + k * 32) >> 4)), "r"(HI_SW128));
            mma_mxf8_ss<1>(d_tmem, ad, bd, idesc_mxf8(BM, BN, k, k), tsf, tsf + 4, (kb | k) != 0);
          }
          mma_commit(empty_bar(stage));
          if (kb == num_k - 1) mma_commit(tfull_bar(acc));
        }
        __syncwarp();
        sf_buf ^= 1;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const int ew = warp - 2;
    const uint32_t lane = lane_id();
    const uint32_t stage_base = sbase + EPI_OFF + ew * 2 * EPI_BUF;
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mt, nt;
      sched.tile(t, mt, nt);
      const int row0 = mt * BM + q * 32;
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
          if (lane == 0) mbar_arrive(tempty_bar(acc));
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
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

// Reorder natural [rows, kb] UE8M0 scales into per-tile atoms:
//   atom(tile, kg, half)[r*16 + c*4 + y] = sf[tile*rows_per_tile + half*128 + 32c + r, 4kg + y]
// (127 = 1.0 outside the matrix).  One thread per output byte.
__global__ void sf_tile_kernel(const uint8_t *__restrict__ sf, int rows, int kb, int rows_per_tile,
                               int halves, int tiles, int kg, uint8_t *__restrict__ out) {
  const int64_t total = (int64_t)tiles * kg * halves * 512;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int byte = (int)(i & 511);
    int64_t atom = i >> 9;
    const int half = (int)(atom % halves);
    atom /= halves;
    const int g = (int)(atom % kg);
    const int tile = (int)(atom / kg);
    const int r = byte >> 4, c = (byte >> 2) & 3, y = byte & 3;
    const int local = half * 128 + 32 * c + r;
    const int row = tile * rows_per_tile + local;
    const int k = 4 * g + y;
    uint8_t v = 127;
    if (local < rows_per_tile && row < rows && k < kb) v = sf[(size_t)row * kb + k];
    out[i] = v;
  }
}

}  // namespace

size_t gemm_mxfp8_workspace(int64_t m, int64_t n, int64_t k) {
  const int64_t kg = (k + BK - 1) / BK;
  const int64_t mt = (m + BM - 1) / BM, nt = (n + BN - 1) / BN;
  return (size_t)(mt * kg * SFA_BYTES + nt * kg * SFB_BYTES);
}

cudaError_t gemm_mxfp8_launch(const Mxfp8Args &g, cudaStream_t stream) {
  const int kg = (int)((g.k + BK - 1) / BK);
  const int num_m = (int)((g.m + BM - 1) / BM), num_n = (int)((g.n + BN - 1) / BN);
  uint8_t *sfa_t = static_cast<uint8_t *>(g.workspace);
  uint8_t *sfb_t = sfa_t + (size_t)num_m * kg * SFA_BYTES;
  const int kb = (int)(g.k / 32);
  {
    int64_t na = (int64_t)num_m * kg * 512, nb = (int64_t)num_n * kg * 2 * 512;
    sf_tile_kernel<<<(int)std::min<int64_t>((na + 255) / 256, 4096), 256, 0, stream>>>(
        static_cast<const uint8_t *>(g.sfa), (int)g.m, kb, BM, 1, num_m, kg, sfa_t);
    sf_tile_kernel<<<(int)std::min<int64_t>((nb + 255) / 256, 4096), 256, 0, stream>>>(
        static_cast<const uint8_t *>(g.sfb), (int)g.n, kb, BN, 2, num_n, kg, sfb_t);
  }
  CUtensorMap tA = make_tmap_2d(g.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.m, g.k, g.lda, BK, BM,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.n, g.k, g.ldb, BK, BN,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tC = make_tmap_2d(g.c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.m, g.n, g.ldc, EPI_COLS,
                                32, CU_TENSOR_MAP_SWIZZLE_64B);
  Sched s;
  s.num_m = num_m;
  s.num_n = num_n;
  s.group = 16;
  s.kg = kg;
  const int tiles = num_m * num_n;
  int grid = sm_count();
  if (grid > tiles) grid = tiles;
  cudaError_t e = cudaFuncSetAttribute(gemm_mxfp8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  gemm_mxfp8_kernel<<<grid, NUM_THREADS, SMEM, stream>>>(tA, tB, tC, sfa_t, sfb_t, (int)g.m, (int)g.n,
                                                           (int)g.k, s);
  return cudaGetLastError();
}

}  // namespace mimw
