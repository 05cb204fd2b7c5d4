// Wide-tile dense bf16 GEMM (included by gemm_bf16.cu, inside its anonymous
// namespace): one CTA pair computes a 256 x 512 tile of C.
//
// Why: at 8192^3 both this kernel's 256 x 256 form and cuBLAS's
// nvjet_tst_256x256_64x4_2x1_2cta keep the tensor pipe ~93% busy per SM
// clock (profiles/r02/gemm_vs_cublas.md), but under the 1 kW cap the clock
// is set by power, and the narrow tile moves 8.6 GB L2 -> SM per launch
// against cuBLAS's 6.4 GB.  Staging 128 A rows against 256 B columns per CTA
// (instead of 128 x 128) cuts the L2 -> SM bytes per FLOP by 25%.
//
// The accumulator is then the whole TMEM (128 lanes x 512 fp32 columns), so
// there is no second accumulator for epilogue/main-loop overlap.  Instead
// eight epilogue warps (two per TMEM lane quarter, one per 256-column half)
// drain the accumulator into registers as packed bf16 (128 registers per
// thread), hand TMEM back at once, and store from registers (swizzled smem
// chunk -> TMA store) while the next tile's main loop runs.  The MMA warp
// waits only for the TMEM -> register drain.
//
// Roles (10 warps): warp 0 TMA producer, warp 1 MMA issuer (pair leader),
// warps 2..9 epilogue.  Per k-step of 16 the leader issues two
// tcgen05.mma.cta_group::2 M=256 N=256 (columns [0,256) and [256,512));
// CTA rank r stages pair-tile columns [h*256 + r*128, +128) of half h.
// 4-stage ring of 48 KiB (A 16 KiB + B 2 x 16 KiB).  Tiles by cluster
// launch control, as the narrow kernel (gemm_clc.mimw:1-34).

// Mutation testing (tests/test_mutation_gpu.py, the GPU form of the reference's
// barrier-deletion test, acceptance.cpp:461-485): a test build with
// -DMIMW_MUTATE_WAIT=t deletes this kernel's mbarrier wait tagged t (the tag
// is also the watchdog tag of that wait).  Product builds leave it 0.
#ifndef MIMW_MUTATE_WAIT
#define MIMW_MUTATE_WAIT 0
#endif
#define WIDE_WAIT(tag, ...)                          \
  do {                                               \
    if constexpr (MIMW_MUTATE_WAIT != (tag)) __VA_ARGS__; \
  } while (0)

// Schedule perturbation for the mutation test (the GPU stand-in for the
// reference simulator's SeededRandom scheduler, sim.cpp:252-316): a test build
// with -DMIMW_PERTURB=seed sleeps 0.5-16.5 us at a quarter of the visits of two
// sites (epilogue before draining a tile; the CLC issuer before a request), so
// the roles drift against each other far more than on an undisturbed run.
#ifdef MIMW_PERTURB
__device__ __forceinline__ void wide_perturb(uint32_t site, uint32_t t) {
  uint32_t h = site * 0x9E3779B9u ^ (t + 1u) * 0x85EBCA6Bu ^ (uint32_t)(MIMW_PERTURB)*0xC2B2AE35u ^
               (blockIdx.x + 1u) * 0x27D4EB2Fu ^ (threadIdx.x >> 5) * 0x165667B1u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  if ((h & 3) == 0) __nanosleep(500 + (h >> 8) % 16000);
}
#else
__device__ __forceinline__ void wide_perturb(uint32_t, uint32_t) {}
#endif
#ifndef MIMW_CLC_SLOTS
#define MIMW_CLC_SLOTS 4  // tile-id response ring (the mutation test also builds it with 2)
#endif

constexpr int WIDE_BN = 512;               // C columns per pair tile
constexpr int WIDE_NB_CTA = 256;           // B columns staged per CTA (two halves of 128)
constexpr int WIDE_EPI_WARPS = 8;
constexpr int WIDE_THREADS = 64 + 32 * WIDE_EPI_WARPS;
constexpr int WIDE_A_BYTES = BM_CTA * BK * 2;          // 16 KiB
constexpr int WIDE_B_BYTES = WIDE_NB_CTA * BK * 2;     // 32 KiB
constexpr int WIDE_STAGE_BYTES = WIDE_A_BYTES + WIDE_B_BYTES;
#ifndef MIMW_WIDE_STAGES
#define MIMW_WIDE_STAGES 4
#endif
constexpr int WIDE_STAGES = MIMW_WIDE_STAGES;
constexpr int WIDE_EPI_BUF = 32 * EPI_COLS * 2;        // 2 KiB: 32 rows x 32 bf16
constexpr int WIDE_EPI_BYTES = WIDE_EPI_WARPS * 2 * WIDE_EPI_BUF;
constexpr int WIDE_BAR_OFF = WIDE_STAGES * WIDE_STAGE_BYTES + WIDE_EPI_BYTES;
constexpr int WIDE_BAR_BYTES = 256;
constexpr int WIDE_SMEM = WIDE_BAR_OFF + WIDE_BAR_BYTES + 1024;  // + align slack
static_assert(WIDE_SMEM <= 232448, "wide GEMM smem");

// Grouped (MoE) problems on the wide tile: every group's rows are cut into
// 256-row M-tiles; N-tiles outer, M-tiles inner per group, so the pairs on
// one weight panel run together and share it in L2.  A group's last tile of
// t < 256 rows is computed with swapped operands (Y^T = W^T X^T: the
// pair's two M = 256 MMAs run over the tile's 512 weight columns and N = t
// rounded to 32 tokens), so its cost follows the weight panel it streams,
// not a padded 256-row tile (swap = 0: padded; rows past m_e are clipped by
// the group's Y map).  Measured at configs[4] (tools/moe_ab.py, 50-launch
// blocks): 3.66 ms swapped, 3.96 padded, 3.80 with 256 x 256 tiles.
struct GroupedWideSched {
  static constexpr bool kGrouped = true;
  CUtensorMap y[MAX_GROUPS];
  CUtensorMap x16;                // X with 16-row boxes: a swapped tail loads only its swap_n/2 rows
  int tile_pref[MAX_GROUPS + 1];  // prefix over groups of m_tiles * num_n
  int mt[MAX_GROUPS];             // 256-row tiles of group e
  int row_off[MAX_GROUPS];
  int rows[MAX_GROUPS];
  int n_groups, num_n, clc;
  int swap;  // a group's < 256-row tail (and a group of < 256 rows) as a swapped-operand tile
  __device__ __forceinline__ int num_tiles() const { return tile_pref[n_groups]; }
  __device__ __forceinline__ TileCoord decode(int t) const {
    int a = 0, b = n_groups - 1;  // last group with tile_pref[g] <= t (empty groups have no tiles)
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (tile_pref[mid] <= t) a = mid; else b = mid - 1;
    }
    const int r = t - tile_pref[a];
    TileCoord c;
    c.e = a;
    c.mt = r % mt[a];
    c.nt = r / mt[a];
    c.row_base = row_off[a];
    c.rows = rows[a];
    const int tail = rows[a] - (mt[a] - 1) * 256;
    c.swap_n = (swap && c.mt == mt[a] - 1 && tail < 256) ? ((tail + 31) & ~31) : 0;
    return c;
  }
  __device__ __forceinline__ const CUtensorMap *c_map(const CUtensorMap *, int e) const { return &y[e]; }
};

template <bool B_MN, typename Prob>
__global__ void __launch_bounds__(WIDE_THREADS, 1)
gemm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, int N, int K, const __grid_constant__ Prob sched) {
  constexpr bool GROUPED = Prob::kGrouped;
  constexpr uint32_t IDESC = idesc_bf16(256, 256, 0, B_MN ? 1 : 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + WIDE_BAR_OFF;
  auto full_bar = [&](int s) { return bar_base + 8 * s; };
  auto empty_bar = [&](int s) { return bar_base + 8 * (WIDE_STAGES + s); };
  const uint32_t tfull_bar = bar_base + 8 * (2 * WIDE_STAGES);
  const uint32_t tempty_bar = tfull_bar + 8;
  const uint32_t tmem_slot = tempty_bar + 8;
  constexpr int CLC_SLOTS = MIMW_CLC_SLOTS;
  constexpr uint32_t CLC_CONSUMERS = 2 * (1 + WIDE_EPI_WARPS) + 1;
  auto clc_resp = [&](int s) { return bar_base + 128 + 16 * s; };
  auto clc_full = [&](int s) { return bar_base + 128 + 16 * CLC_SLOTS + 8 * s; };
  auto clc_empty = [&](int s) { return bar_base + 128 + 24 * CLC_SLOTS + 8 * s; };
  static_assert(8 * (2 * WIDE_STAGES + 3) <= 128 && 128 + 32 * CLC_SLOTS <= WIDE_BAR_BYTES, "barriers");
  const uint32_t *tmem_slot_ptr = reinterpret_cast<const uint32_t *>(smem + WIDE_BAR_OFF + 8 * (2 * WIDE_STAGES + 2));

  const int warp = threadIdx.x / 32;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;
  const uint32_t my_leader = crank & ~1u;
  const bool leader = rank == 0;
  const int cluster = (int)cluster_id_x();
  const int nclusters = (int)nclusters_x();
  const int num_tiles = sched.num_tiles();
  const int num_k = (K + BK - 1) / BK;
  const bool clc = sched.clc != 0;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < WIDE_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(tempty_bar, WIDE_EPI_WARPS * 2);
    if (clc)
      for (int s = 0; s < CLC_SLOTS; ++s) {
        mbar_init(clc_full(s), 1);
        mbar_init(clc_empty(s), CLC_CONSUMERS);
      }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2>(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  auto next_tile = [&](int t, int u, bool arrive) -> int {
    if (!clc) return t + nclusters;
    const int slot = u % CLC_SLOTS;
    WIDE_WAIT(12, mbar_wait(clc_full(slot), (uint32_t)(u / CLC_SLOTS) & 1, 12));
    const int x = clc_query(clc_resp(slot));
    if (arrive) mbar_arrive_cluster(map_to_rank(clc_empty(slot), 0));
    return x < 0 ? num_tiles : x / 2;
  };
  auto clc_request = [&](int u) {
    const int slot = u % CLC_SLOTS;
    if (crank == 0) {
      wide_perturb(2, (uint32_t)u);
      WIDE_WAIT(13, mbar_wait_cluster(clc_empty(slot), ((uint32_t)(u / CLC_SLOTS) & 1) ^ 1, 13));
      mbar_arrive_expect_tx(clc_full(slot), 16);
      clc_try_cancel_multicast(clc_resp(slot), clc_full(slot));
    } else {
      mbar_arrive_expect_tx(clc_full(slot), 16);
    }
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full_target0 = map_to_rank(full_bar(0), my_leader);
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, true)) {
        if (clc) clc_request(u);
        const TileCoord tc = sched.decode(t);
        // swapped tail: this CTA stages tokens [swap_n/2 * rank, +swap_n/2) of the tail as the
        // MMAs' B operand (same 128-row box; the rows past it are not read by the MMA)
        const int m0 = tc.row_base + tc.mt * 256 + (int)rank * (tc.swap_n ? tc.swap_n / 2 : BM_CTA);
        const int n0 = tc.nt * WIDE_BN + (int)rank * 128;
        for (int kb = 0; kb < num_k; ++kb) {
          WIDE_WAIT(1, mbar_wait_cluster(empty_bar(stage), phase ^ 1, 1));
          const uint32_t fb = full_target0 + 8 * stage;
          // swapped tail: only the tail's swap_n / 2 X rows per CTA (16-row boxes), not a 128-row box
          const int xrows = GROUPED && tc.swap_n ? tc.swap_n / 2 : BM_CTA;
          if (leader) mbar_arrive_expect_tx(full_bar(stage), (WIDE_B_BYTES + xrows * BK * 2) * 2);
          const uint32_t sa = sbase + stage * WIDE_STAGE_BYTES;
          const uint32_t sb = sa + WIDE_A_BYTES;
          const int k0 = kb * BK;
          if constexpr (GROUPED) {
            if (tc.swap_n) {
              for (int r = 0; r < xrows; r += 16) tma_load_2d_cg2(sa + r * BK * 2, &sched.x16, fb, k0, m0 + r);
            } else {
              tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
            }
          } else {
            tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if constexpr (GROUPED) {  // W[e] through the 3-D map: (n, k, e) for [G,K,N], (k, n, e) for [G,N,K]
              if constexpr (B_MN) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
                  tma_load_3d_cg2(sb + (2 * h + j) * (64 * BK * 2), &tmB, fb, n0 + h * 256 + j * 64, k0, tc.e);
              } else {
                tma_load_3d_cg2(sb + h * (128 * BK * 2), &tmB, fb, k0, n0 + h * 256, tc.e);
              }
            } else if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tma_load_2d_cg2(sb + (2 * h + j) * (64 * BK * 2), &tmB, fb, n0 + h * 256 + j * 64, k0);
            } else {
              tma_load_2d_cg2(sb + h * (128 * BK * 2), &tmB, fb, k0, n0 + h * 256);
            }
          }
          if (++stage == WIDE_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane_id() == 0)) {
        int swap_n = 0;
        if constexpr (GROUPED) swap_n = sched.decode(t).swap_n;
        // swapped: A = W^T (the B slot; MN-major for [G,K,N]), B = the tail's X rows (the A slot)
        const uint32_t idesc = swap_n ? idesc_bf16(256, swap_n, B_MN ? 1 : 0, 0) : IDESC;
        WIDE_WAIT(2, mbar_wait_cluster(tempty_bar, acc_phase ^ 1, 2));
        tc_fence_after();
        if (lane_id() == 0) TILE_TRACE(t, 0, gtimer());
        for (int kb = 0; kb < num_k; ++kb) {
          WIDE_WAIT(3, mbar_wait(full_bar(stage), phase, 3));
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = sbase + stage * WIDE_STAGE_BYTES;
            const uint32_t sb = sa + WIDE_A_BYTES;
            const uint64_t adesc = smem_desc_sw128(sa, 16, 1024);
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t a_k = adesc + (uint64_t)((k * UMMA_K * 2) >> 4);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t bdesc = B_MN ? smem_desc_sw128(sb + h * (128 * BK * 2), 64 * BK * 2, 1024)
                                            : smem_desc_sw128(sb + h * (128 * BK * 2), 16, 1024);
                const uint64_t b_k = bdesc + (uint64_t)(B_MN ? ((k * UMMA_K * 128) >> 4) : ((k * UMMA_K * 2) >> 4));
                if (GROUPED && swap_n) mma_f16_ss<2>(tmem_base + h * 256, b_k, a_k, idesc, (kb | k) != 0);
                else mma_f16_ss<2>(tmem_base + h * 256, a_k, b_k, idesc, (kb | k) != 0);
              }
            }
            mma_commit_cg2_mc(empty_bar(stage), 0x3);
            if (kb == num_k - 1) mma_commit_cg2_mc(tfull_bar, (uint16_t)(0x3u << my_leader));
          }
          __syncwarp();
          if (++stage == WIDE_STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane_id() == 0) TILE_TRACE(t, 1, gtimer());
        acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int q = warp & 3;              // TMEM lane quarter
    const int ew = warp - 2;             // 0..7
    const int half = ew >> 2;            // 256-column half of the pair tile
    const uint32_t lane = lane_id();
    const uint32_t stage_base = sbase + WIDE_STAGES * WIDE_STAGE_BYTES + ew * 2 * WIDE_EPI_BUF;
    const uint32_t tempty_leader = map_to_rank(tempty_bar, my_leader);
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane == 0)) {
      const TileCoord tc = sched.decode(t);
      const int row0 = tc.mt * 256 + (int)rank * BM_CTA + q * 32;
      const int col0 = tc.nt * WIDE_BN + half * 256;
      WIDE_WAIT(4, mbar_wait(tfull_bar, acc_phase, 4));
      acc_phase ^= 1;
      tc_fence_after();
      wide_perturb(1, (uint32_t)t);
#ifdef MIMW_TILE_TRACE
      if (warp == 2 && leader && lane == 0) TILE_TRACE(t, 2, gtimer());
#endif
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + half * 256;
      // drain 256 fp32 columns (swapped: swap_n token columns) into 128
      // packed-bf16 registers, then release TMEM
      const int ncols = tc.swap_n ? tc.swap_n : 256;
      uint32_t pk[128];
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {
        if (ch * 16 < ncols) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(t_row + ch * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e)
            pk[ch * 8 + e] = pack_bf16(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader);
#ifdef MIMW_TILE_TRACE
      if (warp == 2 && leader && lane == 0) TILE_TRACE(t, 3, gtimer());
#endif
      const CUtensorMap *cmap = sched.c_map(&tmC, tc.e);
      if (GROUPED && tc.swap_n) {
        // swapped: TMEM lane = output feature, column = token.  Transpose 32
        // tokens x 32 features per box through smem (SWIZZLE_64B) into Y rows.
        const int feat0 = col0 + (int)rank * BM_CTA + q * 32;
        if (feat0 >= N) continue;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const int tok0 = tc.mt * 256 + ch * 32;
          if (ch * 32 < tc.swap_n && tok0 < tc.rows) {
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            const uint32_t sbuf = stage_base + buf * WIDE_EPI_BUF;
            const uint32_t cbyte = (lane & 7) * 2;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const uint32_t pc = (lane >> 3) ^ ((r >> 1) & 3);
              const uint32_t w = pk[ch * 16 + (r >> 1)];
              const uint16_t hv = (r & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xFFFF);
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(sbuf + r * 64 + pc * 16 + cbyte), "h"(hv) : "memory");
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(cmap, sbuf, feat0, tok0);
              bulk_commit();
            }
            buf ^= 1;
          }
        }
        continue;
      }
      if (row0 >= tc.rows) continue;
      // store: 32-column chunks through a swizzled 2 KiB box (SWIZZLE_64B:
      // 16-B chunk c of row r at c ^ ((r >> 1) & 3)) and a TMA store
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        if (col0 + ch * EPI_COLS < N) {
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const uint32_t sbuf = stage_base + buf * WIDE_EPI_BUF;
          const uint32_t rbase = sbuf + lane * 64;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t pc = (uint32_t)c ^ ((lane >> 1) & 3);
            st_shared_v4(rbase + pc * 16, pk[ch * 16 + 4 * c], pk[ch * 16 + 4 * c + 1], pk[ch * 16 + 4 * c + 2],
                         pk[ch * 16 + 4 * c + 3]);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(cmap, sbuf, col0 + ch * EPI_COLS, row0);
            bulk_commit();
          }
          buf ^= 1;
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem_base, 512);
  }
}

template <bool B_MN, typename Prob>
cudaError_t launch_wide_kernel(const CUtensorMap &tA, const CUtensorMap &tB, const CUtensorMap &tC, int n, int k,
                               const Prob &s, int tiles, int max_clusters, int clc, cudaStream_t stream) {
  auto kern = gemm_wide_kernel<B_MN, Prob>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, WIDE_SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(WIDE_THREADS, 1, 1);
  cfg.dynamicSmemBytes = WIDE_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = clc ? tiles : std::min(tiles, sm_count() / 2);
  if (!clc && max_clusters > 0) clusters = std::min(clusters, max_clusters);
  if (clusters <= 0) return cudaSuccess;
  cfg.gridDim = dim3(clusters * 2, 1, 1);
  return cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, n, k, s);
}

template <bool B_MN>
cudaError_t launch_wide(const GemmArgs &g, cudaStream_t stream, int clc) {
  CUtensorMap tA = make_tmap_2d(g.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.m, g.k, g.lda, BK, BM_CTA,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = B_MN ? make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.k, g.n, g.ldb, 64, BK,
                                       CU_TENSOR_MAP_SWIZZLE_128B)
                        : make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.n, g.k, g.ldb, BK, 128,
                                       CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tC = make_c_map<__nv_bfloat16>(g.c, g.m, g.n, g.ldc);
  Sched s;
  s.num_m = (int)((g.m + 255) / 256);
  s.num_n = (int)((g.n + WIDE_BN - 1) / WIDE_BN);
  s.group = g.raster_group > 0 ? g.raster_group : 8;
  s.M = (int)g.m;
  s.clc = clc;
  const int tiles = s.num_m * s.num_n;
  return launch_wide_kernel<B_MN>(tA, tB, tC, (int)g.n, (int)g.k, s, tiles, g.max_clusters, clc, stream);
}
