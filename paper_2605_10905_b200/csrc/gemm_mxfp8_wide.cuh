// Wide-tile MXFP8 GEMM (included by gemm_mxfp8.cu inside its anonymous
// namespace): one CTA pair computes a 256 x 448 tile as two 224-column
// sub-tiles, the bf16 wide kernel's layout (gemm_wide.cuh) applied to the
// block-scaled FP8 MMA.
//
// Per CTA and 128-byte K block, the 256 x 224 kernel stages 16 KiB of A and
// 14 KiB of B for 128 x 224 outputs (67 B per SM clock at the FP8 rate); this
// one stages 16 KiB of A and 2 x 14 KiB of B for 128 x 448 outputs (49 B per
// clock), so the L2 -> SM stream and its power drop by 27% per FLOP.
// TMEM: the 448-column accumulator [0, 448) (sub-tile s at 224 s) and a
// double-buffered scale-factor area at 448 + 32 b (SFA 4 columns, then the
// two sub-tiles' SFB atoms at +4 and +12).  The accumulator is drained into
// registers as packed bf16 by 8 epilogue warps (two per TMEM lane quarter,
// one per sub-tile) and stored while the next tile's main loop runs.
// N = 8192 is 18 full tiles and one of 128 columns, whose second sub-tile is
// skipped (no MMA, no store).  Tiles by cluster launch control.

constexpr int MW_BN = 2 * BN;              // 448 output columns per pair tile
constexpr int MW_EPI_WARPS = 8;
constexpr int MW_THREADS = 64 + 32 * MW_EPI_WARPS;
constexpr int MW_A_BYTES = BM_CTA * BK;                // 16 KiB
constexpr int MW_B_SUB = (BN / 2) * BK;                // 14 KiB: 112 B rows of one sub-tile
constexpr int MW_STAGE_BYTES = MW_A_BYTES + 2 * MW_B_SUB;
constexpr int MW_STAGES = 4;
constexpr int MW_SF_STAGE = SFA_BYTES + 2 * SFB_BYTES;  // 2.5 KiB
constexpr int MW_SF_OFF = MW_STAGES * MW_STAGE_BYTES;
constexpr int MW_EPI_OFF = MW_SF_OFF + MW_STAGES * MW_SF_STAGE;
constexpr int MW_EPI_BUF = 32 * EPI_COLS * 2;           // 2 KiB
constexpr int MW_BAR_OFF = MW_EPI_OFF + MW_EPI_WARPS * 2 * MW_EPI_BUF;
constexpr int MW_SMEM = MW_BAR_OFF + 256 + 1024;
static_assert(MW_STAGE_BYTES % 1024 == 0 && MW_SF_OFF % 1024 == 0, "stage alignment");
static_assert(MW_SMEM <= 232448, "wide MXFP8 smem");
constexpr uint32_t MW_TM_SF = 448;

struct WideSched {
  int num_m, num_n, group, clc;  // num_m in 256-row tiles, num_n in 448-column tiles
  int last_partial;              // the last column tile is narrower: dispatch its tiles last
  __device__ __forceinline__ void tile(int t, int &mt, int &nt) const {
    const int nfull = last_partial ? num_n - 1 : num_n;
    if (t >= num_m * nfull) {  // the partial column tiles (cheaper) fill the last wave
      mt = t - num_m * nfull;
      nt = num_n - 1;
      return;
    }
    const int per_group = group * nfull;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gsize = min(num_m - first_m, group);
    const int r = t - g * per_group;
    mt = first_m + r % gsize;
    nt = r / gsize;
  }
};

__global__ void __launch_bounds__(MW_THREADS, 1)
gemm_mxfp8_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmSFA,
                       const __grid_constant__ CUtensorMap tmSFB, int M, int N, int K, int KG, WideSched sched) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + MW_BAR_OFF;
  auto full_bar = [&](int s) { return bar_base + 8 * s; };
  auto empty_bar = [&](int s) { return bar_base + 8 * (MW_STAGES + s); };
  const uint32_t tfull_bar = bar_base + 8 * (2 * MW_STAGES);
  const uint32_t tempty_bar = tfull_bar + 8;
  const uint32_t tmem_slot = tempty_bar + 8;
  constexpr int CLC_SLOTS = 4;
  constexpr uint32_t CLC_CONSUMERS = 2 * (1 + MW_EPI_WARPS) + 1;
  auto clc_resp = [&](int s) { return bar_base + 128 + 16 * s; };
  auto clc_full = [&](int s) { return bar_base + 192 + 8 * s; };
  auto clc_empty = [&](int s) { return bar_base + 224 + 8 * s; };
  const uint32_t *tmem_slot_ptr = reinterpret_cast<const uint32_t *>(smem + MW_BAR_OFF + 8 * (2 * MW_STAGES + 2));

  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = (int)cluster_id_x();
  const int nclusters = (int)nclusters_x();
  const int num_tiles = sched.num_m * sched.num_n;
  const int num_k = (K + BK - 1) / BK;
  const bool clc = sched.clc != 0;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    tma_prefetch_desc(&tmSFA);
    tma_prefetch_desc(&tmSFB);
    for (int s = 0; s < MW_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(tempty_bar, MW_EPI_WARPS * 2);
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
    mbar_wait(clc_full(slot), (uint32_t)(u / CLC_SLOTS) & 1, 12);
    const int x = clc_query(clc_resp(slot));
    if (arrive) mbar_arrive_cluster(map_to_rank(clc_empty(slot), 0));
    return x < 0 ? num_tiles : x / 2;
  };
  auto clc_request = [&](int u) {
    const int slot = u % CLC_SLOTS;
    if (rank == 0) {
      mbar_wait_cluster(clc_empty(slot), ((uint32_t)(u / CLC_SLOTS) & 1) ^ 1, 13);
      mbar_arrive_expect_tx(clc_full(slot), 16);
      clc_try_cancel_multicast(clc_resp(slot), clc_full(slot));
    } else {
      mbar_arrive_expect_tx(clc_full(slot), 16);
    }
  };
  // sub-tile s of column tile nt has any column < N
  auto sub_live = [&](int nt, int s) { return nt * MW_BN + s * BN < N; };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = map_to_rank(full_bar(0), 0);
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, true)) {
        if (clc) clc_request(u);
        int mt, nt;
        sched.tile(t, mt, nt);
        const int m128 = mt * 2 + (int)rank;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait_cluster(empty_bar(stage), phase ^ 1, 1);
          const uint32_t fb = full0 + 8 * stage;
          if (leader) mbar_arrive_expect_tx(full_bar(stage), 2 * (MW_STAGE_BYTES + MW_SF_STAGE));
          const uint32_t sa = sbase + stage * MW_STAGE_BYTES;
          const uint32_t ssf = sbase + MW_SF_OFF + stage * MW_SF_STAGE;
          tma_load_2d_cg2(sa, &tmA, fb, kb * BK, m128 * BM_CTA);
          tma_load_2d_cg2(ssf, &tmSFA, fb, 0, (m128 * KG + kb) * 2);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int t224 = 2 * nt + s;  // the 224-column tile (scale atoms are laid out per 224 columns)
            tma_load_2d_cg2(sa + MW_A_BYTES + s * MW_B_SUB, &tmB, fb, kb * BK, t224 * BN + (int)rank * (BN / 2));
            tma_load_2d_cg2(ssf + SFA_BYTES + s * SFB_BYTES, &tmSFB, fb, 0, (t224 * KG + kb) * 4);
          }
          if (++stage == MW_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0, sf_buf = 0;
      constexpr uint32_t HI_SW128 = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane_id() == 0)) {
        int mt, nt;
        sched.tile(t, mt, nt);
        const bool live1 = sub_live(nt, 1);
        mbar_wait_cluster(tempty_bar, acc_phase ^ 1, 2);
        tc_fence_after();
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(full_bar(stage), phase, 3);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = sbase + stage * MW_STAGE_BYTES;
            const uint32_t ssf = sbase + MW_SF_OFF + stage * MW_SF_STAGE;
            const uint32_t tsf = tmem_base + MW_TM_SF + sf_buf * 32;
            tmem_cp_32x128b_warpx4<2>(tsf, smem_desc_noswz(ssf, 128, 128));
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              tmem_cp_32x128b_warpx4<2>(tsf + 4 + 8 * s, smem_desc_noswz(ssf + SFA_BYTES + s * SFB_BYTES, 128, 128));
              tmem_cp_32x128b_warpx4<2>(tsf + 8 + 8 * s,
                                        smem_desc_noswz(ssf + SFA_BYTES + s * SFB_BYTES + 512, 128, 128));
            }
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              uint64_t ad;
              asm volatile("mov.b64 %0, {%1, %2};" : "=l"(ad) : "r"(LO_KMAJ | ((sa + k * 32) >> 4)), "r"(HI_SW128));
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                if (s == 1 && !live1) continue;
                uint64_t bd;
                asm volatile("mov.b64 %0, {%1, %2};"
                             : "=l"(bd)
                             : "r"(LO_KMAJ | ((sa + MW_A_BYTES + s * MW_B_SUB + k * 32) >> 4)), "r"(HI_SW128));
                mma_mxf8_ss<2>(tmem_base + s * BN, ad, bd, idesc_mxf8(BM_CTA * 2, BN, k, k), tsf, tsf + 4 + 8 * s,
                               (kb | k) != 0);
              }
            }
            mma_commit_cg2_mc(empty_bar(stage), 0x3);
            if (kb == num_k - 1) mma_commit_cg2_mc(tfull_bar, 0x3);
          }
          __syncwarp();
          sf_buf ^= 1;
          if (++stage == MW_STAGES) { stage = 0; phase ^= 1; }
        }
        acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue: drain 224 columns into registers, store ----------------
    const int q = warp & 3;
    const int ew = warp - 2;
    const int s = ew >> 2;  // sub-tile
    const uint32_t lane = lane_id();
    const uint32_t stage_base = sbase + MW_EPI_OFF + ew * 2 * MW_EPI_BUF;
    const uint32_t tempty_leader = map_to_rank(tempty_bar, 0);
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane == 0)) {
      int mt, nt;
      sched.tile(t, mt, nt);
      const int row0 = (mt * 2 + (int)rank) * BM_CTA + q * 32;
      const int col0 = nt * MW_BN + s * BN;
      mbar_wait(tfull_bar, acc_phase, 4);
      acc_phase ^= 1;
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + s * BN;
      const bool live = col0 < N;
      uint32_t pk[BN / 2];  // 112 packed bf16 pairs
      if (live) {
#pragma unroll
        for (int ch = 0; ch < BN / 16; ++ch) {
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
      if (!live || row0 >= M) continue;
#pragma unroll
      for (int ch = 0; ch < BN / EPI_COLS; ++ch) {
        if (col0 + ch * EPI_COLS < N) {
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const uint32_t sbuf = stage_base + buf * MW_EPI_BUF;
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
            tma_store_2d(&tmC, sbuf, col0 + ch * EPI_COLS, row0);
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
