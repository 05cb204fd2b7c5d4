// Persistent warp-specialized bf16 GEMM for sm_100a:  C[M,N] = A[M,K] . B
//
// The B200 form of the reference's warp-specialized GEMM programs
//   proj/kernels/gemm_pipeline.mimw:1-62  (producer task -> smem ring guarded
//       by ready/free barriers -> consumer async_dot -> global_store)
//   proj/kernels/gemm_clc.mimw:1-34       (persistent `while tile != -1`)
//   tests/helpers.hpp:130-146             (collective_dot across a CTA pair)
// computing oracle_gemm (proj/core/src/oracles.cpp:14-26) with fp32
// accumulation in TMEM.
//
// MIMW roles (one CTA = 6 warps, one CTA per SM, CG CTAs per cluster):
//   warp 0      TMA producer: waits `empty[s]`, arms `full[s]` with the
//               stage's byte count, issues cp.async.bulk.tensor loads
//               (barrier_expect / async_copy in the reference).
//   warp 1      TMEM allocator + MMA issuer (leader CTA only): one elected
//               thread issues tcgen05.mma (cta_group::CG), tcgen05.commit
//               frees the smem slot and, per tile, fills `tmem_full[acc]`.
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> bf16/f32 ->
//               swizzled smem -> TMA store; arrive `tmem_empty[acc]` on the
//               leader so the next tile's MMAs can reuse the accumulator.
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap
// the main loop of tile i+1.
//
// CG = 2: a CTA pair runs M=256 tcgen05.mma.cta_group::2.  Each CTA stages
// its own 128 rows of A and half of B's N columns; the hardware combines
// them (the reference's collective_dot replicates B instead,
// sim.cpp:1322-1338 — same product, half the smem traffic).  All TMA loads
// of the pair complete on the leader's `full[s]`; the leader's commits are
// multicast to both CTAs' `empty[s]` / `tmem_full[acc]`.
#include "gemm_bf16.h"
#include "ptx.cuh"
#include "tma_host.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace mimw {

#ifdef MIMW_TILE_TRACE
// Per-tile timeline (tools/moe_trace.py; trace builds only): tile t ->
// {MMA start, last MMA issued, accumulator seen by the epilogue, smid}, ns.
__device__ unsigned long long *g_mimw_tile_trace;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TILE_TRACE(t, slot, v) \
  do { if (g_mimw_tile_trace) g_mimw_tile_trace[(size_t)(t) * 4 + (slot)] = (v); } while (0)
#else
#define TILE_TRACE(t, slot, v) do {} while (0)
#endif

namespace {

constexpr int BK = 64;           // K per stage (one 128-byte swizzle row of bf16)
constexpr int UMMA_K = 16;       // K per tcgen05.mma (kind::f16)
constexpr int BN = 256;          // N per MMA / per cluster tile
constexpr int BM_CTA = 128;      // rows of A per CTA
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int ACC_STAGES = 2;    // TMEM accumulators (2 x 256 columns = 512)
constexpr int EPI_COLS = 32;     // columns per epilogue store chunk

template <int CG, bool B_MN, typename OutT, bool GATHER = false>
struct Cfg {
  static constexpr int NB_CTA = BN / CG;                       // B columns staged per CTA
  static constexpr int A_BYTES = BM_CTA * BK * 2;              // 16 KiB
  static constexpr int B_BYTES = NB_CTA * BK * 2;              // 16 / 32 KiB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (CG == 2) ? 6 : 4;
  static constexpr int EPI_BUF = 32 * EPI_COLS * (int)sizeof(OutT);   // per warp per buffer
  static constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_BUF;
  static constexpr int COMM_EXTRA = GATHER ? 16384 : 0;        // distributed comm warp's buffer
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES + EPI_BYTES + COMM_EXTRA;
  static constexpr int BAR_BYTES = 384;                        // pipeline barriers + TMEM slot + CLC ring
  static constexpr int COMM_BAR_BYTES = 8 * 24 + 32;           // all-gather comm barriers + mailboxes
  static constexpr int SMEM = BAR_OFF + BAR_BYTES + COMM_BAR_BYTES + 1024;  // + align slack
  static constexpr uint32_t IDESC = idesc_bf16(BM_CTA * CG, BN, 0, B_MN ? 1 : 0);
};

// One output tile of a (possibly grouped) problem.  Row `mt * BM` of the
// group starts at A row `row_base + mt * BM`; rows at or beyond `rows` are
// not stored (C/Y map row extent).
// swap_n > 0 marks a grouped tail tile computed with swapped operands
// (Y^T = W^T X^T: M = 256 output columns, N = swap_n rows of the group).
struct TileCoord {
  int e, mt, nt, row_base, rows, swap_n;
};

// Dense problem: one [M,K] x B -> [M,N]; grouped-rasterised tile order
// (`group` M-tiles share each N sweep so B panels are re-read from L2).
template <int PAIRS>
struct SchedT {
  static constexpr bool kGrouped = false;
  static constexpr bool kGather = false;
  static constexpr bool kClc = true;
  static constexpr int kPairs = PAIRS;  // CTA pairs per cluster sharing each B tile (multicast)
  int num_m, num_n, group, M;           // num_m in cluster tiles (PAIRS M-tiles each)
  int clc;                              // tiles dispatched by cluster launch control
  __device__ __forceinline__ int num_tiles() const { return num_m * num_n; }
  __device__ __forceinline__ TileCoord decode(int t) const {
    int per_group = group * num_n;
    int g = t / per_group;
    int first_m = g * group;
    int gsize = min(num_m - first_m, group);
    int r = t - g * per_group;
    TileCoord c;
    c.e = 0;
    c.mt = first_m + r % gsize;
    c.nt = r / gsize;
    if (g & 1) c.nt = num_n - 1 - c.nt;  // boustrophedon: reuse the B panels still in L2
    c.row_base = 0;
    c.rows = M;
    c.swap_n = 0;
    return c;
  }
  __device__ __forceinline__ const CUtensorMap *c_map(const CUtensorMap *tmC, int) const { return tmC; }
};
using Sched = SchedT<1>;

// Grouped (MoE) problem: Y_e[m_e, N] = X[row_off_e : row_off_e + m_e, K] . W_e
// for e < n_groups.  X rows are packed by group; W is one [G, K, N] (or
// [G, N, K]) tensor read through a 3-D tensor map; every group has its own
// Y tensor map whose row extent m_e clips the tail tile's store.
// Tile order: the non-empty groups are visited in `order` and cut into chunks
// of consecutive slots; inside a chunk, N-tiles outer, then (group, M-tile),
// so the CTA pairs working on one weight panel W_e[:, n-tile] run at the same
// time and share it in L2, and a chunk that mixes heavy and light groups
// keeps compute-bound and weight-streaming tiles running side by side.
// One group per chunk is plain "groups in turn".
constexpr int MAX_GROUPS = 128;
struct GroupedSched {
  static constexpr bool kGrouped = true;
  static constexpr bool kGather = false;
  static constexpr bool kClc = true;
  static constexpr int kPairs = 1;
  CUtensorMap y[MAX_GROUPS];
  int order[MAX_GROUPS];           // slot -> group
  int mt_pref[MAX_GROUPS + 1];     // prefix over slots of m_tiles(group)
  int chunk_off[MAX_GROUPS + 1];   // first tile of chunk c
  int chunk_slot[MAX_GROUPS + 1];  // first slot of chunk c
  int row_off[MAX_GROUPS];         // first row of group e in X / Y
  int rows[MAX_GROUPS];            // m_e
  int n_chunks, num_n, bm;         // bm = rows per cluster tile (128 * CG)
  int swap;                        // tail tiles (< bm rows) use swapped operands (CG == 2)
  int clc;                         // tiles dispatched by cluster launch control (grid = one cluster per tile)
  int prefetch;                    // W k-blocks prefetched into L2 ahead of the TMA loads (0 = off)
  __device__ __forceinline__ int num_tiles() const { return chunk_off[n_chunks]; }
  __device__ __forceinline__ TileCoord decode(int t) const {
    int lo = 0, hi = n_chunks - 1;  // last chunk with chunk_off[c] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (chunk_off[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const int s0 = chunk_slot[lo], s1 = chunk_slot[lo + 1];
    const int per_n = mt_pref[s1] - mt_pref[s0];
    const int r = t - chunk_off[lo];
    const int q = mt_pref[s0] + r % per_n;
    int a = s0, b = s1 - 1;  // last slot with mt_pref[slot] <= q (slots are non-empty)
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (mt_pref[mid] <= q) a = mid; else b = mid - 1;
    }
    const int e = order[a];
    const int full = rows[e] / bm;
    const int tail = rows[e] - full * bm;
    TileCoord c;
    c.e = e;
    c.mt = q - mt_pref[a];
    c.nt = r / per_n;
    c.row_base = row_off[e];
    c.rows = rows[e];
    c.swap_n = (swap && c.mt == full && tail > 0) ? ((tail + 31) & ~31) : 0;
    return c;
  }
  __device__ __forceinline__ const CUtensorMap *c_map(const CUtensorMap *, int e) const { return &y[e]; }
};


#include "gemm_gather.cuh"

// all-gather GEMM CTAs carry two more warps: 6 = comm agent, 7 = signaler
template <typename Prob>
constexpr int kernel_threads() { return Prob::kGather ? NUM_THREADS + 64 : NUM_THREADS; }

template <int CG, bool B_MN, typename OutT, typename Prob>
__global__ void __launch_bounds__(kernel_threads<Prob>(), 1)
gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, int N, int K,
                 const __grid_constant__ Prob sched) {
  using C = Cfg<CG, B_MN, OutT, Prob::kGather>;
  constexpr bool GROUPED = Prob::kGrouped;
  // PAIRS = 2: a cluster of two CTA pairs computes two vertically adjacent
  // 256x256 tiles; each B half-tile is loaded once and multicast to the
  // same-rank CTA of both pairs (half the L2->smem traffic for B).
  constexpr int PAIRS = Prob::kPairs;
  static_assert(PAIRS == 1 || CG == 2, "multicast pairs need cta_group::2");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + C::BAR_OFF;
  auto full_bar = [&](int s) { return bar_base + 8 * s; };
  auto empty_bar = [&](int s) { return bar_base + 8 * (C::STAGES + s); };
  auto tfull_bar = [&](int a) { return bar_base + 8 * (2 * C::STAGES + a); };
  auto tempty_bar = [&](int a) { return bar_base + 8 * (2 * C::STAGES + ACC_STAGES + a); };
  const uint32_t tmem_slot = bar_base + 8 * (2 * C::STAGES + 2 * ACC_STAGES);
  // CLC response ring (gemm_clc.mimw's clc_producer / clc_consumer): slot s =
  // 16-byte response + full barrier (completed by the response bytes) + empty
  // barrier on the pair leader (released by every consumer of both CTAs)
  constexpr int CLC_SLOTS = 4;
  // consumers: every CTA's producer and epilogue warps, and each pair leader's MMA warp
  constexpr uint32_t CLC_CONSUMERS = CG * Prob::kPairs * (1 + EPI_WARPS) + Prob::kPairs;
  auto clc_resp = [&](int s) { return bar_base + 256 + 16 * s; };
  auto clc_full = [&](int s) { return bar_base + 256 + 16 * CLC_SLOTS + 8 * s; };
  auto clc_empty = [&](int s) { return bar_base + 256 + 24 * CLC_SLOTS + 8 * s; };
  static_assert(256 + 32 * CLC_SLOTS <= C::BAR_BYTES, "CLC ring");
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + C::BAR_OFF + 8 * (2 * C::STAGES + 2 * ACC_STAGES));

  const int warp = threadIdx.x / 32;
  const uint32_t crank = (CG == 2) ? cluster_ctarank() : 0;
  const uint32_t rank = crank & (CG - 1);   // rank inside the CTA pair
  const int pair = (int)(crank >> 1);       // pair inside the cluster (PAIRS == 2)
  const uint32_t my_leader = crank & ~1u;
  const bool leader = (rank == 0);
  int cluster = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
  int nclusters = (CG == 2) ? (int)nclusters_x() : (int)gridDim.x;
  const int num_tiles = sched.num_tiles();
  int num_k = (K + BK - 1) / BK;
  bool clc = false;
  if constexpr (Prob::kClc) clc = sched.clc != 0;
  bool comm = false;  // all-gather GEMM: the low cluster ids are comm pairs
  if constexpr (Prob::kGather) {
    static_assert(CG == 2 && B_MN && PAIRS == 1, "all-gather GEMM: 2-CTA, B as [K, N]");
    comm = cluster < sched.comm_clusters;
    cluster -= sched.comm_clusters;
    nclusters -= sched.comm_clusters;
    num_k = sched.kblocks;
  }

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), PAIRS);
    }
    for (int a = 0; a < ACC_STAGES; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), EPI_WARPS * CG);
    }
    if (clc)
      for (int s = 0; s < CLC_SLOTS; ++s) {
        mbar_init(clc_full(s), 1);
        mbar_init(clc_empty(s), CLC_CONSUMERS);
      }
    if constexpr (Prob::kGather)
      for (int i = 0; i < 8; ++i)  // comm mailboxes
        st_release_cta_shared(bar_base + C::BAR_BYTES + 8 * COMM_MAX_BUFS + 4 * i, 0u);
    fence_mbar_init();
  }
  if (warp == 1 && !comm) tmem_alloc<CG>(tmem_slot, 512);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  // Next tile after tile t (use index u): static striding, or the u-th CLC
  // response (the cancelled cluster's tile; num_tiles once the grid is
  // exhausted).  Every consumer reads every response, `arrive` once per warp.
  auto next_tile = [&](int t, int u, bool arrive) -> int {
    if (!clc) return t + nclusters;
    const int slot = u % CLC_SLOTS;
    mbar_wait(clc_full(slot), (uint32_t)(u / CLC_SLOTS) & 1, 12);
    const int x = clc_query(clc_resp(slot));
    if (arrive) {
      if constexpr (CG == 2) mbar_arrive_cluster(map_to_rank(clc_empty(slot), 0));  // on cluster rank 0
      else mbar_arrive(clc_empty(slot));
    }
    return x < 0 ? num_tiles : x / (CG * PAIRS);
  };
  // Producer, at the start of tile u: cluster rank 0 asks for tile u + 1
  // (multicast to every CTA of the cluster); each CTA arms its own full barrier.
  auto clc_request = [&](int u) {
    const int slot = u % CLC_SLOTS;
    if (crank == 0) {
      mbar_wait_cluster(clc_empty(slot), ((uint32_t)(u / CLC_SLOTS) & 1) ^ 1, 13);
      mbar_arrive_expect_tx(clc_full(slot), 16);
      if constexpr (CG == 2) clc_try_cancel_multicast(clc_resp(slot), clc_full(slot));
      else clc_try_cancel(clc_resp(slot), clc_full(slot));
    } else {
      mbar_arrive_expect_tx(clc_full(slot), 16);
    }
  };

  if (comm) {
    if constexpr (Prob::kGather)
      gather_comm_cta(sched, sbase, C::STAGES * C::STAGE_BYTES, bar_base + C::BAR_BYTES,
                      bar_base + C::BAR_BYTES + 8 * COMM_MAX_BUFS,
                      (cluster + sched.comm_clusters) * CG + (int)crank, sched.comm_clusters * CG);
  } else if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full_target0 = (CG == 2) ? map_to_rank(full_bar(0), my_leader) : full_bar(0);
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, true)) {
        if (clc) clc_request(u);
        const TileCoord tc = sched.decode(t);
        // swapped tail tile: this CTA stages rows [swap_n/2 * rank, +swap_n/2) of the
        // group's tail as the MMA's B operand (same 128-row box; extra rows unused)
        const int m0 = tc.row_base + (tc.mt * PAIRS + pair) * BM_CTA * CG +
                       (int)rank * (tc.swap_n ? tc.swap_n / 2 : BM_CTA);
        const int n0 = tc.nt * BN + (int)rank * C::NB_CTA;
        if constexpr (Prob::kGather) {
          // splits in rotation order; remote slabs gated on their counters
          for (int q = 0; q < sched.nsplit; ++q) {
            const int nk = (sched.ks[q] + BK - 1) / BK;
            for (int kb = 0; kb < nk; ++kb) {
              if (q > 0 && kb % (COMM_SLAB / BK) == 0) {
                const int j = kb / (COMM_SLAB / BK);
                flag_wait_geq<false>(sched.ctr + q * sched.max_slabs + j, sched.pieces(q, j), 25);
                fence_proxy_async_global();
              }
              mbar_wait_cluster(empty_bar(stage), phase ^ 1, 1);
              const uint32_t fb = full_target0 + 8 * stage;
              if (leader) mbar_arrive_expect_tx(full_bar(stage), C::STAGE_BYTES * CG);
              const uint32_t sa = sbase + stage * C::STAGE_BYTES;
              const uint32_t sb = sa + C::A_BYTES;
              const int k0 = kb * BK;
              tma_load_2d_cg2(sa, &sched.ga[q], fb, k0, m0);
#pragma unroll
              for (int j = 0; j < C::NB_CTA / 64; ++j)
                tma_load_2d_cg2(sb + j * (64 * BK * 2), &sched.gb[q], fb, n0 + j * 64, k0);
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        } else {
        for (int kb = 0; kb < num_k; ++kb) {
          if constexpr (CG == 2) mbar_wait_cluster(empty_bar(stage), phase ^ 1, 1);
          else mbar_wait(empty_bar(stage), phase ^ 1, 1);
          const uint32_t fb = full_target0 + 8 * stage;
          if (leader) mbar_arrive_expect_tx(full_bar(stage), C::STAGE_BYTES * CG);
          const uint32_t sa = sbase + stage * C::STAGE_BYTES;
          const uint32_t sb = sa + C::A_BYTES;
          const int k0 = kb * BK;
          if constexpr (GROUPED) {
            // Weight panels stream from DRAM once per group, and each CTA keeps
            // only ~96 KiB of them in flight, so the loads run at the
            // latency-bound per-SM rate (tools/moe_trace.py).  Warm L2 `prefetch`
            // k-blocks ahead of the ring instead.
            if (sched.prefetch > 0) {
              const int k_lo = kb == 0 ? 0 : kb + sched.prefetch - 1;
              const int k_hi = min(num_k - 1, kb + sched.prefetch - 1);
              for (int kp = k_lo; kp <= k_hi; ++kp) {
                if constexpr (B_MN) {
#pragma unroll
                  for (int j = 0; j < C::NB_CTA / 64; ++j) tma_prefetch_l2_3d(&tmB, n0 + j * 64, kp * BK, tc.e);
                } else {
                  tma_prefetch_l2_3d(&tmB, kp * BK, n0, tc.e);
                }
              }
            }
            // W[e] through the 3-D map: (n, k, e) for [G,K,N], (k, n, e) for [G,N,K]
            if constexpr (CG == 2) tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
            else tma_load_2d(sa, &tmA, fb, k0, m0);
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < C::NB_CTA / 64; ++j) {
                if constexpr (CG == 2) tma_load_3d_cg2(sb + j * (64 * BK * 2), &tmB, fb, n0 + j * 64, k0, tc.e);
                else tma_load_3d(sb + j * (64 * BK * 2), &tmB, fb, n0 + j * 64, k0, tc.e);
              }
            } else {
              if constexpr (CG == 2) tma_load_3d_cg2(sb, &tmB, fb, k0, n0, tc.e);
              else tma_load_3d(sb, &tmB, fb, k0, n0, tc.e);
            }
          } else if constexpr (PAIRS == 2) {
            tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
            if (pair == (int)rank) {  // one issuer per B half, multicast to both pairs
              const uint16_t mask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
              if constexpr (B_MN) {
#pragma unroll
                for (int j = 0; j < C::NB_CTA / 64; ++j)
                  tma_load_2d_cg2_mc(sb + j * (64 * BK * 2), &tmB, fb, n0 + j * 64, k0, mask);
              } else {
                tma_load_2d_cg2_mc(sb, &tmB, fb, k0, n0, mask);
              }
            }
          } else if constexpr (CG == 2) {
            tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < C::NB_CTA / 64; ++j)
                tma_load_2d_cg2(sb + j * (64 * BK * 2), &tmB, fb, n0 + j * 64, k0);
            } else {
              tma_load_2d_cg2(sb, &tmB, fb, k0, n0);
            }
          } else {
            tma_load_2d(sa, &tmA, fb, k0, m0);
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < C::NB_CTA / 64; ++j)
                tma_load_2d(sb + j * (64 * BK * 2), &tmB, fb, n0 + j * 64, k0);
            } else {
              tma_load_2d(sb, &tmB, fb, k0, n0);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        }  // !kGather
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane_id() == 0)) {
        int swap_n = 0;
        if constexpr (GROUPED) swap_n = sched.decode(t).swap_n;
        // swapped tail: A = W^T (the B slot, MN-major for [G,K,N]), B = X rows (the A slot)
        const uint32_t idesc = swap_n ? idesc_bf16(BM_CTA * CG, swap_n, B_MN ? 1 : 0, 0) : C::IDESC;
        mbar_wait_cluster(tempty_bar(acc), acc_phase ^ 1, 2);
        tc_fence_after();
        if (lane_id() == 0) TILE_TRACE(t, 0, gtimer());
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(full_bar(stage), phase, 3);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = sbase + stage * C::STAGE_BYTES;
            const uint32_t sb = sa + C::A_BYTES;
            const uint64_t adesc = smem_desc_sw128(sa, 16, 1024);
            const uint64_t bdesc = B_MN ? smem_desc_sw128(sb, 64 * BK * 2, 1024)
                                        : smem_desc_sw128(sb, 16, 1024);
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              // K-major A: +32 B per K=16 inside the 128-B swizzle row.
              // MN-major B: +16 rows x 128 B per K=16.  K-major B: +32 B.
              const uint64_t a_k = adesc + (uint64_t)((k * UMMA_K * 2) >> 4);
              const uint64_t b_k = bdesc + (uint64_t)(B_MN ? ((k * UMMA_K * 128) >> 4)
                                                          : ((k * UMMA_K * 2) >> 4));
              if (GROUPED && swap_n) mma_f16_ss<CG>(d_tmem, b_k, a_k, idesc, (kb | k) != 0);
              else mma_f16_ss<CG>(d_tmem, a_k, b_k, idesc, (kb | k) != 0);
            }
            if constexpr (CG == 2) {
              // a stage is free once every pair that received its B has consumed it
              mma_commit_cg2_mc(empty_bar(stage), PAIRS == 2 ? 0xF : 0x3);
              if (kb == num_k - 1) mma_commit_cg2_mc(tfull_bar(acc), (uint16_t)(0x3u << my_leader));
            } else {
              mma_commit(empty_bar(stage));
              if (kb == num_k - 1) mma_commit(tfull_bar(acc));
            }
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane_id() == 0) TILE_TRACE(t, 1, gtimer());
        if (++acc == ACC_STAGES) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 2 + EPI_WARPS) {
    // ---------------- all-gather comm warps (distributed mode) ----------------
    // comm_clusters == 0: every GEMM CTA pulls 1/(2 x pairs) of the remote
    // boxes through its own 16 KiB buffer (warp 6), warp 7 signals the slabs.
    if constexpr (Prob::kGather) {
      if (sched.comm_clusters == 0 && lane_id() == 0) {
        const int agent = cluster * CG + (int)crank, nagents = nclusters * CG;
        const uint32_t mbox = bar_base + C::BAR_BYTES + 8 * COMM_MAX_BUFS;
        if (warp == 2 + EPI_WARPS) {
          gather_entry(sched, agent == 0);
          gather_agent_lag(sched, sbase + C::BAR_OFF - C::COMM_EXTRA, bar_base + C::BAR_BYTES,
                           C::COMM_EXTRA / (sched.box * COMM_W * 2), agent, nagents, mbox);
          gather_exit(sched, agent == 0, (uint32_t)nagents);
        } else {
          gather_signaler(sched, agent, 1, nagents, mbox);
        }
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int q = warp & 3;                         // TMEM lane quarter this warp may access
    const int ew = warp - 2;                        // epilogue warp index (staging buffers)
    const uint32_t lane = lane_id();
    const uint32_t stage_base = sbase + C::STAGES * C::STAGE_BYTES + ew * 2 * C::EPI_BUF;
    const uint32_t tempty_leader0 = (CG == 2) ? map_to_rank(tempty_bar(0), my_leader) : tempty_bar(0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int t = cluster, u = 0; t < num_tiles; t = next_tile(t, u++, lane == 0)) {
      const TileCoord tc = sched.decode(t);
      const int row0 = (tc.mt * PAIRS + pair) * BM_CTA * CG + (int)rank * BM_CTA + q * 32;  // C-map row
      const int col0 = tc.nt * BN;
      const CUtensorMap *cmap = sched.c_map(&tmC, tc.e);
      if (GROUPED && tc.swap_n) {
        // swapped tail: TMEM lane = output column, TMEM column = group row.
        // Transpose 32 x 32 chunks through the staging buffer (SWIZZLE_64B).
        mbar_wait(tfull_bar(acc), acc_phase, 4);
        tc_fence_after();
#ifdef MIMW_TILE_TRACE
        if (warp == 2 && leader && lane == 0) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
          TILE_TRACE(t, 2, gtimer());
          TILE_TRACE(t, 3, smid);
        }
#endif
        const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
        const int feat0 = tc.nt * BN + (int)rank * BM_CTA + q * 32;
        const int nch = tc.swap_n / EPI_COLS;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + ch * EPI_COLS, v);
          tmem_ld_wait();
          if (ch == nch - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader0 + 8 * acc);
          }
          const int tok0 = tc.mt * BM_CTA * CG + ch * EPI_COLS;
          if (tok0 < tc.rows && feat0 < N) {
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            const uint32_t sbuf = stage_base + buf * C::EPI_BUF;
            const uint32_t cbyte = (lane & 7) * 2;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const uint32_t pc = (lane >> 3) ^ ((r >> 1) & 3);
              const __nv_bfloat16 hv = __float2bfloat16_rn(__uint_as_float(v[r]));
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(sbuf + r * 64 + pc * 16 + cbyte),
                           "h"(*reinterpret_cast<const uint16_t *>(&hv))
                           : "memory");
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
        if (++acc == ACC_STAGES) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      mbar_wait(tfull_bar(acc), acc_phase, 4);
      tc_fence_after();
#ifdef MIMW_TILE_TRACE
      if (warp == 2 && leader && lane == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        TILE_TRACE(t, 2, gtimer());
        TILE_TRACE(t, 3, smid);
      }
#endif
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int ch = 0; ch < BN / EPI_COLS; ++ch) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + ch * EPI_COLS, v);
        tmem_ld_wait();
        if (ch == BN / EPI_COLS - 1) {
          // accumulator fully drained into registers: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + 8 * acc);
            else mbar_arrive(tempty_bar(acc));
          }
        }
        const bool live = (row0 < tc.rows) && (col0 + ch * EPI_COLS < N);
        if (live) {
          // staging buffer `buf` was used two chunks ago: its store must have read smem
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const uint32_t sbuf = stage_base + buf * C::EPI_BUF;
          if constexpr (sizeof(OutT) == 2) {
            // 32 rows x 64 B, SWIZZLE_64B: 16-B chunk c of row r at c ^ ((r >> 1) & 3)
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
          } else {
            // 32 rows x 128 B, SWIZZLE_128B: 16-B chunk c of row r at c ^ (r & 7)
            const uint32_t rbase = sbuf + lane * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t pc = (uint32_t)c ^ (lane & 7);
              st_shared_v4(rbase + pc * 16, v[4 * c + 0], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            }
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
      if (++acc == ACC_STAGES) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1 && !comm) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, 512);
  }
}

template <int CG, bool B_MN, typename OutT, typename Prob>
cudaError_t launch_kernel(const CUtensorMap &tA, const CUtensorMap &tB, const CUtensorMap &tC, int n,
                          int k, const Prob &prob_in, int tiles, int max_clusters, cudaStream_t stream,
                          int comm_clusters = 0) {
  using C = Cfg<CG, B_MN, OutT, Prob::kGather>;
  constexpr int CS = CG * Prob::kPairs;  // CTAs per cluster
  auto kern = gemm_bf16_kernel<CG, B_MN, OutT, Prob>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kernel_threads<Prob>(), 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be co-resident (GPC packing may
  // leave SMs idle for clusters > 2), never more than there are tiles
  int clusters = sm_count() / CS;
  {
    cfg.gridDim = dim3(clusters * CS, 1, 1);
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) == cudaSuccess && active > 0 &&
        active < clusters)
      clusters = active;
    cudaGetLastError();
  }
  // all-gather GEMM: comm pairs come out of the co-resident budget (they must
  // run alongside the GEMM pairs that wait on them)
  clusters -= comm_clusters;
  if (max_clusters > 0 && max_clusters < clusters) clusters = max_clusters;
  if (clusters > tiles) clusters = tiles;
  if constexpr (Prob::kClc)
    if (prob_in.clc) clusters = tiles;  // CLC: one cluster per tile, running clusters cancel the rest
  if (clusters <= 0 && tiles > 0) return cudaErrorInvalidConfiguration;
  if (clusters < 0) clusters = 0;
  if (clusters + comm_clusters == 0) return cudaSuccess;
  cfg.gridDim = dim3((clusters + comm_clusters) * CS, 1, 1);
  if constexpr (Prob::kGather) {
    Prob prob = prob_in;
    prob.comm_clusters = comm_clusters;
    return cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, n, k, prob);
  } else {
    return cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, n, k, prob_in);
  }
}

template <typename OutT>
CUtensorMap make_c_map(const void *c, int64_t rows, int64_t n, int64_t ldc) {
  const CUtensorMapDataType cdt =
      sizeof(OutT) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return make_tmap_2d(c, cdt, sizeof(OutT), rows, n, ldc, EPI_COLS, 32,
                      sizeof(OutT) == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
}

#include "gemm_wide.cuh"

template <int CG, bool B_MN, typename OutT>
cudaError_t launch_impl(const GemmArgs &g, cudaStream_t stream) {
  using C = Cfg<CG, B_MN, OutT>;
  CUtensorMap tA = make_tmap_2d(g.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.m, g.k, g.lda, BK,
                                BM_CTA, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = B_MN ? make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.k, g.n, g.ldb,
                                       64, BK, CU_TENSOR_MAP_SWIZZLE_128B)
                        : make_tmap_2d(g.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.n, g.k, g.ldb,
                                       BK, C::NB_CTA, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tC = make_c_map<OutT>(g.c, g.m, g.n, g.ldc);
  const int mt = (int)((g.m + BM_CTA * CG - 1) / (BM_CTA * CG));
  const int num_n = (int)((g.n + BN - 1) / BN);
  const int group = g.raster_group > 0 ? g.raster_group : 8;
  static const int clc_env = getenv("MIMW_GEMM_CLC_DENSE") ? atoi(getenv("MIMW_GEMM_CLC_DENSE")) : 1;  // A/B knob (CLC measured +0.4%)
  const int clc = (clc_env != 0 && g.max_clusters <= 0) ? 1 : 0;
  if constexpr (CG == 2 && sizeof(OutT) == 2) {
    // 256 x 512 pair tiles (gemm_wide.cuh) when asked for, or by default when
    // the problem still fills >= 3 waves of CTA pairs with them
    static const int wide_env = getenv("MIMW_GEMM_WIDE") ? atoi(getenv("MIMW_GEMM_WIDE")) : 1;  // A/B knob
    const int64_t wide_tiles = ((g.m + 255) / 256) * ((g.n + WIDE_BN - 1) / WIDE_BN);
    const bool wide = g.cluster_pairs != 2 &&
                      (g.tile_n == WIDE_BN || (g.tile_n == 0 && wide_env != 0 && wide_tiles >= 3 * (sm_count() / 2)));
    if (wide) return launch_wide<B_MN>(g, stream, clc);
  }
  if constexpr (CG == 2) {
    if (g.cluster_pairs == 2) {
      SchedT<2> s;
      s.num_m = (mt + 1) / 2;
      s.num_n = num_n;
      s.group = (group + 1) / 2;
      s.M = (int)g.m;
      s.clc = clc;
      return launch_kernel<CG, B_MN, OutT>(tA, tB, tC, (int)g.n, (int)g.k, s, s.num_m * s.num_n,
                                           g.max_clusters, stream);
    }
  }
  Sched s;
  s.num_m = mt;
  s.num_n = num_n;
  s.group = group;
  s.M = (int)g.m;
  s.clc = clc;
  return launch_kernel<CG, B_MN, OutT>(tA, tB, tC, (int)g.n, (int)g.k, s, s.num_m * s.num_n,
                                       g.max_clusters, stream);
}

// Slot order of the non-empty groups for chunks of `chunk` groups: groups
// sorted by rows, dealt to the chunks in a snake (chunk 0 gets the heaviest and
// the lightest, ...) so every chunk mixes compute-bound full tiles with
// weight-streaming light groups.  chunk <= 1 keeps the natural order.
std::vector<int> grouped_order(const std::vector<int> &live, const int *rows, int chunk) {
  static const int sort_env = getenv("MIMW_MOE_SORT") ? atoi(getenv("MIMW_MOE_SORT")) : 0;  // A/B knob
  if (chunk <= 1 && sort_env != 0) {
    std::vector<int> v = live;
    std::stable_sort(v.begin(), v.end(), [&](int x, int y) { return sort_env > 0 ? rows[x] > rows[y] : rows[x] < rows[y]; });
    return v;
  }
  if (chunk <= 1) return live;
  std::vector<int> by_rows = live;
  std::stable_sort(by_rows.begin(), by_rows.end(), [&](int a, int b) { return rows[a] > rows[b]; });
  const int nc = (int)((live.size() + chunk - 1) / chunk);
  std::vector<std::vector<int>> chunks((size_t)nc);
  for (size_t i = 0; i < by_rows.size(); ++i) {
    const int round = (int)(i / nc), pos = (int)(i % nc);
    chunks[(size_t)((round & 1) ? nc - 1 - pos : pos)].push_back(by_rows[i]);
  }
  std::vector<int> out;
  for (auto &c : chunks) out.insert(out.end(), c.begin(), c.end());
  return out;
}

// Grouped GEMM on the 256 x 512 wide tile (gemm_wide.cuh, padded tails):
// one launch per <= MAX_GROUPS groups.
template <bool B_MN>
cudaError_t grouped_wide_impl(const GroupedGemmArgs &g, cudaStream_t stream, int clc) {
  const int64_t total_rows = g.m_offsets[g.n_groups];
  CUtensorMap tA = make_tmap_2d(g.x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, total_rows, g.k, g.k, BK, BM_CTA,
                                CU_TENSOR_MAP_SWIZZLE_128B);
  auto *gs = new GroupedWideSched;
  cudaError_t err = cudaSuccess;
  for (int64_t g0 = 0; g0 < g.n_groups && err == cudaSuccess; g0 += MAX_GROUPS) {
    const int cnt = (int)std::min<int64_t>(MAX_GROUPS, g.n_groups - g0);
    const char *wbase = static_cast<const char *>(g.w) + (size_t)g0 * g.k * g.n * 2;
    CUtensorMap tB = B_MN ? make_tmap_3d(wbase, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.n, g.k, cnt, g.n,
                                         g.k * g.n, 64, BK, 1, CU_TENSOR_MAP_SWIZZLE_128B)
                          : make_tmap_3d(wbase, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.k, g.n, cnt, g.k,
                                         g.k * g.n, BK, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    std::memset(gs, 0, sizeof(GroupedWideSched));
    gs->x16 = make_tmap_2d(g.x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, total_rows, g.k, g.k, BK, 16,
                           CU_TENSOR_MAP_SWIZZLE_128B);
    gs->n_groups = cnt;
    gs->num_n = (int)((g.n + WIDE_BN - 1) / WIDE_BN);
    gs->clc = clc;
    // default swapped: configs[4] in 50-launch blocks 3.66 ms vs 3.96 padded vs 3.80 (256 x 256 tiles);
    // padded is faster only from a cold start (3.20 vs 3.33 ms), where it does 20% more MMA work
    gs->swap = g.swap_tails != 0 ? 1 : 0;
    int first_live = -1, tiles = 0;
    for (int i = 0; i < cnt; ++i) {
      const int64_t r0 = g.m_offsets[g0 + i], r1 = g.m_offsets[g0 + i + 1];
      gs->row_off[i] = (int)r0;
      gs->rows[i] = (int)(r1 - r0);
      gs->mt[i] = (int)((r1 - r0 + 255) / 256);
      gs->tile_pref[i] = tiles;
      tiles += gs->mt[i] * gs->num_n;
      if (r1 > r0) {
        gs->y[i] = make_c_map<__nv_bfloat16>(static_cast<char *>(g.y) + (size_t)r0 * g.n * 2, r1 - r0, g.n, g.n);
        if (first_live < 0) first_live = i;
      }
    }
    gs->tile_pref[cnt] = tiles;
    if (first_live < 0) continue;
    for (int i = 0; i < cnt; ++i)
      if (gs->rows[i] == 0) gs->y[i] = gs->y[first_live];  // never stored through
    err = launch_wide_kernel<B_MN>(tA, tB, gs->y[first_live], (int)g.n, (int)g.k, *gs, tiles, g.max_clusters, clc,
                                   stream);
  }
  delete gs;
  return err;
}

// One launch per chunk of <= MAX_GROUPS groups (the Y maps travel in the
// kernel's parameter block).
template <int CG, bool B_MN>
cudaError_t grouped_impl(const GroupedGemmArgs &g, cudaStream_t stream) {
  using C = Cfg<CG, B_MN, __nv_bfloat16>;
  const int64_t total_rows = g.m_offsets[g.n_groups];
  CUtensorMap tA = make_tmap_2d(g.x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, total_rows, g.k, g.k, BK,
                                BM_CTA, CU_TENSOR_MAP_SWIZZLE_128B);
  auto *gs = new GroupedSched;  // ~20 KB: keep it off the host stack
  static const int chunk_env = getenv("MIMW_MOE_CHUNK") ? atoi(getenv("MIMW_MOE_CHUNK")) : -1;  // A/B knob
  const int chunk = chunk_env >= 0 ? chunk_env : 1;
  static const int clc_env = getenv("MIMW_GEMM_CLC") ? atoi(getenv("MIMW_GEMM_CLC")) : 1;  // A/B knob
  cudaError_t err = cudaSuccess;
  for (int64_t g0 = 0; g0 < g.n_groups && err == cudaSuccess; g0 += MAX_GROUPS) {
    const int cnt = (int)std::min<int64_t>(MAX_GROUPS, g.n_groups - g0);
    const char *wbase = static_cast<const char *>(g.w) + (size_t)g0 * g.k * g.n * 2;
    CUtensorMap tB = B_MN ? make_tmap_3d(wbase, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.n, g.k, cnt,
                                         g.n, g.k * g.n, 64, BK, 1, CU_TENSOR_MAP_SWIZZLE_128B)
                          : make_tmap_3d(wbase, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.k, g.n, cnt,
                                         g.k, g.k * g.n, BK, C::NB_CTA, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    std::memset(gs, 0, sizeof(GroupedSched));
    gs->num_n = (int)((g.n + BN - 1) / BN);
    gs->bm = BM_CTA * CG;
    gs->swap = (CG == 2 && g.swap_tails != 0) ? 1 : 0;
    gs->clc = (clc_env != 0 && g.max_clusters <= 0) ? 1 : 0;  // max_clusters bounds a persistent grid
    static const int pf_env = getenv("MIMW_MOE_PREFETCH") ? atoi(getenv("MIMW_MOE_PREFETCH")) : 0;  // A/B knob (16: 3.58 vs 3.47 ms, not kept)
    gs->prefetch = pf_env;
    int first_live = -1;
    std::vector<int> live;
    for (int i = 0; i < cnt; ++i) {
      const int64_t r0 = g.m_offsets[g0 + i], r1 = g.m_offsets[g0 + i + 1];
      gs->row_off[i] = (int)r0;
      gs->rows[i] = (int)(r1 - r0);
      if (r1 > r0) {
        gs->y[i] = make_c_map<__nv_bfloat16>(static_cast<char *>(g.y) + (size_t)r0 * g.n * 2,
                                             r1 - r0, g.n, g.n);
        if (first_live < 0) first_live = i;
        live.push_back(i);
      }
    }
    if (live.empty()) continue;
    for (int i = 0; i < cnt; ++i)
      if (gs->rows[i] == 0) gs->y[i] = gs->y[first_live];  // never stored through
    const std::vector<int> order = grouped_order(live, gs->rows, chunk);
    const int per_chunk = std::max(1, chunk);
    int tiles = 0, ns = 0;
    gs->n_chunks = 0;
    gs->mt_pref[0] = 0;
    for (size_t s0 = 0; s0 < order.size(); s0 += per_chunk) {
      gs->chunk_off[gs->n_chunks] = tiles;
      gs->chunk_slot[gs->n_chunks] = ns;
      int mts = 0;
      for (size_t j = s0; j < std::min(order.size(), s0 + per_chunk); ++j, ++ns) {
        const int e = order[j];
        gs->order[ns] = e;
        mts += (gs->rows[e] + gs->bm - 1) / gs->bm;
        gs->mt_pref[ns + 1] = gs->mt_pref[ns] + (gs->rows[e] + gs->bm - 1) / gs->bm;
      }
      tiles += mts * gs->num_n;
      ++gs->n_chunks;
    }
    gs->chunk_off[gs->n_chunks] = tiles;
    gs->chunk_slot[gs->n_chunks] = ns;
    err = launch_kernel<CG, B_MN, __nv_bfloat16>(tA, tB, gs->y[first_live], (int)g.n, (int)g.k, *gs,
                                                 tiles, g.max_clusters, stream);
  }
  delete gs;
  return err;
}


// ---- all-gather (K-gathered) multi-device GEMM -------------------------------
struct GatherLayout {
  int max_slabs = 0;
  size_t ctr_off = 0, ctr_bytes = 0;
  size_t land_a[MAX_SPLITS] = {}, land_b[MAX_SPLITS] = {};  // by rotation index q
  size_t total = 0;
};

GatherLayout gather_layout(int rank, int world, const int64_t *k, int64_t rows, int64_t n) {
  GatherLayout L;
  auto align = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  int64_t kmax = 0;
  for (int s = 0; s < world; ++s) kmax = std::max(kmax, k[s]);
  L.max_slabs = (int)((kmax + COMM_SLAB - 1) / COMM_SLAB);
  L.ctr_bytes = align(sizeof(uint32_t) * (MAX_SPLITS * (size_t)std::max(L.max_slabs, 1) + 4));
  size_t off = L.ctr_bytes;
  for (int q = 1; q < world; ++q) {
    const int64_t kq = k[(rank + q) % world];
    L.land_a[q] = off;
    off = align(off + (size_t)rows * kq * 2);
    L.land_b[q] = off;
    off = align(off + (size_t)kq * n * 2);
  }
  L.total = off;
  return L;
}
}  // namespace

#ifdef MIMW_TILE_TRACE
cudaError_t set_tile_trace(void *buf) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  return cudaMemcpyToSymbol(g_mimw_tile_trace, &p, sizeof(p));
}
#endif

cudaError_t gemm_bf16_launch(const GemmArgs &g, cudaStream_t stream) {
  if (g.k == 0) {
    // no K: C = 0 (the oracle's float accumulator starts at 0.0f, oracles.cpp:19)
    size_t es = g.c_f32 ? 4 : 2;
    return cudaMemset2DAsync(g.c, g.ldc * es, 0, g.n * es, g.m, stream);
  }
  const bool cg2 = g.cta_group != 1;
  if (g.b_kn) {
    if (g.c_f32) return cg2 ? launch_impl<2, true, float>(g, stream) : launch_impl<1, true, float>(g, stream);
    return cg2 ? launch_impl<2, true, __nv_bfloat16>(g, stream)
               : launch_impl<1, true, __nv_bfloat16>(g, stream);
  }
  if (g.c_f32) return cg2 ? launch_impl<2, false, float>(g, stream) : launch_impl<1, false, float>(g, stream);
  return cg2 ? launch_impl<2, false, __nv_bfloat16>(g, stream)
             : launch_impl<1, false, __nv_bfloat16>(g, stream);
}

cudaError_t grouped_gemm_bf16_launch(const GroupedGemmArgs &g, cudaStream_t stream) {
  if (g.n_groups <= 0 || g.n == 0 || g.m_offsets[g.n_groups] == g.m_offsets[0]) return cudaSuccess;
  if (g.k == 0) {
    const int64_t r0 = g.m_offsets[0], r1 = g.m_offsets[g.n_groups];
    return cudaMemsetAsync(static_cast<char *>(g.y) + (size_t)r0 * g.n * 2, 0,
                           (size_t)(r1 - r0) * g.n * 2, stream);
  }
  if (g.cta_group == 1)
    return g.w_kn ? grouped_impl<1, true>(g, stream) : grouped_impl<1, false>(g, stream);
  // 256 x 512 pair tiles (gemm_wide.cuh): configs[4] 3.20 vs 3.45 ms with 256 x 256
  static const int wide_env = getenv("MIMW_MOE_WIDE") ? atoi(getenv("MIMW_MOE_WIDE")) : 1;  // A/B knob
  static const int clc_env = getenv("MIMW_GEMM_CLC") ? atoi(getenv("MIMW_GEMM_CLC")) : 1;
  if (g.tile_n == WIDE_BN || (g.tile_n == 0 && wide_env != 0 && g.n >= WIDE_BN)) {
    const int clc = (clc_env != 0 && g.max_clusters <= 0) ? 1 : 0;
    return g.w_kn ? grouped_wide_impl<true>(g, stream, clc) : grouped_wide_impl<false>(g, stream, clc);
  }
  return g.w_kn ? grouped_impl<2, true>(g, stream) : grouped_impl<2, false>(g, stream);
}

size_t multi_device_gemm_workspace_bytes(int rank, int world, const int64_t *k, int64_t rows, int64_t n) {
  return gather_layout(rank, world, k, rows, n).total;
}

cudaError_t multi_device_gemm_launch(const MultiDeviceGemmArgs &g, cudaStream_t stream) {
  const GatherLayout L = gather_layout(g.rank, g.world, g.k, g.rows, g.n);
  if (g.ws_bytes < L.total) return cudaErrorInvalidValue;
  const bool barrier = g.pads[g.rank] != nullptr;
  const bool work = g.rows > 0 && g.n > 0;
  if (!work && !barrier) return cudaSuccess;
  char *ws = static_cast<char *>(g.ws);
  uint32_t *ctr = reinterpret_cast<uint32_t *>(ws + L.ctr_off);
  cudaError_t e = cudaMemsetAsync(ctr, 0, L.ctr_bytes, stream);
  if (e != cudaSuccess) return e;
  auto *gs = new GatherSched;  // ~6 KB of tensor maps: keep it off the host stack
  std::memset(gs, 0, sizeof(GatherSched));
  // comm_clusters > 0: dedicated comm CTA pairs; < 0: distributed (a comm warp
  // in every GEMM CTA, 16 KiB boxes).  A rank with no rows still meets its
  // peers in the barrier, through one dedicated pair.
  int comm = g.world > 1 ? (g.comm_clusters == 0 ? kDefaultCommPairs : g.comm_clusters) : 0;
  if (comm < 0 && !work) comm = 1;
  const bool distributed = comm < 0;
  if (distributed) comm = 0;
  const int box = distributed ? 32
                  : (g.comm_box == 32 || g.comm_box == 64 || g.comm_box == 128) ? g.comm_box : 64;
  gs->num_m = work ? (int)((g.rows + BM_CTA * 2 - 1) / (BM_CTA * 2)) : 0;
  gs->num_n = work ? (int)((g.n + BN - 1) / BN) : 0;
  gs->group = 8;
  gs->M = (int)g.rows;
  gs->rank = g.rank;
  gs->world = g.world;
  gs->epoch = g.epoch;
  {
    // MIMW_PEER_WAIT_S: seconds a rank waits for its peers at the device-side
    // entry / exit barriers before trapping (default 600; 0 = wait forever)
    static const double peer_s = getenv("MIMW_PEER_WAIT_S") ? atof(getenv("MIMW_PEER_WAIT_S")) : 600.0;
    gs->peer_budget = peer_s > 0 ? (uint64_t)(peer_s * 2.1e9) : 0;
  }
  gs->ctr = ctr;
  gs->max_slabs = L.max_slabs;
  gs->box = box;
  gs->agents = std::min(6, std::max(1, g.comm_agents > 0 ? g.comm_agents : 2));  // warps 0..5
  gs->lag = g.comm_lag > 0 ? g.comm_lag : (distributed ? 4 : 8);
  gs->rbox = (int)((g.rows + box - 1) / box);
  gs->nbox = (int)((g.n + COMM_W - 1) / COMM_W);
  gs->pad_local = g.pads[g.rank];
  for (int p = 0; p < g.world; ++p) gs->pad_peer[p] = g.pads[p];
  // never-dereferenced stand-in for maps of empty operands
  const CUtensorMap dummy = make_tmap_2d(ws, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 32, EPI_COLS, EPI_COLS,
                                         EPI_COLS, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  int kblocks = 0;
  int64_t ktot = 0;
  for (int q = 0; q < g.world; ++q) {
    const int s = (g.rank + q) % g.world;
    const int64_t kq = g.k[s];
    ktot += kq;
    gs->ks[q] = (int)kq;
    kblocks += (int)((kq + BK - 1) / BK);
    gs->ga[q] = gs->gb[q] = gs->src_a[q] = gs->dst_a[q] = gs->src_b[q] = gs->dst_b[q] = dummy;
    if (kq == 0 || !work) continue;
    const void *abase = static_cast<const char *>(g.a[s]) + (size_t)g.row0 * kq * 2;
    const void *la = q == 0 ? abase : ws + L.land_a[q];
    const void *lb = q == 0 ? g.b[s] : ws + L.land_b[q];
    gs->ga[q] = make_tmap_2d(la, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.rows, kq, kq, BK, BM_CTA,
                             CU_TENSOR_MAP_SWIZZLE_128B);
    gs->gb[q] = make_tmap_2d(lb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kq, g.n, g.n, 64, BK,
                             CU_TENSOR_MAP_SWIZZLE_128B);
    if (q == 0) continue;
    // comm boxes {256, box rows}, unswizzled (pure copies)
    gs->src_a[q] = make_tmap_2d(abase, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.rows, kq, kq, COMM_W,
                                box, CU_TENSOR_MAP_SWIZZLE_NONE);
    gs->dst_a[q] = make_tmap_2d(la, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.rows, kq, kq, COMM_W, box,
                                CU_TENSOR_MAP_SWIZZLE_NONE);
    gs->src_b[q] = make_tmap_2d(g.b[s], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kq, g.n, g.n, COMM_W,
                                box, CU_TENSOR_MAP_SWIZZLE_NONE);
    gs->dst_b[q] = make_tmap_2d(lb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kq, g.n, g.n, COMM_W, box,
                                CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  gs->nsplit = g.world;
  gs->kblocks = kblocks;
  gs->pull = work && ktot > 0;
  if (work && ktot == 0) {  // C = 0 (oracles.cpp:19); the barrier below still runs
    e = cudaMemset2DAsync(g.c, g.ldc * 2, 0, g.n * 2, g.rows, stream);
    gs->num_m = 0;
  }
  const CUtensorMap tC = (work && ktot > 0) ? make_c_map<__nv_bfloat16>(g.c, g.rows, g.n, g.ldc) : dummy;
  if (e == cudaSuccess && (gs->num_m > 0 || comm > 0))
    e = launch_kernel<2, true, __nv_bfloat16>(tC, tC, tC, (int)g.n, (int)ktot, *gs,
                                              gs->num_m * gs->num_n, g.max_clusters, stream, comm);
  delete gs;
  return e;
}

}  // namespace mimw
