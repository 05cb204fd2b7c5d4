// Warp-specialized flash-attention forward for sm_100a (bf16 in, fp32 accum).
//
// Computes, per (batch, head), the reference's windowed causal softmax
// attention  oracle_attention(q, k, v, w, scale)  (proj/core/src/
// oracles.cpp:119-145): keys j in [max(0, i-w+1), i], softmax in the exp
// domain, o = P.V.  Also returns lse = m + log(l) as the simplicial program
// does (oracles.cpp:116, simplicial_attention.mimw:88-93).
//
// MIMW structure (the B200 form of proj/kernels/simplicial_attention.mimw:
// a producer task staging K/V blocks through barriers, consumers running an
// online softmax), one persistent CTA per SM, 12 warps in 3 warpgroups:
//   WG0 (warps 0-3)  softmax/correction for Q tile 0 (rows q0 .. q0+127)
//   WG1 (warps 4-7)  softmax/correction for Q tile 1 (rows q0+128 .. q0+255)
//   WG2 warp 8       TMA producer + tile scheduler (atomic work counter,
//                    published through a 2-slot mbarrier ring: the CLC
//                    clc_producer/clc_consumer protocol of sim.cpp:1213-1286)
//   WG2 warp 9       MMA issuer for S = Q_h K_j^T (SS), releases K slots
//   WG2 warp 10      MMA issuer for O_h += P_h V_j (TS), releases V slots.
//                    tcgen05.mma issue blocks at the tensor-pipe rate, so a
//                    single issuer drains the pipe at every dependency wait
//                    (measured: tools/fa_events.py); two keep it fed.
//   WG2 warp 11      idle (donates registers via setmaxnreg)
//
// TMEM (512 columns x 128 lanes): S [0,128) fp32 (ONE buffer shared by both
// Q tiles), P_0 [128,192) P_1 [192,256) bf16, O_0 [256,384) O_1 [384,512).
// A softmax warp releases S right after tcgen05.ld has it in registers, so the
// next S MMA overlaps the exponentials; P lives in its own columns, and the
// P.V product lags one KV step.  MMA issue order per step j:
//     S_0(j)  PV_0(j-1)  S_1(j)  PV_1(j-1)
// keeping the tensor pipe busy while both softmax warpgroups compute.
// Correction (O *= 2^(m_old - m_new), only when the running max grows by
// > 8 in log2 units) runs in the softmax warpgroup after PV_h(j-1) completes
// and before P_h(j) is published.  The epilogue (O / l, lse) goes through a
// per-warp 4 KiB swizzled smem box and TMA stores.  Q_h is released by a
// tcgen05.commit after its last S MMA, so the next item's Q load overlaps the
// current item's tail.
#include "attention_fwd.h"
#include "ptx.cuh"
#include "softmax.cuh"
#include "pool.h"
#include "tma_host.h"

#include <atomic>
#include <cstdlib>
#include <mutex>

namespace mimw {

namespace {

constexpr int D = 128;           // head dim (QK^T K-extent, PV N-extent)
constexpr int BQ = 128;          // rows per Q tile (MMA M)
constexpr int BKV = 128;         // keys per KV tile (S N-extent, PV K-extent)
constexpr int NSLOT = 4;         // K/V ring slots (32 KiB each; 5 measured the same)
constexpr int TILE_BYTES = BKV * D * 2;  // 32 KiB: one Q, K or V tile
constexpr int HALF_BYTES = TILE_BYTES / 2;  // one 64-column (128-B) swizzle panel
constexpr int NUM_THREADS = 384;  // 3 warpgroups
constexpr int SMEM_Q = 0;
constexpr int SMEM_KV = 2 * TILE_BYTES;
constexpr int SMEM_O = SMEM_KV + NSLOT * TILE_BYTES;  // O staging: 8 softmax warps x 4 KiB (32 rows x 64 cols bf16)
constexpr int SMEM_BAR = SMEM_O + 8 * 4096;
constexpr int SMEM_TOTAL = SMEM_BAR + 512 + 1024;
constexpr uint32_t IDESC_S = idesc_bf16(BQ, BKV, 0, 0);   // Q (K-major) x K (K-major)
constexpr uint32_t IDESC_PV = idesc_bf16(BQ, D, 0, 1);    // P (TMEM) x V (MN-major)
constexpr uint32_t TM_S = 0, TM_P = 128, TM_O = 256;       // TMEM column bases
constexpr float LOG2E = 1.4426950408889634f;
#ifdef MIMW_FA_SPIN
#define MMA_WAIT mbar_wait_spin
#else
#define MMA_WAIT mbar_wait
#endif
constexpr int kDefaultEmu = 0;  // exp2 pairs (of 8) evaluated on the FMA pipe (0: measured fastest, tools/fa_sweep.py)
constexpr int kDefaultEmuCg2 = 2;  // same, 2-CTA kernel
#ifndef MIMW_FA_HEAD_BAND
#define MIMW_FA_HEAD_BAND 8  // 1346-1349 vs 1333-1336 TFLOPS with 4 (tools/fa_ab.py; 1: 1325, 2: 1323, 16: 1343-1348)
#endif
constexpr int HEAD_BAND = MIMW_FA_HEAD_BAND;  // heads per scheduling band (K/V of a band stays in L2)

struct Params {
  int bh;            // batch * heads
  int seq;
  int window;        // keys j in [i - window + 1, i]
  int causal;        // 0: every key of the sequence (non-causal, PAPER.md:702-716 AFN rows)
  int nqb;           // 256-row blocks per head
  float scale_log2;  // scale * log2(e)
  float *lse;        // [bh, seq] or null
  __nv_bfloat16 *o;  // [bh, seq, 128]
  int scale_pos;     // scale > 0: max on raw scores, scale folded into FFMA2
  int *work_counter; // {claims, retired}: dynamic scheduler counter, zeroed by the last CTA
  unsigned long long *trace;  // optional per-warp cycle accounting [grid][12][8]
  int dbg;           // timing-only probes (MIMW_FA_DEBUG): 1 = skip the O stores
};

// KV tile range [lo, hi] needed by Q rows [r0, r0 + 127]
__device__ __forceinline__ void kv_range(int r0, const Params &p, int &lo, int &hi) {
  int last = p.causal ? min(r0 + BQ - 1, p.seq - 1) : p.seq - 1;
  int first_key = p.causal ? max(0, r0 - p.window + 1) : 0;
  lo = first_key / BKV;
  hi = last / BKV;
}

// Work order: bands of HEAD_BAND heads (their K/V stay L2-resident while the
// band is in flight); inside a band, longest (largest causal q-block) first.
__device__ __forceinline__ void work_item(int idx, const Params &p, int &bh, int &qb) {
  const int per_band = HEAD_BAND * p.nqb;
  const int band = idx / per_band;
  const int r = idx - band * per_band;
  const int heads_in_band = min(HEAD_BAND, p.bh - band * HEAD_BAND);
  qb = p.nqb - 1 - r / heads_in_band;
  bh = band * HEAD_BAND + r % heads_in_band;
}

template <int EMU>
__global__ void __launch_bounds__(NUM_THREADS, 1)
attention_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + SMEM_BAR;
  auto q_full = [&](int h) { return bars + 8 * h; };
  auto q_empty = [&](int h) { return bars + 16 + 8 * h; };
  auto s_full = [&](int h) { return bars + 32 + 8 * h; };
  auto p_full = [&](int h) { return bars + 48 + 8 * h; };
  auto o_done = [&](int h) { return bars + 64 + 8 * h; };
  const uint32_t s_free = bars + 80;
  auto sched_full = [&](int s) { return bars + 88 + 8 * s; };
  auto sched_empty = [&](int s) { return bars + 104 + 8 * s; };
  auto kv_full = [&](int s) { return bars + 120 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 120 + 8 * NSLOT + 8 * s; };
  const uint32_t tmem_slot = bars + 120 + 16 * NSLOT;
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + SMEM_BAR + 120 + 16 * NSLOT);
  volatile int *sched_slot = reinterpret_cast<int *>(smem + SMEM_BAR + 128 + 16 * NSLOT);  // [2]

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const int num_items = p.bh * p.nqb;
#ifdef MIMW_FA_EVENTS
  // event log of CTA 0 (tools/fa_events.py): warps 0, 4 (softmax lane quarter 0) and 9 (MMA)
  int ev_n = 0;
#define EV(code)                                                                          \
  do {                                                                                    \
    if (blockIdx.x == 0 && lane == 0 && ev_n < 1024 && p.trace)                           \
      p.trace[warp * 1024 + ev_n++] = ((unsigned long long)clock64() << 8) | (code);     \
  } while (0)
#else
#define EV(code) do {} while (0)
#endif

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int h = 0; h < 2; ++h) {
      mbar_init(q_full(h), 1);
      mbar_init(q_empty(h), 1);
      mbar_init(s_full(h), 1);
      mbar_init(p_full(h), 4);
      mbar_init(o_done(h), 1);
      mbar_init(sched_full(h), 1);
      mbar_init(sched_empty(h), 10);  // 2 MMA warps + 8 softmax warps
    }
    mbar_init(s_free, 4);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp >= 8) {
  // control warpgroup gives registers to the two softmax warpgroups.  Budget:
  // the pool only holds what dec releases: 8 warps x (208-168) <= 4 x (168-88).
  asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
  if (warp == 8) {
    // ================= scheduler + TMA producer =================
    if (lane == 0) {
      int slot = 0;
      uint32_t slot_phase = 0;
      uint32_t qe_phase[2] = {0, 0};  // per Q tile: a tile beyond seq is neither loaded nor released
      int it = blockIdx.x;
      for (int n = 0;; ++n) {
        // publish the work item (or -1) to the consumers
        const int ss = n & 1;
        mbar_wait(sched_empty(ss), ((n >> 1) & 1) ^ 1, 12);
        sched_slot[ss] = it < num_items ? it : -1;
        mbar_arrive(sched_full(ss));
        EV(33);
        if (it >= num_items) {
          // self-reset of this launch's counter slot: the last CTA to retire
          // (after every CTA's final claim, fenced) zeroes it for the next
          // launch that draws the slot
          __threadfence();
          if (atomicAdd(p.work_counter + 1, 1) == (int)gridDim.x - 1) {
            p.work_counter[0] = 0;
            p.work_counter[1] = 0;
            __threadfence();
          }
          break;
        }
        int bh, qb;
        work_item(it, p, bh, qb);
        const int r0 = qb * 2 * BQ;
        int lo0, hi0, lo1, hi1;
        kv_range(r0, p, lo0, hi0);
        kv_range(r0 + BQ, p, lo1, hi1);
        if (r0 + BQ >= p.seq) hi1 = hi0;  // Q tile 1 entirely beyond seq: no extra tile
        const int lo = min(lo0, lo1), hi = max(hi0, hi1);
        for (int h = 0; h < 2; ++h) {
          // Q tile 1 beyond seq: skipped on every side (no load, no q_full
          // wait, no release), so q_empty(h) completes exactly once per load
          // and can never run two phases ahead of this wait
          if (h == 1 && r0 + BQ >= p.seq) continue;
          mbar_wait(q_empty(h), qe_phase[h] ^ 1, 10);
          EV(40 + h);
          mbar_arrive_expect_tx(q_full(h), TILE_BYTES);
          const uint32_t dq = sbase + SMEM_Q + h * TILE_BYTES;
          tma_load_3d(dq, &tmQ, q_full(h), 0, r0 + h * BQ, bh);
          tma_load_3d(dq + HALF_BYTES, &tmQ, q_full(h), 64, r0 + h * BQ, bh);
          qe_phase[h] ^= 1;
        }
        // next item: claimed now so the consumers never wait on the atomic
        it = atomicAdd(p.work_counter, 1) + (int)gridDim.x;
        for (int j = lo; j <= hi; ++j) {
#pragma unroll 1
          for (int kv = 0; kv < 2; ++kv) {
            mbar_wait(kv_empty(slot), slot_phase ^ 1, 11);
            mbar_arrive_expect_tx(kv_full(slot), TILE_BYTES);
            const uint32_t dst = sbase + SMEM_KV + slot * TILE_BYTES;
            const CUtensorMap *tm = kv == 0 ? &tmK : &tmV;
            tma_load_3d(dst, tm, kv_full(slot), 0, j * BKV, bh);
            tma_load_3d(dst + HALF_BYTES, tm, kv_full(slot), 64, j * BKV, bh);
            if (++slot == NSLOT) { slot = 0; slot_phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 9 || warp == 10) {
    // ================= MMA issuers (S: warp 9, PV: warp 10) =================
    // The whole warp runs the schedule (so descriptor math stays on the
    // uniform datapath); one elected lane issues tcgen05.mma / commit.
    const bool s_role = warp == 9;
    uint32_t ring = 0;  // K/V ring positions consumed so far (K_j at 2(j-lo), V_j at 2(j-lo)+1)
    uint32_t q_phase[2] = {0, 0}, sf_phase = 0;
    uint32_t p_phase0 = 0, p_phase1 = 0;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t sb = __shfl_sync(0xffffffffu, sbase, 0);
    constexpr uint32_t HI_KMAJ = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO, version, SW128
    constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;                         // LBO (unused)
    constexpr uint32_t LO_VMN = ((uint32_t)HALF_BYTES >> 4) << 16;         // LBO = D-panel stride
#ifdef MIMW_FA_TRACE
    long long mt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define MIMW_TR_BEGIN const long long _t0 = clock64();
#define MIMW_TR_END(i) mt_acc[i] += clock64() - _t0;
#else
#define MIMW_TR_BEGIN
#define MIMW_TR_END(i)
#endif
    auto ring_wait = [&](uint32_t pos) {
      MIMW_TR_BEGIN
      MMA_WAIT(kv_full(pos % NSLOT), (pos / NSLOT) & 1, 23);
      MIMW_TR_END(2)
    };
    auto issue_S = [&](int h, uint32_t kslot, bool last) {
      {
        MIMW_TR_BEGIN
        MMA_WAIT(s_free, sf_phase ^ 1, 24);  // S buffer released by its last reader
        MIMW_TR_END(3)
      }
      EV(1 + 2 * h);
      sf_phase ^= 1;
      tc_fence_after();
      const uint32_t qa = (sb + SMEM_Q + h * TILE_BYTES) >> 4;
      const uint32_t kb = (sb + SMEM_KV + kslot * TILE_BYTES) >> 4;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k >> 2) * HALF_BYTES + (k & 3) * 32) >> 4;
          mma_f16_ss<1>(tm + TM_S, make_desc(LO_KMAJ | (qa + off), HI_KMAJ),
                        make_desc(LO_KMAJ | (kb + off), HI_KMAJ), IDESC_S, k != 0);
        }
        mma_commit(s_full(h));
        // Q_h's last reader: release it when this MMA completes (not when the
        // softmax has loaded S), so the next item's Q load starts earlier
        if (last) mma_commit(q_empty(h));
      }
      __syncwarp();
      EV(21 + 2 * h);
    };
    auto issue_PV = [&](int h, uint32_t vslot, bool acc) {
      {
        MIMW_TR_BEGIN
        MMA_WAIT(p_full(h), h ? p_phase1 : p_phase0, 25 + h);
        MIMW_TR_END(h)
      }
      EV(2 + 2 * h);
      if (h) p_phase1 ^= 1; else p_phase0 ^= 1;
      tc_fence_after();
      const uint32_t vb = (sb + SMEM_KV + vslot * TILE_BYTES) >> 4;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          mma_f16_ts<1>(tm + TM_O + h * 128, tm + TM_P + h * 64 + k * 8,
                        make_desc(LO_VMN | (vb + k * (2048 >> 4)), HI_KMAJ), IDESC_PV,
                        (acc || k != 0) ? 1u : 0u);
        mma_commit(o_done(h));
      }
      __syncwarp();
      EV(22 + 2 * h);
    };
    auto release = [&](uint32_t slot) {
      if (elect_one()) mma_commit(kv_empty(slot));
      __syncwarp();
    };
    for (int n = 0;; ++n) {
      const int ss = n & 1;
      mbar_wait(sched_full(ss), (n >> 1) & 1, 20);
      const int it = sched_slot[ss];
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty(ss));
      if (it < 0) break;
      int bh, qb;
      work_item(it, p, bh, qb);
      const int r0 = qb * 2 * BQ;
      int lo0, hi0, lo1, hi1;
      kv_range(r0, p, lo0, hi0);
      kv_range(r0 + BQ, p, lo1, hi1);
      const bool has1 = r0 + BQ < p.seq;
      if (!has1) hi1 = hi0;
      const int lo = min(lo0, lo1), hi = max(hi0, hi1);
      if (s_role) {
        MIMW_TR_BEGIN
        mbar_wait(q_full(0), q_phase[0], 21);
        if (has1) mbar_wait(q_full(1), q_phase[1], 22);
        MIMW_TR_END(6)
      }
      q_phase[0] ^= 1;
      if (has1) q_phase[1] ^= 1;
      // Two issuers keep the tensor pipe fed: tcgen05.mma issue blocks at the
      // pipe rate, so while one warp waits on a dependency the other's group
      // is already queued.  Warp 9 issues every S = Q K^T (and releases K
      // slots), warp 10 every O += P V (and releases V slots).
      for (int j = lo; j <= hi; ++j) {
        const uint32_t kpos = ring + 2 * (j - lo);
        if (s_role) {
          ring_wait(kpos);
          if (j >= lo0 && j <= hi0) issue_S(0, kpos % NSLOT, j == hi0);
          if (has1 && j >= lo1 && j <= hi1) issue_S(1, kpos % NSLOT, j == hi1);
          release(kpos % NSLOT);  // K_j: both S products issued
        } else {
          const uint32_t vpos = kpos + 1;  // V_j
          ring_wait(vpos);
          EV(20);
          if (j >= lo0 && j <= hi0) issue_PV(0, vpos % NSLOT, j != lo0);
          if (has1 && j >= lo1 && j <= hi1) issue_PV(1, vpos % NSLOT, j != lo1);
          release(vpos % NSLOT);  // V_j
        }
      }
      ring += 2 * (hi - lo + 1);
#ifdef MIMW_FA_TRACE
      mt_acc[4] += hi - lo + 1;
#endif
    }
#ifdef MIMW_FA_TRACE
    if (p.trace && lane == 0)
      for (int e = 0; e < 8; ++e) p.trace[((size_t)blockIdx.x * 12 + warp) * 8 + e] = mt_acc[e];
#endif
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    // ================= softmax / correction / epilogue (WG h) =================
    const int h = warp >> 2;             // Q tile owned by this warpgroup
    const int q = warp & 3;              // TMEM lane quarter
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const uint32_t t_s = tmem + t_lane + TM_S;
    const uint32_t t_p = tmem + t_lane + TM_P + h * 64;
    const uint32_t t_o = tmem + t_lane + TM_O + h * 128;
    uint32_t s_phase = 0;
    uint32_t od_count = 0;  // o_done[h] phases consumed (one per PV_h)
#ifdef MIMW_FA_TRACE
    long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    for (int n = 0;; ++n) {
      const int ss = n & 1;
      mbar_wait(sched_full(ss), (n >> 1) & 1, 28);
      EV(32);
      const int it = sched_slot[ss];
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty(ss));
      if (it < 0) break;
      int bh, qb;
      work_item(it, p, bh, qb);
      const int rt = qb * 2 * BQ + h * BQ;  // first row of this Q tile
      const int row = rt + q * 32 + (int)lane;
      const bool tile_live = rt < p.seq;
      int lo, hi;
      kv_range(rt, p, lo, hi);
      float m_used = -INFINITY;  // log2-domain max the exponentials are taken against
      float l = 0.f;
      if (!tile_live) continue;  // tile beyond seq: never loaded, nothing to release
      for (int j = lo; j <= hi; ++j) {
#ifdef MIMW_FA_TRACE
        const long long tr0 = clock64();
#endif
        mbar_wait(s_full(h), s_phase, 30 + h);
        s_phase ^= 1;
        tc_fence_after();
        EV(10);
#ifdef MIMW_FA_TRACE
        const long long tr1 = clock64();
#endif
        uint32_t s[128];
        // two halves: the second pair of loads overlaps the first half's max
        tmem_ld_32x32b_x32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld_32x32b_x32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld_wait();
        EV(15);
        tmem_ld_32x32b_x32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
        tmem_ld_32x32b_x32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        const int k0 = j * BKV;
        // tile needs masking if any (row, key) pair of the whole Q tile is invalid
        const bool need_mask = (p.causal && ((k0 + BKV - 1 > rt) || (k0 < rt + BQ - p.window))) ||
                               (k0 + BKV > p.seq) || !p.scale_pos;
        if (!need_mask) {
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              m4[e] = fmax3(m4[e], __uint_as_float(s[c + 2 * e]), __uint_as_float(s[c + 2 * e + 1]));
          }
        }
        EV(16);
        tmem_ld_wait();
        EV(11);
        // S is in registers: hand the buffer back
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        EV(12);
#ifdef MIMW_FA_TRACE
        const long long tr2 = clock64();
#endif
        if (need_mask) {
          if (!p.scale_pos) {
            // non-positive scale: move to the log2 domain first (max must see scaled values)
#pragma unroll
            for (int c = 0; c < 128; ++c) s[c] = __float_as_uint(__uint_as_float(s[c]) * p.scale_log2);
          }
          // valid keys of this row form one contiguous column range [c_lo, c_hi]
          const int c_lo = p.causal ? row - p.window + 1 - k0 : -k0;
          const int c_hi = (p.causal ? min(row, p.seq - 1) : p.seq - 1) - k0;
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c < c_lo || c > c_hi) s[c] = 0xff800000u;  // -inf
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              m4[e] = fmax3(m4[e], __uint_as_float(s[c + 2 * e]), __uint_as_float(s[c + 2 * e + 1]));
          }
        }
        // row max over the second half: four independent 3-input max chains
#pragma unroll
        for (int c = 64; c < 128; c += 8) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            m4[e] = fmax3(m4[e], __uint_as_float(s[c + 2 * e]), __uint_as_float(s[c + 2 * e + 1]));
        }
        const float sl = p.scale_pos ? p.scale_log2 : 1.f;
        const float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * sl;
        // online softmax: only move the reference max when it grows by > 8
        // (2^8 headroom in fp32 / bf16 P), which makes O rescales rare.
        float corr = 1.f;
        bool rescale = false;
        if (mx > m_used + 8.f || (m_used == -INFINITY && mx > -INFINITY)) {
          corr = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
          rescale = (j != lo);
          m_used = mx;
        }
        l *= corr;
#ifdef MIMW_FA_TRACE
        const long long tr3 = clock64();
#endif
#ifdef MIMW_FA_TRACE
        const long long tr4 = clock64();
#endif
        // exponentials first, into registers: they do not touch TMEM, so they
        // overlap the tail of PV_h(j-1), which still reads P_h / writes O_h
        const float nm = (m_used == -INFINITY) ? 0.f : -m_used;
        const uint64_t sl2 = f2_pack(sl, sl), nm2 = f2_pack(nm, nm);
        uint64_t acc[4] = {0, 0, 0, 0};
        uint32_t pk[64];
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const int c = 2 * e;
          // x = s * scale*log2e - m, two lanes per FFMA2
          const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sl2, nm2);
          const uint64_t p2 = ((e & 7) < EMU) ? ex2_poly2(x2) : ex2_mufu2(x2);
          acc[e & 3] = f2_add(acc[e & 3], p2);
          pk[e] = pack_bf16_2(p2);
        }
        {
          float a0, a1, b0, b1;
          f2_unpack(f2_add(acc[0], acc[1]), a0, a1);
          f2_unpack(f2_add(acc[2], acc[3]), b0, b1);
          l += (a0 + a1) + (b0 + b1);
        }
        // PV_h(j-1) must be complete before P_h is overwritten / O_h rescaled.
        // o_done[h] can be at most one phase ahead of the one awaited here
        // (PV_h(j) needs this P), so the parity wait is unambiguous.
        if (j > lo) {
          mbar_wait(o_done(h), od_count & 1, 32 + h);
          ++od_count;
          tc_fence_after();
        }
        EV(13);
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int c = 0; c < 128; c += 32) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x16(t_o + c, *reinterpret_cast<uint32_t(*)[16]>(&o[0]));
            tmem_st_32x32b_x16(t_o + c + 16, *reinterpret_cast<uint32_t(*)[16]>(&o[16]));
          }
        }
#pragma unroll
        for (int c = 0; c < 64; c += 16)
          tmem_st_32x32b_x16(t_p + c, *reinterpret_cast<uint32_t(*)[16]>(&pk[c]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full(h));
        EV(14);
#ifdef MIMW_FA_TRACE
        {
          tr_acc[0] += tr1 - tr0;  // waiting for S
          tr_acc[1] += tr2 - tr1;  // TMEM load of S
          tr_acc[2] += tr3 - tr2;  // max + online-softmax bookkeeping
          tr_acc[3] += tr4 - tr3;  // wait PV_h(j-1) + rare O rescale
          tr_acc[5] += clock64() - tr4;  // exp2 + streamed P store + arrive
          tr_acc[4] += 1;
        }
#endif
      }
      // ---------------- epilogue: O / l, lse, straight to HBM ----------------
      mbar_wait(o_done(h), od_count & 1, 40 + h);
      ++od_count;
      tc_fence_after();
      EV(30);
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      if (row < p.seq) {
        if (p.lse != nullptr) p.lse[(size_t)bh * p.seq + row] = (m_used + __log2f(l)) * (1.0f / LOG2E);
      }
      // O / l through a per-warp 4 KiB smem box (32 rows x 64 columns, SW128)
      // and a TMA store per half: coalesced, asynchronous, rows >= seq
      // clipped by the tensor map (a thread per row storing straight to HBM
      // touched 32 lines per warp store: ~3k cycles per item, measured)
      const uint32_t obuf = sbase + SMEM_O + (uint32_t)(warp & 7) * 4096;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t w[32];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(t_o + 64 * half + 32 * cc, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            w[16 * cc + e] = pack_bf16(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
        }
        if (lane == 0) bulk_wait_read<0>();  // the previous store from this box has read it
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(obuf + lane * 128 + ((c ^ (lane & 7)) << 4), w[4 * c], w[4 * c + 1], w[4 * c + 2],
                       w[4 * c + 3]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && p.dbg != 1) {
          tma_store_3d(&tmO, obuf, 64 * half, rt + q * 32, bh);
          bulk_commit();
        }
      }
      tc_fence_before();  // O_h read before the next item's first PV_h overwrites it
      EV(31);
    }
    if (lane == 0) bulk_wait<0>();  // this warp's O stores done before its smem box goes away
    __syncwarp();
#ifdef MIMW_FA_TRACE
    if (p.trace && lane == 0)
      for (int e = 0; e < 8; ++e) p.trace[((size_t)blockIdx.x * 12 + warp) * 8 + e] = tr_acc[e];
#endif
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

#include "attention_fwd_cg2.cuh"

template <int EMU>
cudaError_t launch_cg2(const AttnArgs &a, const Params &p, cudaStream_t stream) {
  const uint64_t bh = (uint64_t)a.batch * a.heads;
  CUtensorMap tQ = make_tmap_3d(a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tK = make_tmap_3d(a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tV = make_tmap_3d(a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tO = make_tmap_3d(a.o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  auto kern = attention_fwd_cg2_kernel<EMU>;
#ifdef MIMW_FA_EVENTS
  constexpr int smem_total = C2_SMEM_TOTAL + 12 * 128 * 8;  // + the event log
#else
  constexpr int smem_total = C2_SMEM_TOTAL;
#endif
  static_assert(smem_total <= 232448, "FA smem");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_total);
  if (e != cudaSuccess) return e;
  const int items = p.bh * p.nqb;
  if (items == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * items, 1, 1);  // one cluster per work item; CLC hands them out
  cfg.blockDim = dim3(C2_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem_total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tQ, tK, tV, tO, p);
}

constexpr int kCounterSlots = 1024;

int *fa_counter_slot() {
  static std::once_flag once[64];
  static int *ring[64] = {};
  static std::atomic<uint32_t> next[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::call_once(once[dev], [dev] {
    int *r = nullptr;
    if (cudaMalloc(&r, sizeof(int) * 2 * kCounterSlots) == cudaSuccess &&
        cudaMemset(r, 0, sizeof(int) * 2 * kCounterSlots) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess)
      ring[dev] = r;
    else
      cudaGetLastError();
  });
  if (!ring[dev]) return nullptr;
  return ring[dev] + 2 * (next[dev].fetch_add(1) % kCounterSlots);
}

}  // namespace

cudaError_t attention_fwd_launch(const AttnArgs &a, cudaStream_t stream) {
  const uint64_t bh = (uint64_t)a.batch * a.heads;
  CUtensorMap tQ = make_tmap_3d(a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tK = make_tmap_3d(a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tO = make_tmap_3d(a.o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tV = make_tmap_3d(a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  Params p;
  p.bh = (int)bh;
  p.seq = (int)a.seq;
  p.causal = a.window > 0 ? 1 : 0;  // window <= 0: non-causal (every key)
  p.window = (int)(a.window > 0 && a.window < a.seq ? a.window : a.seq);
  p.nqb = (int)((a.seq + 2 * BQ - 1) / (2 * BQ));
  p.scale_log2 = (float)(a.scale * 1.4426950408889634);
  p.lse = a.lse;
  p.o = static_cast<__nv_bfloat16 *>(a.o);
  p.trace = a.trace;
  static const int dbg = getenv("MIMW_FA_DEBUG") ? atoi(getenv("MIMW_FA_DEBUG")) : 0;
  p.dbg = dbg;
  p.scale_pos = a.scale > 0 ? 1 : 0;
  // 2-CTA kernel (attention_fwd_cg2.cuh) when asked for (measured slower
  // than the one-CTA kernel on configs[3]: DESIGN.md §4.1)
  static const int cg2_env = getenv("MIMW_FA_CG2") ? atoi(getenv("MIMW_FA_CG2")) : 0;  // A/B knob
  if ((a.cta_group == 2 || cg2_env != 0) && a.max_ctas <= 0) {
    switch (a.emu < 0 ? kDefaultEmuCg2 : a.emu) {
      case 0: return launch_cg2<0>(a, p, stream);
      case 1: return launch_cg2<1>(a, p, stream);
      case 2: return launch_cg2<2>(a, p, stream);
      case 3: return launch_cg2<3>(a, p, stream);
      default: return launch_cg2<4>(a, p, stream);
    }
  }
  const int items = p.bh * p.nqb;
  int grid = sm_count();
  if (a.max_ctas > 0 && a.max_ctas < grid) grid = a.max_ctas;
  if (grid > items) grid = items;
  // Scheduler counter: a slot of a per-device ring of zeroed {claims, retired}
  // pairs, drawn round-robin per launch, so launches on different streams or
  // host threads never share one while in flight; the kernel's last CTA
  // zeroes its slot (no per-launch allocation or memset).
  p.work_counter = fa_counter_slot();
  cudaError_t e = p.work_counter ? cudaSuccess : cudaErrorMemoryAllocation;
  auto launch = [&](auto kern) {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e2 != cudaSuccess) return e2;
    kern<<<grid, NUM_THREADS, SMEM_TOTAL, stream>>>(tQ, tK, tV, tO, p);
    return cudaGetLastError();
  };
  if (e == cudaSuccess) {
    switch (a.emu < 0 ? kDefaultEmu : a.emu) {
      case 0: e = launch(attention_fwd_kernel<0>); break;
      case 1: e = launch(attention_fwd_kernel<1>); break;
      case 2: e = launch(attention_fwd_kernel<2>); break;
      case 3: e = launch(attention_fwd_kernel<3>); break;
      default: e = launch(attention_fwd_kernel<4>); break;
    }
  }
  return e;
}

}  // namespace mimw
