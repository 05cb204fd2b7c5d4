// Warp-specialized flash-attention backward for sm_100a (bf16 in, fp32 accum).
//
// SURVEY.md §8f rank 4 (the ABC rows): gradients of
// o = softmax(scale q k^T) v for every (batch, head), causal (optionally
// windowed, the key range of oracle_attention, oracles.cpp:123-126) or
// non-causal.  The reference has no backward; the oracle is the f64
// restatement in oracle/oracle.c (orc_attention_bwd).
//
//   P = exp(scale S - lse)       S = Q K^T   (lse from the forward)
//   dV = P^T dO    dP = dO V^T    D_i = rowsum(dO_i o O_i)
//   dS = P o (dP - D)    dK = scale dS^T Q    dQ = scale dS K
//
// One CTA per (128-key KV tile, head), K_j / V_j resident in smem; the CTA
// walks the 64-query tiles i that see its keys.  Everything is computed in
// the transposed (key-major) orientation so the key dimension sits on the
// TMEM lanes and P^T / dS^T feed the dV / dK MMAs straight from TMEM:
//   S^T  = K Q_i^T        (SS, M=128 keys, N=64 queries)
//   dP^T = V dO_i^T       (SS)
//   dV  += P^T dO_i       (TS: P^T bf16 in TMEM, dO_i MN-major)
//   dK  += dS^T Q_i       (TS)
//   dQ_i^T = K^T dS^T     (SS: K MN-major, dS^T staged in smem)
// MIMW roles (16 warps):
//   warp 0      TMA producer: K, V once; Q_i, dO_i per step (3 stages)
//   warp 1      MMA issuer (one elected lane), tcgen05.commit -> mbarriers
//   warps 4-11  two "softmax" warpgroups, one per 32-query half of the step:
//               P^T, dS^T from S^T / dP^T (lane = key), P^T / dS^T -> TMEM,
//               dS^T -> smem (double-buffered); final dK, dV epilogue
//   warps 12-15 dQ drain: dQ_i^T TMEM -> smem -> TMA reduce-add (fp32) into
//               a transposed dQ accumulator [bh, 128, seq] in HBM
// TMEM columns: S^T x2 [0,128) (fp32; each warpgroup overwrites its own 32
// columns with P^T | dS^T bf16 once read), dP^T [128,192), dQ^T [192,256),
// dV [256,384), dK [384,512).
// S^T of step i+2 reuses step i's buffer: it is issued after dV_i / dK_i
// (tcgen05.mma ops of one thread execute in issue order).
#include "attention_bwd.h"
#include "ptx.cuh"
#include "pool.h"
#include "tma_host.h"

#include <type_traits>

namespace mimw {

namespace {

constexpr int D = 128;
constexpr int BQ = 64;                    // queries per step (MMA N of S^T / dP^T)
constexpr int BKV = 128;                  // keys per CTA (MMA M)
constexpr int NUM_THREADS = 512;
constexpr int KPANEL = BKV * 128;         // 16 KiB: [128 keys][64 d] bf16, SW128
constexpr int QPANEL = BQ * 128;          // 8 KiB:  [64 queries][64 d]
constexpr int QT_BYTES = 2 * QPANEL;      // one Q_i or dO_i tile
constexpr int SM_K = 0;
constexpr int SM_V = SM_K + 2 * KPANEL;
constexpr int NST = 3;                            // Q_i / dO_i / lse_i / D_i stages
constexpr int SM_Q = SM_V + 2 * KPANEL;
constexpr int SM_DO = SM_Q + NST * QT_BYTES;
constexpr int SM_DS = SM_DO + NST * QT_BYTES;     // 2 x [128 keys][64 queries] bf16, SW128 (16 KiB each)
constexpr int SM_DQ = SM_DS + 2 * BKV * 128;      // 4 warps x 2 boxes x [32 d][32 q] f32 (32 KiB)
constexpr int SM_LD = SM_DQ + 4 * 8192;           // 2 x (lse2[64] + D[64]) f32, softmax warps' double buffer
constexpr int SM_BAR = SM_LD + 2 * 512;
static_assert(SM_BAR + 256 + 1024 <= 232448, "smem");
constexpr int SMEM_TOTAL = SM_BAR + 256 + 1024;
constexpr uint32_t TM_S = 0, TM_DP = 128, TM_DQ = 192, TM_DV = 256, TM_DK = 384;
constexpr uint32_t IDESC_SDP = idesc_bf16(BKV, BQ, 0, 0);  // K-major A, K-major B
constexpr uint32_t IDESC_KV = idesc_bf16(BKV, D, 0, 1);    // A from TMEM, B MN-major
constexpr uint32_t IDESC_DQ = idesc_bf16(D, BQ, 1, 1);     // A = K^T MN-major, B = dS^T MN-major
constexpr float LOG2E = 1.4426950408889634f;

struct BwdParams {
  int bh, seq, window, causal, nkv, nq;
  float scale_log2;    // scale * log2(e)
  float scale;
  const float *lse2;   // [bh, nq * 64] lse * log2(e), zero padded
  const float *dvec;   // [bh, nq * 64] rowsum(dO o O), zero padded
  __nv_bfloat16 *dk, *dv;
};

// Query tiles [i_lo, i_hi] that see keys [128 j, 128 j + 127]
__device__ __forceinline__ void q_range(int j, const BwdParams &p, int &lo, int &hi) {
  if (!p.causal) {
    lo = 0;
    hi = p.nq - 1;
    return;
  }
  lo = (j * BKV) / BQ;
  hi = min(p.nq - 1, (j * BKV + BKV - 1 + p.window - 1) / BQ);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tma_reduce_add_3d(const void *tmap, uint32_t src, int32_t x, int32_t y,
                                                  int32_t z) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(src), "r"(x), "r"(y), "r"(z)
      : "memory");
}

#ifdef MIMW_BWD_TRACE
// per-warp cycle accounting of the first 4 CTAs (tools/bwd_trace.py):
// [cta][warp][8] = role-specific wait buckets, [7] = total
__device__ unsigned long long g_bwd_trace[4 * 16 * 8];
#define TR_DECL unsigned long long tr_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; const long long tr_t0 = clock64();
#define TR(i, stmt) do { const long long t_ = clock64(); stmt; tr_[i] += clock64() - t_; } while (0)
#define TR_END \
  if (blockIdx.x < 4 && lane == 0) { tr_[7] = clock64() - tr_t0; \
    for (int e_ = 0; e_ < 8; ++e_) g_bwd_trace[(blockIdx.x * 16 + warp) * 8 + e_] = tr_[e_]; }
#else
#define TR_DECL
#define TR(i, stmt) stmt
#define TR_END
#endif

__global__ void __launch_bounds__(NUM_THREADS, 1)
attention_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmDQ, BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + SM_BAR;
  const uint32_t kv_full = bars;
  auto ld_full = [&](int s) { return bars + 8 + 8 * s; };
  auto ld_empty = [&](int s) { return bars + 8 + 8 * NST + 8 * s; };
  const uint32_t b0 = bars + 8 + 16 * NST;
  const uint32_t s_full = b0, dp_free = b0 + 8, p_full = b0 + 16;
  auto ds_free = [&](int b) { return b0 + 24 + 8 * b; };
  const uint32_t dq_full = b0 + 40, dq_free = b0 + 48, acc_full = b0 + 56;
  const uint32_t tmem_slot = b0 + 64;
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + SM_BAR + 8 + 16 * NST + 64);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  // Head-major order: the KV tiles of one head run together, so the head's
  // Q / dO (read by every one of them) and its dQ accumulator (reduced into by
  // every one of them) stay L2-resident.  Measured with the KV-tile-major
  // order: 157 GB of DRAM traffic per ABC4 launch (dQ reductions missing L2).
  const int bh = blockIdx.x / p.nkv;
  const int j = blockIdx.x % p.nkv;
  int i_lo, i_hi;
  q_range(j, p, i_lo, i_hi);
  const int n = i_hi - i_lo + 1;
  // step t visits query tile i_lo + (t + j) % n: the head's KV tiles start at
  // different query tiles, so their dQ reductions do not pile onto one tile
  auto q_tile = [&](int t) { int r = t + j; r -= (r / n) * n; return i_lo + r; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    tma_prefetch_desc(&tmDQ);
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(ld_full(s), 1);
      mbar_init(ld_empty(s), 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_free, 8);
    mbar_init(p_full, 8);
    mbar_init(ds_free(0), 1);
    mbar_init(ds_free(1), 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  TR_DECL

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0 && n > 0) {
      mbar_arrive_expect_tx(kv_full, 4 * KPANEL);
      for (int h = 0; h < 2; ++h) {
        tma_load_3d(sbase + SM_K + h * KPANEL, &tmK, kv_full, 64 * h, j * BKV, bh);
        tma_load_3d(sbase + SM_V + h * KPANEL, &tmV, kv_full, 64 * h, j * BKV, bh);
      }
      for (int t = 0; t < n; ++t) {
        const int s = t % NST;
        const int i = q_tile(t);
        TR(1, mbar_wait(ld_empty(s), ((t / NST) & 1) ^ 1, 1));
        mbar_arrive_expect_tx(ld_full(s), 2 * QT_BYTES);
        for (int h = 0; h < 2; ++h) {
          tma_load_3d(sbase + SM_Q + s * QT_BYTES + h * QPANEL, &tmQ, ld_full(s), 64 * h, i * BQ, bh);
          tma_load_3d(sbase + SM_DO + s * QT_BYTES + h * QPANEL, &tmDO, ld_full(s), 64 * h, i * BQ, bh);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (n > 0) {
      const uint32_t tm = tmem;
      constexpr uint32_t HI = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, version 1, SW128
      constexpr uint32_t LO_K = (16u >> 4) << 16;                       // K-major: LBO unused
      auto issue_S = [&](int t, bool dp) {
        const int st = t % NST;
        if (!dp) TR(1, mbar_wait(ld_full(st), (t / NST) & 1, 2));
        tc_fence_after();
        const uint32_t a0 = (sbase + (dp ? SM_V : SM_K)) >> 4;
        const uint32_t b0 = (sbase + (dp ? SM_DO : SM_Q) + st * QT_BYTES) >> 4;
        const uint32_t d = tm + (dp ? TM_DP : TM_S + 64 * (t & 1));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t offa = ((k >> 2) * KPANEL + (k & 3) * 32) >> 4;
            const uint32_t offb = ((k >> 2) * QPANEL + (k & 3) * 32) >> 4;
            mma_f16_ss<1>(d, make_desc(LO_K | (a0 + offa), HI), make_desc(LO_K | (b0 + offb), HI),
                          IDESC_SDP, k != 0);
          }
        }
        __syncwarp();
      };
      mbar_wait(kv_full, 0, 3);
      issue_S(0, false);
      issue_S(0, true);
      if (elect_one()) mma_commit(s_full);
      __syncwarp();
      if (n > 1) issue_S(1, false);
      for (int t = 0; t < n; ++t) {
        const int s = t & 1;      // S^T buffer and dS^T smem buffer
        const int st = t % NST;   // Q / dO stage
        if (t + 1 < n) {
          TR(2, mbar_wait(dp_free, t & 1, 4));  // dP^T_t is in the softmax warps' registers
          issue_S(t + 1, true);
          if (elect_one()) mma_commit(s_full);
          __syncwarp();
        }
        TR(3, mbar_wait(p_full, t & 1, 5));
        tc_fence_after();
        if (t >= 1) {
          TR(4, mbar_wait(dq_free, (t - 1) & 1, 6));  // dQ^T_{t-1} drained
          tc_fence_after();
        }
        if (elect_one()) {
          const uint32_t bq = (sbase + SM_Q + st * QT_BYTES) >> 4;
          const uint32_t bdo = (sbase + SM_DO + st * QT_BYTES) >> 4;
          constexpr uint32_t LO_QMN = ((uint32_t)QPANEL >> 4) << 16;  // LBO: D-panel stride
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k) {  // K = 64 queries: 16 query rows (2 KiB) per step
            // query half h = k / 2 lives in columns [32h, 32h + 32): P^T | dS^T
            const uint32_t a_p = tm + TM_S + 64 * s + 32 * (k >> 1) + 8 * (k & 1);
            const uint32_t a_ds = a_p + 16;
            mma_f16_ts<1>(tm + TM_DV, a_p, make_desc(LO_QMN | (bdo + k * (2048 >> 4)), HI), IDESC_KV,
                          (t | k) != 0);
            mma_f16_ts<1>(tm + TM_DK, a_ds, make_desc(LO_QMN | (bq + k * (2048 >> 4)), HI), IDESC_KV,
                          (t | k) != 0);
          }
          const uint32_t ak = (sbase + SM_K) >> 4;
          const uint32_t bds = (sbase + SM_DS + s * BKV * 128) >> 4;
          constexpr uint32_t LO_KMN = ((uint32_t)KPANEL >> 4) << 16;  // LBO: D-panel stride of K
          constexpr uint32_t LO_DSMN = ((uint32_t)(BKV * 128) >> 4) << 16;
#pragma unroll
          for (int k = 0; k < BKV / 16; ++k)  // K = 128 keys
            mma_f16_ss<1>(tm + TM_DQ, make_desc(LO_KMN | (ak + k * (2048 >> 4)), HI),
                          make_desc(LO_DSMN | (bds + k * (2048 >> 4)), HI), IDESC_DQ, k != 0);
          mma_commit(dq_full);
          mma_commit(ld_empty(st));
          mma_commit(ds_free(s));
          if (t == n - 1) mma_commit(acc_full);
        }
        __syncwarp();
        if (t + 2 < n) issue_S(t + 2, false);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= softmax warpgroups (lane = key, ch = query half) =================
    const int qq = warp & 3;
    const int ch = (warp - 4) >> 2;
    const int krow = qq * 32 + (int)lane;      // key row inside the tile
    const int key = j * BKV + krow;
    const uint32_t t_lane = (uint32_t)(qq * 32) << 16;
    const int ctid = (int)threadIdx.x - 128;  // 0..255 over the softmax warps
    if (n > 0 && ctid < 128) {
      const float *src = ctid < 64 ? p.lse2 : p.dvec;
      sts_f32(sbase + SM_LD + ctid * 4, __ldg(src + ((size_t)bh * p.nq + q_tile(0)) * BQ + (ctid & 63)));
    }
    named_bar_sync(1, 256);
    for (int t = 0, i = q_tile(0); t < n; ++t, i = (i == i_hi) ? i_lo : i + 1) {  // i = q_tile(t)
      const int s = t & 1;
      const int i_next = (i == i_hi) ? i_lo : i + 1;
      // lse2 / D of the NEXT step: one value per thread (threads 0-63 lse2,
      // 64-127 D), loaded now, published into the smem double buffer at the end
      // of this step (named barrier among the softmax warps)
      float pre = 0.f;
      if (t + 1 < n && ctid < 128) {
        const float *src = ctid < 64 ? p.lse2 : p.dvec;
        pre = __ldg(src + ((size_t)bh * p.nq + i_next) * BQ + (ctid & 63));
      }
      TR(1, mbar_wait(s_full, t & 1, 7));
      tc_fence_after();
      uint32_t sv[32], dp[32];
      const uint32_t t_s = tmem + t_lane + TM_S + 64 * s + 32 * ch;
      tmem_ld_32x32b_x32(t_s, sv);
      tmem_ld_32x32b_x32(tmem + t_lane + TM_DP + 32 * ch, dp);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dp_free);
      const int q0 = i * BQ + 32 * ch;
      uint32_t pk[16], dk2[16];
      // per-score causal/window test only where some (key, query) pair of
      // this CTA's 128 keys x this half's 32 queries is outside the band
      const bool full = !p.causal || (j * BKV + BKV - 1 <= q0 && q0 + 31 - j * BKV < p.window);
      auto scores = [&](auto masked) {
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        // explicit ld.shared (a generic pointer here compiled to LD.E: address
        // translation and 2 wavefronts per broadcast load)
        const float4 l4 = lds_f4(sbase + SM_LD + (t & 1) * 512 + (32 * ch + 4 * c4) * 4);
        const float4 d4 = lds_f4(sbase + SM_LD + (t & 1) * 512 + 256 + (32 * ch + 4 * c4) * 4);
        const float la[4] = {l4.x, l4.y, l4.z, l4.w};
        const float da[4] = {d4.x, d4.y, d4.z, d4.w};
        float pv[4], dsv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = 4 * c4 + e;
          const int qi = q0 + c;
          const bool valid = !decltype(masked)::value || (key <= qi && qi - key < p.window);
          const float x = __uint_as_float(sv[c]) * p.scale_log2 - la[e];
          const float pe = valid ? ex2(x) : 0.f;
          pv[e] = pe;
          dsv[e] = pe * (__uint_as_float(dp[c]) - da[e]);
        }
        pk[2 * c4] = pack_bf16(pv[0], pv[1]);
        pk[2 * c4 + 1] = pack_bf16(pv[2], pv[3]);
        dk2[2 * c4] = pack_bf16(dsv[0], dsv[1]);
        dk2[2 * c4 + 1] = pack_bf16(dsv[2], dsv[3]);
      }
      };
      if (full) scores(std::false_type{});
      else scores(std::true_type{});
      // P^T | dS^T (bf16) over this half's S^T columns, already read
      tmem_st_32x32b_x16(t_s, pk);
      tmem_st_32x32b_x16(t_s + 16, dk2);
      // dS^T half-row -> smem buffer s (B operand of dQ^T, MN-major SW128:
      // 16-B chunk c of row r at c ^ (r & 7)); buffer s was last read by dQ_{t-2}
      if (t >= 2) TR(2, mbar_wait(ds_free(s), ((t - 2) >> 1) & 1, 9));
      const uint32_t rbase = sbase + SM_DS + s * BKV * 128 + krow * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        st_shared_v4(rbase + (((4 * ch + c) ^ (krow & 7)) * 16), dk2[4 * c], dk2[4 * c + 1],
                     dk2[4 * c + 2], dk2[4 * c + 3]);
      fence_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (ctid < 128) sts_f32(sbase + SM_LD + ((t + 1) & 1) * 512 + ctid * 4, pre);
      TR(3, named_bar_sync(1, 256));  // next step's lse2 / D visible; this step's reads done
    }
    // ---------------- epilogue: dV, dK (x scale) -> bf16 HBM ----------------
    if (n > 0) {
      mbar_wait(acc_full, 0, 10);
      tc_fence_after();
    }
    {
      const int which = ch;  // warpgroup 0 writes dV, warpgroup 1 dK
      __nv_bfloat16 *dst = which == 0 ? p.dv : p.dk;
      const float mul = which == 0 ? 1.f : p.scale;
      uint4 *orow = reinterpret_cast<uint4 *>(dst + ((size_t)bh * p.seq + key) * D);
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        uint32_t v[32];
        if (n > 0) {
          tmem_ld_32x32b_x32(tmem + t_lane + (which == 0 ? TM_DV : TM_DK) + c, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
        if (key < p.seq) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(v[8 * g + 0]) * mul, __uint_as_float(v[8 * g + 1]) * mul);
            w.y = pack_bf16(__uint_as_float(v[8 * g + 2]) * mul, __uint_as_float(v[8 * g + 3]) * mul);
            w.z = pack_bf16(__uint_as_float(v[8 * g + 4]) * mul, __uint_as_float(v[8 * g + 5]) * mul);
            w.w = pack_bf16(__uint_as_float(v[8 * g + 6]) * mul, __uint_as_float(v[8 * g + 7]) * mul);
            orow[c / 8 + g] = w;
          }
        }
      }
    }
  } else if (warp >= 12) {
    // ================= dQ drain (lane = head-dim row of dQ^T) =================
    const int dd = warp & 3;
    const uint32_t t_lane = (uint32_t)(dd * 32) << 16;
    const uint32_t stage = sbase + SM_DQ + dd * 8192;
    for (int t = 0; t < n; ++t) {
      const int i = q_tile(t);
      TR(1, mbar_wait(dq_full, t & 1, 11));
      tc_fence_after();
      uint32_t v[64];
      tmem_ld_32x32b_x32(tmem + t_lane + TM_DQ, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      tmem_ld_32x32b_x32(tmem + t_lane + TM_DQ + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(dq_free);
        TR(2, bulk_wait_read<0>());  // the previous reduce has read the staging buffer
      }
      __syncwarp();
      // two boxes [32 d][32 queries] f32, SWIZZLE_128B: chunk c of row r at c ^ (r & 7)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const uint32_t rb = stage + b * 4096 + lane * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(rb + ((c ^ (lane & 7)) * 16), v[32 * b + 4 * c], v[32 * b + 4 * c + 1],
                       v[32 * b + 4 * c + 2], v[32 * b + 4 * c + 3]);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_reduce_add_3d(&tmDQ, stage, i * BQ, dd * 32, bh);
        tma_reduce_add_3d(&tmDQ, stage + 4096, i * BQ + 32, dd * 32, bh);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  TR_END
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

// D = rowsum(dO o O) and lse2 = lse * log2(e), both zero padded to nq * 64
// per head; one warp per PREP_ROWS rows, every row's loads issued before the
// first reduction (more bytes in flight per warp than one row at a time).
constexpr int PREP_ROWS = 4;
__global__ void attention_bwd_prep(const __nv_bfloat16 *o, const __nv_bfloat16 *dout, const float *lse,
                                   float *lse2, float *dvec, int bh, int seq, int npad) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const int r0 = warp * PREP_ROWS;  // npad is a multiple of 64, so a warp's rows share one head
  if (r0 >= bh * npad) return;
  const int b = r0 / npad, s0 = r0 % npad;
  uint2 ov[PREP_ROWS], dv[PREP_ROWS];
  float l2[PREP_ROWS];
#pragma unroll
  for (int i = 0; i < PREP_ROWS; ++i) {
    const int s = s0 + i;
    ov[i] = make_uint2(0, 0);
    dv[i] = make_uint2(0, 0);
    l2[i] = 0.f;
    if (s < seq) {
      const size_t row = (size_t)b * seq + s;
      ov[i] = reinterpret_cast<const uint2 *>(o + row * D)[lane];
      dv[i] = reinterpret_cast<const uint2 *>(dout + row * D)[lane];
      l2[i] = lse[row] * LOG2E;
    }
  }
#pragma unroll
  for (int i = 0; i < PREP_ROWS; ++i) {
    const __nv_bfloat162 *o2 = reinterpret_cast<const __nv_bfloat162 *>(&ov[i]);
    const __nv_bfloat162 *d2 = reinterpret_cast<const __nv_bfloat162 *>(&dv[i]);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float2 of = __bfloat1622float2(o2[e]);
      const float2 df = __bfloat1622float2(d2[e]);
      acc += of.x * df.x + of.y * df.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == i) {
      dvec[(size_t)b * npad + s0 + i] = acc;
      lse2[(size_t)b * npad + s0 + i] = l2[i];
    }
  }
}

// dQ[bh, s, d] = bf16(scale * dQacc^T[bh, d, s]) through 64 (d) x 32 (s) smem
// tiles: 128-B coalesced loads along s, and each warp stores one dQ row
// segment of 64 d as bf16x2 (128 B), so both sides move whole lines.
__global__ void __launch_bounds__(256) attention_bwd_dq(const float *acc, __nv_bfloat16 *dq, int seq, int ld,
                                                        float scale) {
  __shared__ float tile[64][33];
  const int b = blockIdx.z;
  const int s0 = blockIdx.x * 32, d0 = blockIdx.y * 64;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 8 warps
  const float *src = acc + (size_t)b * D * ld;
#pragma unroll
  for (int r = w; r < 64; r += 8) {
    const int s = s0 + lane;
    tile[r][lane] = s < seq ? src[(size_t)(d0 + r) * ld + s] : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int r = w; r < 32; r += 8) {
    const int s = s0 + r;
    if (s < seq) {
      const __nv_bfloat162 v = __floats2bfloat162_rn(tile[2 * lane][r] * scale, tile[2 * lane + 1][r] * scale);
      reinterpret_cast<__nv_bfloat162 *>(dq + ((size_t)b * seq + s) * D + d0)[lane] = v;
    }
  }
}

}  // namespace

cudaError_t attention_bwd_launch(const AttnBwdArgs &a, cudaStream_t stream) {
  const int bh = (int)(a.batch * a.heads);
  const int seq = (int)a.seq;
  if (bh == 0 || seq == 0) return cudaSuccess;
  const int nq = (seq + BQ - 1) / BQ;
  const int nkv = (seq + BKV - 1) / BKV;
  const int npad = nq * BQ;
  // workspace: dQ accumulator [bh, 128, npad] f32 (rows padded to the query
  // tile so the TMA row stride is a 256-B multiple for any seq), lse2 / D
  // [bh, npad] f32
  const size_t acc_bytes = (size_t)bh * D * npad * 4;
  const size_t vec_bytes = (size_t)bh * npad * 4;
  char *ws = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void **>(&ws), acc_bytes + 2 * vec_bytes + 256, stream);
  if (e != cudaSuccess) return e;
  float *acc = reinterpret_cast<float *>(ws);
  float *lse2 = reinterpret_cast<float *>(ws + acc_bytes);
  float *dvec = reinterpret_cast<float *>(ws + acc_bytes + vec_bytes);
  e = cudaMemsetAsync(acc, 0, acc_bytes, stream);
  if (e == cudaSuccess) {
    const int rows = bh * npad;
    attention_bwd_prep<<<(rows + 8 * PREP_ROWS - 1) / (8 * PREP_ROWS), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16 *>(a.o), static_cast<const __nv_bfloat16 *>(a.dout), a.lse, lse2,
        dvec, bh, seq, npad);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    const uint64_t ubh = (uint64_t)bh;
    CUtensorMap tQ = make_tmap_3d(a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, seq, ubh, D, (uint64_t)seq * D, 64,
                                  BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tDO = make_tmap_3d(a.dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, seq, ubh, D,
                                   (uint64_t)seq * D, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tK = make_tmap_3d(a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, seq, ubh, D, (uint64_t)seq * D, 64,
                                  BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tV = make_tmap_3d(a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, seq, ubh, D, (uint64_t)seq * D, 64,
                                  BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tDQ = make_tmap_3d(acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, seq, D, ubh, npad, (uint64_t)D * npad,
                                   32, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    BwdParams p;
    p.bh = bh;
    p.seq = seq;
    p.causal = a.window > 0 ? 1 : 0;
    p.window = (int)(a.window > 0 && a.window < a.seq ? a.window : a.seq);
    p.nkv = nkv;
    p.nq = nq;
    p.scale = (float)a.scale;
    p.scale_log2 = (float)(a.scale * 1.4426950408889634);
    p.lse2 = lse2;
    p.dvec = dvec;
    p.dk = static_cast<__nv_bfloat16 *>(a.dk);
    p.dv = static_cast<__nv_bfloat16 *>(a.dv);
    e = cudaFuncSetAttribute(attention_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e == cudaSuccess) {
      attention_bwd_kernel<<<nkv * bh, NUM_THREADS, SMEM_TOTAL, stream>>>(tQ, tK, tV, tDO, tDQ, p);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) {
    attention_bwd_dq<<<dim3((seq + 31) / 32, D / 64, bh), 256, 0, stream>>>(
        acc, static_cast<__nv_bfloat16 *>(a.dq), seq, npad, (float)a.scale);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(ws, stream);
  return e != cudaSuccess ? e : e2;
}

}  // namespace mimw

// Debug hook (not in the public header): per-warp cycle buckets of the first
// 4 CTAs when built with -DMIMW_BWD_TRACE (tools/bwd_trace.py).
extern "C" int mimw_b200_debug_bwd_trace(unsigned long long *host, int n) {
#ifdef MIMW_BWD_TRACE
  if (n > 4 * 16 * 8) n = 4 * 16 * 8;
  return cudaMemcpyFromSymbol(host, mimw::g_bwd_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 3;
#else
  (void)host;
  (void)n;
  return 2;
#endif
}
