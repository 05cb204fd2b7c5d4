// Warp-specialized flash-attention forward for sm_100a (bf16 in, fp32 accum).
//
// Computes, per (batch, head), the reference's windowed causal softmax
// attention  oracle_attention(q, k, v, w, scale)  (proj/core/src/
// oracles.cpp:119-145): keys j in [max(0, i-w+1), i], softmax in the exp
// domain, o = P.V.  Also returns lse = m + log(l) as the simplicial program
// does (oracles.cpp:116, simplicial_attention.mimw:88-93).
//
// MIMW structure (the B200 form of proj/kernels/simplicial_attention.mimw:
// producer task staging K/V blocks through barriers + consumer online
// softmax), one persistent CTA per SM, 10 warps:
//   warps 0-3  softmax WG 0 : Q tile 0 (rows q0 .. q0+127), one row per thread
//   warps 4-7  softmax WG 1 : Q tile 1 (rows q0+128 .. q0+255)  (ping-pong)
//   warp 8     TMA producer : Q0, Q1, then K_j / V_j through a 5-slot ring
//   warp 9     MMA issuer   : S_h = Q_h K_j^T (SS-MMA into TMEM),
//                             O_h += P_h V_j (TS-MMA, P read from TMEM)
// The softmax WG owning Q tile h also performs the online-softmax correction
// (conditional O rescale in TMEM when the running max grows by > 2^8) and the
// epilogue (O / l -> bf16 -> smem -> TMA store, lse -> HBM).
//
// MMA issue order per KV step j:  PV_0(j), S_0(j+1), PV_1(j), S_1(j+1).
// tcgen05 ops of one thread complete in order and a commit covers all prior
// ops, so when softmax h sees S_h(j+1) complete, PV_h(j) is complete too:
// O_h is stable for the in-place rescale without an extra barrier, and P_h(j)
// (which aliases S_h's TMEM columns) has been consumed before S_h(j+1)
// overwrites it.
//
// TMEM (512 columns x 128 lanes, fp32): S_0 [0,128) S_1 [128,256)
//   O_0 [256,384) O_1 [384,512); P_h (bf16, 64 columns) aliases S_h.
#include "attention_fwd.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace mimw {

namespace {

constexpr int D = 128;           // head dim (QK^T K-extent, PV N-extent)
constexpr int BQ = 128;          // rows per Q tile (MMA M)
constexpr int BKV = 128;         // keys per KV tile (S N-extent, PV K-extent)
constexpr int NSLOT = 5;         // K/V ring slots (32 KiB each)
constexpr int TILE_BYTES = BKV * D * 2;  // 32 KiB: one Q, K or V tile
constexpr int HALF_BYTES = TILE_BYTES / 2;  // one 64-column (128-B) swizzle panel
constexpr int NUM_THREADS = 384;  // 3 warpgroups: softmax 0, softmax 1, {load, MMA, 2 spare}
constexpr int SMEM_Q = 0;
constexpr int SMEM_KV = 2 * TILE_BYTES;
constexpr int SMEM_BAR = SMEM_KV + NSLOT * TILE_BYTES;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
constexpr uint32_t IDESC_S = idesc_bf16(BQ, BKV, 0, 0);   // Q (K-major) x K (K-major)
constexpr uint32_t IDESC_PV = idesc_bf16(BQ, D, 0, 1);    // P (TMEM) x V (MN-major)
constexpr float LOG2E = 1.4426950408889634f;
constexpr int kDefaultEmu = 2;  // exp2 pairs (of 8) evaluated on the FMA pipe

struct Params {
  int bh;            // batch * heads
  int seq;
  int window;        // keys j in [i - window + 1, i]
  int nqb;           // 256-row blocks per head
  float scale_log2;  // scale * log2(e)
  float *lse;        // [bh, seq] or null
  int scale_pos;     // scale > 0: max on raw scores, scale folded into FFMA2
  unsigned long long *trace;  // optional per-warp cycle accounting [grid][12][8]
};

// KV tile range [lo, hi] needed by Q rows [r0, r0 + 127]
__device__ __forceinline__ void kv_range(int r0, const Params &p, int &lo, int &hi) {
  int last = min(r0 + BQ - 1, p.seq - 1);
  int first_key = max(0, r0 - p.window + 1);
  lo = first_key / BKV;
  hi = last / BKV;
}

__device__ __forceinline__ void work_item(int idx, const Params &p, int &bh, int &qb) {
  // longest-first: largest q-block (most KV tiles under the causal mask) first
  qb = p.nqb - 1 - idx / p.bh;
  bh = idx % p.bh;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ uint64_t ex2_mufu2(uint64_t x2) {
  float a, b;
  f2_unpack(x2, a, b);
  return f2_pack(ex2(a), ex2(b));
}

// exp2 on the FMA pipe (offloads the MUFU, the FA-forward co-bottleneck):
// x = n + f, n = rint(x) via the 1.5*2^23 magic, f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. err 7.5e-5, far below the
// bf16 rounding of P); 2^n folded into the exponent bits.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float a, b;
  f2_unpack(x2, a, b);
  a = fmaxf(a, -126.f);  // 2^-126 keeps the exponent field >= 0 (no wrap to NaN)
  b = fmaxf(b, -126.f);
  const uint64_t x = f2_pack(a, b);
  const uint64_t t = f2_add(x, f2_pack(12582912.f, 12582912.f));
  const uint64_t r = f2_add(t, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = f2_fma(r, f2_pack(-1.f, -1.f), x);
  uint64_t q = f2_fma(f2_pack(0.0551824f, 0.0551824f), f, f2_pack(0.24261211f, 0.24261211f));
  q = f2_fma(q, f, f2_pack(0.693259f, 0.693259f));
  q = f2_fma(q, f, f2_pack(0.99992794f, 0.99992794f));
  float t0, t1, q0, q1;
  f2_unpack(t, t0, t1);
  f2_unpack(q, q0, q1);
  const float y0 = __int_as_float((__float_as_int(t0) << 23) + __float_as_int(q0));
  const float y1 = __int_as_float((__float_as_int(t1) << 23) + __float_as_int(q1));
  return f2_pack(y0, y1);
}

__device__ __forceinline__ uint32_t pack_bf16_2(uint64_t v) {
  float a, b;
  f2_unpack(v, a, b);
  return pack_bf16(a, b);
}

template <int EMU>
__global__ void __launch_bounds__(NUM_THREADS, 1)
attention_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + SMEM_BAR;
  auto q_full = [&](int h) { return bars + 8 * h; };
  auto q_empty = [&](int h) { return bars + 16 + 8 * h; };
  auto s_full = [&](int h) { return bars + 32 + 8 * h; };
  auto p_full = [&](int h) { return bars + 48 + 8 * h; };
  auto o_full = [&](int h) { return bars + 64 + 8 * h; };
  auto kv_full = [&](int s) { return bars + 80 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 80 + 8 * NSLOT + 8 * s; };
  const uint32_t tmem_slot = bars + 80 + 16 * NSLOT;
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + SMEM_BAR + 80 + 16 * NSLOT);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const int num_items = p.bh * p.nqb;

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    for (int h = 0; h < 2; ++h) {
      mbar_init(q_full(h), 1);
      mbar_init(q_empty(h), 4);
      mbar_init(s_full(h), 1);
      mbar_init(p_full(h), 4);
      mbar_init(o_full(h), 1);
    }
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
  // control warpgroup gives registers to the two softmax warpgroups
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 8) {
    // ================= TMA producer =================
    if (lane == 0) {
      int slot = 0;
      uint32_t slot_phase = 0;
      uint32_t qe_phase = 0;
      for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
        int bh, qb;
        work_item(it, p, bh, qb);
        const int r0 = qb * 2 * BQ;
        int lo0, hi0, lo1, hi1;
        kv_range(r0, p, lo0, hi0);
        kv_range(r0 + BQ, p, lo1, hi1);
        if (r0 + BQ >= p.seq) hi1 = hi0;  // Q tile 1 entirely beyond seq: no extra tile
        const int lo = min(lo0, lo1), hi = max(hi0, hi1);
        for (int h = 0; h < 2; ++h) {
          mbar_wait(q_empty(h), qe_phase ^ 1, 10);
          mbar_arrive_expect_tx(q_full(h), TILE_BYTES);
          const uint32_t dq = sbase + SMEM_Q + h * TILE_BYTES;
          tma_load_3d(dq, &tmQ, q_full(h), 0, r0 + h * BQ, bh);
          tma_load_3d(dq + HALF_BYTES, &tmQ, q_full(h), 64, r0 + h * BQ, bh);
        }
        qe_phase ^= 1;
        for (int j = lo; j <= hi; ++j) {
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
  } else if (warp == 9) {
    // ================= MMA issuer =================
    if (lane == 0) {
      int slot = 0;
      uint32_t slot_phase = 0;
      uint32_t q_phase = 0;
      uint32_t p_phase[2] = {0, 0};
      // Descriptors are rebuilt per MMA from 32-bit pieces (cheap ALU) so the
      // register-starved control warpgroup does not hoist 64-bit constants.
      constexpr uint32_t HI_KMAJ = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO, version, SW128
      constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;                         // LBO (unused)
      constexpr uint32_t LO_VMN = ((uint32_t)HALF_BYTES >> 4) << 16;         // LBO = D-panel stride
      auto issue_S = [&](int h, uint32_t kslot) {
        const uint32_t qa = (sbase + SMEM_Q + h * TILE_BYTES) >> 4;
        const uint32_t kb = (sbase + SMEM_KV + kslot * TILE_BYTES) >> 4;
        const uint32_t d = tmem + h * 128;
#pragma unroll 1
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k >> 2) * HALF_BYTES + (k & 3) * 32) >> 4;
          mma_f16_ss<1>(d, make_desc(LO_KMAJ | (qa + off), HI_KMAJ), make_desc(LO_KMAJ | (kb + off), HI_KMAJ),
                        IDESC_S, k != 0);
        }
        mma_commit(s_full(h));
      };
      auto issue_PV = [&](int h, uint32_t vslot, bool acc) {
        const uint32_t vb = (sbase + SMEM_KV + vslot * TILE_BYTES) >> 4;
        const uint32_t d = tmem + 256 + h * 128;
        const uint32_t a = tmem + h * 128;
#pragma unroll 1
        for (int k = 0; k < BKV / 16; ++k) {
          mma_f16_ts<1>(d, a + k * 8, make_desc(LO_VMN | (vb + k * (2048 >> 4)), HI_KMAJ), IDESC_PV,
                        (acc || k != 0) ? 1u : 0u);
        }
      };
      long long mt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
        int bh, qb;
        work_item(it, p, bh, qb);
        const int r0 = qb * 2 * BQ;
        int lo0, hi0, lo1, hi1;
        kv_range(r0, p, lo0, hi0);
        kv_range(r0 + BQ, p, lo1, hi1);
        const bool has1 = r0 + BQ < p.seq;
        if (!has1) hi1 = hi0;
        const int lo = min(lo0, lo1), hi = max(hi0, hi1);
        auto in0 = [&](int j) { return j >= lo0 && j <= hi0; };
        auto in1 = [&](int j) { return has1 && j >= lo1 && j <= hi1; };

        mbar_wait(q_full(0), q_phase, 20);
        mbar_wait(q_full(1), q_phase, 21);
        q_phase ^= 1;
        tc_fence_after();
        // prologue: S_h(lo)
        int kslot = slot;
        mbar_wait(kv_full(kslot), slot_phase, 22);
        tc_fence_after();
        if (in0(lo)) issue_S(0, kslot);
        if (in1(lo)) issue_S(1, kslot);
        mma_commit(kv_empty(kslot));
        if (++slot == NSLOT) { slot = 0; slot_phase ^= 1; }
        for (int j = lo; j <= hi; ++j) {
          const int vslot = slot;
          const long long m2 = p.trace ? clock64() : 0;
          mbar_wait(kv_full(vslot), slot_phase, 23);
          if (p.trace) { mt_acc[2] += clock64() - m2; mt_acc[4] += 1; }
          if (++slot == NSLOT) { slot = 0; slot_phase ^= 1; }
          int nslot = -1;
          if (j + 1 <= hi) {
            nslot = slot;
            mbar_wait(kv_full(nslot), slot_phase, 24);
            if (++slot == NSLOT) { slot = 0; slot_phase ^= 1; }
          }
          tc_fence_after();
          if (in0(j)) {
            const long long m0 = p.trace ? clock64() : 0;
            mbar_wait(p_full(0), p_phase[0], 25);
            if (p.trace) mt_acc[0] += clock64() - m0;
            p_phase[0] ^= 1;
            tc_fence_after();
            issue_PV(0, vslot, j != lo0);
            if (j == hi0) mma_commit(o_full(0));
          }
          if (nslot >= 0 && in0(j + 1)) issue_S(0, nslot);
          if (in1(j)) {
            const long long m1 = p.trace ? clock64() : 0;
            mbar_wait(p_full(1), p_phase[1], 26);
            if (p.trace) mt_acc[1] += clock64() - m1;
            p_phase[1] ^= 1;
            tc_fence_after();
            issue_PV(1, vslot, j != lo1);
            if (j == hi1) mma_commit(o_full(1));
          }
          mma_commit(kv_empty(vslot));
          if (nslot >= 0) {
            if (in1(j + 1)) issue_S(1, nslot);
            mma_commit(kv_empty(nslot));
          }
        }
      }
      if (p.trace)
        for (int e = 0; e < 8; ++e) p.trace[((size_t)blockIdx.x * 12 + warp) * 8 + e] = mt_acc[e];
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ================= softmax / correction / epilogue (WG h) =================
    const int h = warp >> 2;             // Q tile owned by this warpgroup
    const int q = warp & 3;              // TMEM lane quarter
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const uint32_t t_s = tmem + t_lane + h * 128;
    const uint32_t t_o = tmem + t_lane + 256 + h * 128;
    uint32_t s_phase = 0, o_phase = 0;
    long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
      int bh, qb;
      work_item(it, p, bh, qb);
      const int rt = qb * 2 * BQ + h * BQ;  // first row of this Q tile
      const int row = rt + q * 32 + (int)lane;
      const bool tile_live = rt < p.seq;
      int lo, hi;
      kv_range(rt, p, lo, hi);
      float m_used = -INFINITY;  // log2-domain max the exponentials are taken against
      float l = 0.f;
      if (tile_live) {
        for (int j = lo; j <= hi; ++j) {
          const long long tr0 = p.trace ? clock64() : 0;
          mbar_wait(s_full(h), s_phase, 30 + h);
          s_phase ^= 1;
          tc_fence_after();
          const long long tr1 = p.trace ? clock64() : 0;
          uint32_t s[128];
          tmem_ld_32x32b_x32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
          tmem_ld_32x32b_x32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
          tmem_ld_32x32b_x32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
          tmem_ld_32x32b_x32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
          tmem_ld_wait();
          const long long tr2 = p.trace ? clock64() : 0;
          const int k0 = j * BKV;
          if (!p.scale_pos) {
            // non-positive scale: move to the log2 domain first (max must see scaled values)
#pragma unroll
            for (int c = 0; c < 128; ++c) s[c] = __float_as_uint(__uint_as_float(s[c]) * p.scale_log2);
          }
          // tile needs masking if any (row, key) pair of the whole Q tile is invalid
          const bool need_mask = (k0 + BKV - 1 > rt) || (k0 < rt + BQ - p.window) ||
                                 (k0 + BKV > p.seq);
          if (need_mask) {
            // valid keys of this row form one contiguous column range [c_lo, c_hi]
            const int c_lo = row - p.window + 1 - k0;
            const int c_hi = min(row, p.seq - 1) - k0;
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (c < c_lo || c > c_hi) s[c] = 0xff800000u;  // -inf
          }
          // row max: four independent 3-input max chains
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 128; c += 8) {
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
          const float nm = (m_used == -INFINITY) ? 0.f : -m_used;
          const uint64_t sl2 = f2_pack(sl, sl), nm2 = f2_pack(nm, nm);
          uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
          for (int g = 0; g < 8; ++g) {  // 16 keys per group -> 8 packed P columns
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int c = g * 16 + 2 * e;
              // x = s * scale*log2e - m, two lanes per FFMA2
              const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sl2, nm2);
              const uint64_t p2 = (e < EMU) ? ex2_poly2(x2) : ex2_mufu2(x2);
              acc[e & 3] = f2_add(acc[e & 3], p2);
              pk[e] = pack_bf16_2(p2);
            }
            // P_h(j) -> TMEM (aliases S_h columns [0, 64)); S is already in registers
            tmem_st_32x32b_x8(t_s + g * 8, pk);
          }
          {
            float a0, a1, b0, b1, c0, c1, d0, d1;
            f2_unpack(f2_add(acc[0], acc[1]), a0, a1);
            f2_unpack(f2_add(acc[2], acc[3]), b0, b1);
            (void)c0; (void)c1; (void)d0; (void)d1;
            l += (a0 + a1) + (b0 + b1);
          }
          // correction: O_h (complete through PV_h(j-1)) *= corr for rows whose max moved
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
          const long long tr3 = p.trace ? clock64() : 0;
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full(h));
          if (p.trace) {
            tr_acc[0] += tr1 - tr0;  // waiting for S
            tr_acc[1] += tr2 - tr1;  // TMEM load of S
            tr_acc[2] += tr3 - tr2;  // max / exp2 / P store issue (+ rare O rescale)
            tr_acc[3] += clock64() - tr3;  // st wait + arrive
            tr_acc[4] += 1;
          }
        }
      }
      // ---------------- epilogue: O / l, lse ----------------
      // (always arrive q_empty so the producer's phase accounting stays aligned)
      if (tile_live) {
        mbar_wait(o_full(h), o_phase, 40 + h);
        tc_fence_after();
      }
      o_phase ^= tile_live ? 1 : 0;
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      if (tile_live && p.lse != nullptr && row < p.seq)
        p.lse[(size_t)bh * p.seq + row] = (m_used + __log2f(l)) * (1.0f / LOG2E);
      const uint32_t qbuf = sbase + SMEM_Q + h * TILE_BYTES;
      if (tile_live) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          // rows of this warp: 32 x 128 B in panel `half`; SWIZZLE_128B chunk c at c ^ (r & 7)
          const uint32_t wbuf = qbuf + half * HALF_BYTES + q * 32 * 128;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + half * 64 + c2 * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t chunk = (uint32_t)(c2 * 4 + c) ^ (lane & 7);
              st_shared_v4(wbuf + lane * 128 + chunk * 16,
                           pack_bf16(__uint_as_float(o[8 * c + 0]) * inv_l, __uint_as_float(o[8 * c + 1]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * c + 2]) * inv_l, __uint_as_float(o[8 * c + 3]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * c + 4]) * inv_l, __uint_as_float(o[8 * c + 5]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * c + 6]) * inv_l, __uint_as_float(o[8 * c + 7]) * inv_l));
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmO, wbuf, half * 64, rt + q * 32, bh);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      if (lane == 0) {
        bulk_wait_read<0>();
        mbar_arrive(q_empty(h));
      }
      __syncwarp();
    }
    if (p.trace && lane == 0)
      for (int e = 0; e < 8; ++e) p.trace[((size_t)blockIdx.x * 12 + warp) * 8 + e] = tr_acc[e];
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace

cudaError_t attention_fwd_launch(const AttnArgs &a, cudaStream_t stream) {
  const uint64_t bh = (uint64_t)a.batch * a.heads;
  CUtensorMap tQ = make_tmap_3d(a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tK = make_tmap_3d(a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tV = make_tmap_3d(a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tO = make_tmap_3d(a.o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                (uint64_t)a.seq * D, 64, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  Params p;
  p.bh = (int)bh;
  p.seq = (int)a.seq;
  p.window = (int)(a.window < a.seq ? a.window : a.seq);
  p.nqb = (int)((a.seq + 2 * BQ - 1) / (2 * BQ));
  p.scale_log2 = (float)(a.scale * 1.4426950408889634);
  p.lse = a.lse;
  p.trace = a.trace;
  const int items = p.bh * p.nqb;
  int grid = sm_count();
  if (a.max_ctas > 0 && a.max_ctas < grid) grid = a.max_ctas;
  if (grid > items) grid = items;
  p.scale_pos = a.scale > 0 ? 1 : 0;
  auto launch = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    kern<<<grid, NUM_THREADS, SMEM_TOTAL, stream>>>(tQ, tK, tV, tO, p);
    return cudaGetLastError();
  };
  switch (a.emu < 0 ? kDefaultEmu : a.emu) {
    case 0: return launch(attention_fwd_kernel<0>);
    case 1: return launch(attention_fwd_kernel<1>);
    case 2: return launch(attention_fwd_kernel<2>);
    case 3: return launch(attention_fwd_kernel<3>);
    default: return launch(attention_fwd_kernel<4>);
  }
}

}  // namespace mimw
