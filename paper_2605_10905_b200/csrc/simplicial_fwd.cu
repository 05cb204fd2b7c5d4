// 2-simplicial (trilinear) attention forward for sm_100a:
//
//   s(i, j1, j2) = scale * sum_x q[i,x] k1[j1,x] k2[j2,x]
//   o[i,x]       = sum_{j1,j2} softmax_{(j1,j2)}(s) v1[j1,x] v2[j2,x]
//   lse[i]       = log sum exp s
//   j1 in [max(0, i-w1+1), i],  j2 in [max(0, i-w2+1), i]
//
// i.e. oracle_simplicial_attention (proj/core/src/oracles.cpp:82-117), the
// computation of proj/kernels/simplicial_attention.mimw:1-95.  The tensor-core
// form the paper describes (form Q (.) K1 elementwise, GEMM
// against K2, online softmax, P.V2 GEMM, apply V1 after) maps to B200 as a
// loop over the K1 offset d = i - j1 (0 <= d < w1), each d a windowed
// flash-attention sweep over K2/V2 tiles:
//   Q'_d[i]  = q[i] (.) k1[i - d]             (softmax warps -> smem, SW128)
//   S        = Q'_d K2_t^T                    (tcgen05.mma SS -> TMEM)
//   U_d     += P V2_t                          (tcgen05.mma TS, P in TMEM)
//   O[i]    += v1[i - d] (.) U_d[i]           (softmax warps, TMEM -> TMEM)
// with ONE running max / sum per row across all (d, j2), so O and U are
// rescaled together (only when the max grows by > 8 in log2 units).
//
// MIMW roles (one CTA = 128 query rows of one (batch, head), 12 warps):
//   warp 0     TMA producer of the K2/V2 tile ring (repeated for every d)
//   warp 1     TMEM allocator + single-thread MMA issuer, running two S tiles
//              ahead: S(n+2) is issued right after PV(n) (tcgen05.mma ops of
//              one thread execute in order, so it may overwrite P_n)
//   warps 2-9  two softmax warpgroups, each one row/thread over half the
//              keys of the step (and half the head dim of U / O); row max
//              exchanged through smem: softmax, U -> O fold, epilogue
//   warps 10-11 operand prep (2 rows/thread): Q'_{d+1} = q (.) k1[i-d-1] into
//              the Q' double buffer and the v1[i-d] rows of the fold into smem,
//              off the softmax warps' critical path (their global-load latency
//              was ~25% of the kernel, measured)
// TMEM: S double buffer [0,128) [128,256) f32 (P_n bf16 written over the first
// 64 columns of its own S buffer once read), U [256,384) f32, O [384,512) f32.
// The softmax warps wait on a PV only to rescale (the running max grew) or to
// fold U_d into O; otherwise the tensor pipe always holds the next S.
#include "simplicial_fwd.h"
#include "ptx.cuh"
#include "softmax.cuh"
#include "tma_host.h"

#include <algorithm>
#include <cstdlib>

namespace mimw {

namespace {

constexpr int D = 128;
constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int NSLOT = 4;
constexpr int TILE_BYTES = BKV * D * 2;     // 32 KiB
constexpr int HALF_BYTES = TILE_BYTES / 2;  // one 64-column swizzle panel
constexpr int NUM_THREADS = 384;
constexpr int SMEM_QP = 0;                               // 2 Q' buffers
constexpr int SMEM_KV = 2 * TILE_BYTES;                  // K2/V2 ring
constexpr int SMEM_V1 = SMEM_KV + NSLOT * TILE_BYTES;     // v1[i - d] rows of the fold
constexpr int SMEM_BAR = SMEM_V1 + TILE_BYTES;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024 + 1024;  // barriers, max/sum exchange, align
static_assert(SMEM_TOTAL <= 232448, "smem");
constexpr uint32_t IDESC_S = idesc_bf16(BQ, BKV, 0, 0);
constexpr uint32_t IDESC_PV = idesc_bf16(BQ, D, 0, 1);
constexpr uint32_t TM_S = 0, TM_U = 256, TM_O = 384;  // S buffer b at TM_S + 128 b
constexpr float LOG2E = 1.4426950408889634f;

struct Params {
  const __nv_bfloat16 *q, *k1, *v1;  // [bh, seq, 128]
  __nv_bfloat16 *o;
  float *lse;
  int seq, w1, w2, nqt;
  float scale_log2;
  int scale_pos;     // scale > 0: max on raw scores, scale folded into the FFMA2
};

// K2/V2 tile range [lo, hi] needed by query rows [i0, i0+127]
__device__ __forceinline__ void kv2_range(int i0, const Params &p, int &lo, int &hi) {
  lo = max(0, i0 - p.w2 + 1) / BKV;
  hi = min(i0 + BQ - 1, p.seq - 1) / BKV;
}

#ifdef MIMW_SIMP_TRACE
// per-warp cycle accounting of the first 4 CTAs (tools/simp_trace.py):
// [cta][warp][8] = role-specific wait buckets, [7] = total
__device__ unsigned long long g_simp_trace[4 * 12 * 8];
#define TR_DECL unsigned long long tr_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; const long long tr_t0 = clock64();
#define TR(i, stmt) do { const long long t_ = clock64(); stmt; tr_[i] += clock64() - t_; } while (0)
#define TR_END \
  if (blockIdx.x < 4 && lane == 0) { tr_[7] = clock64() - tr_t0; \
    for (int e_ = 0; e_ < 8; ++e_) g_simp_trace[(blockIdx.x * 12 + warp) * 8 + e_] = tr_[e_]; }
#else
#define TR_DECL
#define TR(i, stmt) stmt
#define TR_END
#endif

template <int EMU>  // exponentials per 8 computed by the FMA-pipe polynomial instead of MUFU
__global__ void __launch_bounds__(NUM_THREADS, 1)
simplicial_fwd_kernel(const __grid_constant__ CUtensorMap tmK2, const __grid_constant__ CUtensorMap tmV2,
                      Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + SMEM_BAR;
  auto qp_full = [&](int b) { return bars + 8 * b; };
  auto qp_empty = [&](int b) { return bars + 16 + 8 * b; };
  auto s_full = [&](int b) { return bars + 32 + 8 * b; };
  // Step n uses p_full(n & 1) / u_done(n & 1): the softmax warps run up to
  // two steps ahead of the MMA warp's P waits and wait on a PV up to two steps
  // late, which a single parity-tracked barrier could not disambiguate.
  auto p_full = [&](int b) { return bars + 48 + 8 * b; };
  auto u_done = [&](int b) { return bars + 64 + 8 * b; };
  auto kv_full = [&](int s) { return bars + 80 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 80 + 8 * NSLOT + 8 * s; };
  // v1 row buffer handoff prep warps <-> softmax warps: named barriers 9 (full)
  // and 10 (empty) over the 2 + 8 warps (producer/consumer bar.arrive / bar.sync)
  constexpr uint32_t V1_FULL = 9, V1_EMPTY = 10, V1_THREADS = 320;
  const uint32_t tmem_slot = bars + 80 + 16 * NSLOT + 16;
  volatile uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem + SMEM_BAR + 96 + 16 * NSLOT);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const int bh = blockIdx.x / p.nqt;
  const int qt = p.nqt - 1 - (int)(blockIdx.x % p.nqt);  // heavier (later) tiles first
  const int i0 = qt * BQ;
  int lo, hi;
  kv2_range(i0, p, lo, hi);
  const int ntile = hi - lo + 1;
  const int nd = min(p.w1, i0 + BQ);  // K1 offsets d with at least one valid row
  const int nsteps = nd * ntile;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK2);
    tma_prefetch_desc(&tmV2);
    for (int b = 0; b < 2; ++b) {
      mbar_init(qp_full(b), 2);  // the two prep warps
      mbar_init(qp_empty(b), 1);
    }
    mbar_init(s_full(0), 1);
    mbar_init(s_full(1), 1);
    mbar_init(p_full(0), 8);
    mbar_init(p_full(1), 8);
    mbar_init(u_done(0), 1);
    mbar_init(u_done(1), 1);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  TR_DECL

  if (warp == 0) {
    // ================= TMA producer: K2_t, V2_t for every (d, t) =================
    // Ring positions follow the MMA warp's consumption order
    //   K(0) K(1) | V(0) K(2) | V(1) K(3) | ... (S runs two steps ahead of PV),
    // so a K tile never queues behind a V slot that waits on a PV.
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      auto load = [&](bool is_k, int n) {
        const int t = lo + n % ntile;
        TR(0, mbar_wait(kv_empty(slot), ph ^ 1, 70));
        mbar_arrive_expect_tx(kv_full(slot), TILE_BYTES);
        const uint32_t dst = sbase + SMEM_KV + slot * TILE_BYTES;
        const CUtensorMap *tm = is_k ? &tmK2 : &tmV2;
        tma_load_3d(dst, tm, kv_full(slot), 0, t * BKV, bh);
        tma_load_3d(dst + HALF_BYTES, tm, kv_full(slot), 64, t * BKV, bh);
        if (++slot == NSLOT) { slot = 0; ph ^= 1; }
      };
      if (nsteps > 0) load(true, 0);
      if (nsteps > 1) load(true, 1);
#pragma unroll 1
      for (int n = 0; n < nsteps; ++n) {
        load(false, n);
        if (n + 2 < nsteps) load(true, n + 2);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    constexpr uint32_t HI_KMAJ = (1024u >> 4) | (1u << 14) | (2u << 29);
    constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;
    constexpr uint32_t LO_VMN = ((uint32_t)HALF_BYTES >> 4) << 16;
    int rpos = 0;  // ring position: the MMA consumes in the producer's order
    auto ring_next = [&]() {
      const int pos = rpos++;
      TR(1, mbar_wait(kv_full(pos % NSLOT), (pos / NSLOT) & 1, 71));
      return pos % NSLOT;
    };
    auto issue_S = [&](int n) {  // S of step n = (d, t) into buffer n & 1
      const int d = n / ntile;
      const int t = n % ntile;
      if (t == 0) TR(2, mbar_wait(qp_full(d & 1), (d >> 1) & 1, 72));
      const int kslot = ring_next();
      tc_fence_after();
      const uint32_t qa = (sbase + SMEM_QP + (d & 1) * TILE_BYTES) >> 4;
      const uint32_t kb = (sbase + SMEM_KV + kslot * TILE_BYTES) >> 4;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k >> 2) * HALF_BYTES + (k & 3) * 32) >> 4;
          mma_f16_ss<1>(tmem + TM_S + 128 * (n & 1), make_desc(LO_KMAJ | (qa + off), HI_KMAJ),
                        make_desc(LO_KMAJ | (kb + off), HI_KMAJ), IDESC_S, k != 0);
        }
        mma_commit(s_full(n & 1));
        mma_commit(kv_empty(kslot));
        if (t == ntile - 1) mma_commit(qp_empty(d & 1));  // last read of Q'_d
      }
      __syncwarp();
    };
    auto issue_PV = [&](int n) {
      const int t = n % ntile;
      const int vslot = ring_next();
      TR(3, mbar_wait(p_full(n & 1), (uint32_t)((n >> 1) & 1), 74));
      tc_fence_after();
      const uint32_t vb = (sbase + SMEM_KV + vslot * TILE_BYTES) >> 4;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          mma_f16_ts<1>(tmem + TM_U, tmem + TM_S + 128 * (n & 1) + 64 * (k >> 2) + 8 * (k & 3),
                        make_desc(LO_VMN | (vb + k * (2048 >> 4)), HI_KMAJ), IDESC_PV,
                        (t != 0 || k != 0) ? 1u : 0u);
        mma_commit(u_done(n & 1));
        mma_commit(kv_empty(vslot));
      }
      __syncwarp();
    };
    if (nsteps > 0) issue_S(0);
    if (nsteps > 1) issue_S(1);
    for (int n = 0; n < nsteps; ++n) {
      issue_PV(n);
      if (n + 2 < nsteps) issue_S(n + 2);  // overwrites P_n: after PV(n) in issue order
    }
  } else if (warp >= 10) {
    // ================= operand prep: Q'_d and v1 rows (rows r, r + 32) =================
    const int pw0 = (warp - 10) * 64 + (int)lane;
    // ---- Q'_d = q (.) k1[i - d] into smem buffer d&1 (SW128 K-major) ----
    auto prep_qp = [&](int d) {
      if (d >= 2) TR(1, mbar_wait(qp_empty(d & 1), ((d >> 1) & 1) ^ 1, 75));
      const uint32_t buf = sbase + SMEM_QP + (d & 1) * TILE_BYTES;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
      const int row = pw0 + 32 * h;
      const int i = i0 + row;
      const bool row_live = i < p.seq;
      const uint4 *qv = reinterpret_cast<const uint4 *>(p.q + ((size_t)bh * p.seq + min(i, p.seq - 1)) * D);
      const int j1 = i - d;
      const bool ok = row_live && j1 >= 0;
      const uint4 *kv = reinterpret_cast<const uint4 *>(p.k1 + ((size_t)bh * p.seq + max(j1, 0)) * D);
      // all 32 loads of the row in flight at once (one L2 round trip per row)
      uint4 a[16], bk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        a[c] = ok ? __ldg(qv + c) : make_uint4(0, 0, 0, 0);
        bk[c] = ok ? __ldg(kv + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) {  // 16 chunks of 8 bf16
        uint4 w;
        const uint32_t *pa = &a[c].x, *pb = &bk[c].x;
        uint32_t *pw = &w.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(pa + e));
          const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(pb + e));
          pw[e] = pack_bf16(fa.x * fb.x, fa.y * fb.y);
        }
        const int panel = c >> 3, cc = c & 7;
        st_shared_v4(buf + panel * HALF_BYTES + (row >> 3) * 1024 + (row & 7) * 128 +
                         ((cc ^ (row & 7)) << 4),
                     w.x, w.y, w.z, w.w);
      }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(qp_full(d & 1));
    };
    // ---- v1[i - d] row for the fold of d: 16-B chunk c of row r at c ^ (r & 15) ----
    auto prep_v1 = [&](int d) {
      if (d >= 1) TR(2, named_bar_sync(V1_EMPTY, V1_THREADS));  // the fold of d - 1 has read the rows
      uint4 w[2][16];  // both rows' loads in flight at once
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + pw0 + 32 * h;
        const int j1 = i - d;
        const bool ok = i < p.seq && j1 >= 0;
        const uint4 *vv = reinterpret_cast<const uint4 *>(p.v1 + ((size_t)bh * p.seq + max(j1, 0)) * D);
#pragma unroll
        for (int c = 0; c < 16; ++c) w[h][c] = ok ? __ldg(vv + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = pw0 + 32 * h;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          st_shared_v4(sbase + SMEM_V1 + row * 256 + ((c ^ (row & 15)) << 4), w[h][c].x, w[h][c].y,
                       w[h][c].z, w[h][c].w);
      }
      __syncwarp();
      named_bar_arrive(V1_FULL, V1_THREADS);
    };
    if (nd > 0) prep_qp(0);
    for (int d = 0; d < nd; ++d) {
      if (d + 1 < nd) prep_qp(d + 1);
      prep_v1(d);
    }
  } else if (warp >= 2) {
    // ================= softmax / U->O fold / epilogue =================
    // Two warpgroups split each step's 128 keys (g = 0: keys 0-63, g = 1:
    // 64-127) and the head dim of U / O the same way; the row max is
    // exchanged through smem every step (one named barrier per lane quarter),
    // so both keep the same running max and rescale decisions.
    const int q = warp & 3;
    const int g = (warp - 2) >> 2;
    const int row = q * 32 + (int)lane;  // row of the tile == TMEM lane
    const int i = i0 + row;
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const bool row_live = i < p.seq;
    const uint32_t xbuf = sbase + SMEM_BAR + 256;  // [2 groups][128 rows] f32
    float m_used = -INFINITY, l = 0.f;
    auto wait_pv = [&](int k) {  // PV of step k complete
      TR(2, mbar_wait(u_done(k & 1), (uint32_t)((k >> 1) & 1), 77));
      tc_fence_after();
    };
    auto exchange = [&](float v) {  // the other group's value for this row
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(xbuf + (g * 128 + row) * 4), "f"(v) : "memory");
      TR(3, named_bar_sync(1 + q, 64));
      float o;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(xbuf + ((g ^ 1) * 128 + row) * 4) : "memory");
      TR(3, named_bar_sync(5 + q, 64));  // both read before either writes the next value
      return o;
    };
    bool o_live = false;  // O holds a folded U
    bool fold_pending = false;  // U holds the complete U_d of the previous d
    // ---- fold U_dd into O: O += v1[i - dd] (.) U_dd ----
    auto fold = [&](int dd) {
      TR(4, named_bar_sync(V1_FULL, V1_THREADS));
#pragma unroll 1
      for (int c = 64 * g; c < 64 * g + 64; c += 32) {
        uint32_t u[32], o[32];
        tmem_ld_32x32b_x32(tmem + t_lane + TM_U + c, u);
        if (o_live) tmem_ld_32x32b_x32(tmem + t_lane + TM_O + c, o);
        tmem_ld_wait();
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          uint4 w;
          const int ch = c / 8 + gg;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                       : "r"(sbase + SMEM_V1 + row * 256 + ((ch ^ (row & 15)) << 4)));
          const uint32_t *pw = &w.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(pw + e));
            const int x = gg * 8 + e * 2;
            const float b0 = o_live ? __uint_as_float(o[x]) : 0.f;
            const float b1 = o_live ? __uint_as_float(o[x + 1]) : 0.f;
            o[x] = __float_as_uint(b0 + f.x * __uint_as_float(u[x]));
            o[x + 1] = __float_as_uint(b1 + f.y * __uint_as_float(u[x + 1]));
          }
        }
        tmem_st_32x32b_x16(tmem + t_lane + TM_O + c, *reinterpret_cast<uint32_t(*)[16]>(&o[0]));
        tmem_st_32x32b_x16(tmem + t_lane + TM_O + c + 16, *reinterpret_cast<uint32_t(*)[16]>(&o[16]));
      }
      tmem_st_wait();
      __syncwarp();
      if (dd + 1 < nd) named_bar_arrive(V1_EMPTY, V1_THREADS);  // v1 rows of dd read
      o_live = true;
    };
    const float sl = p.scale_pos ? p.scale_log2 : 1.f;
    const uint64_t sl2 = f2_pack(sl, sl);
    for (int n = 0, d = 0, t = 0; n < nsteps; ++n, t = (t + 1 == ntile) ? 0 : t + 1, d += (t == 0)) {
      const int j1 = i - d;
      const int b = n & 1;
      // ---- S of step n (this group's 64 keys) ----
      TR(1, mbar_wait(s_full(b), (uint32_t)((n >> 1) & 1), 76));
      tc_fence_after();
      uint32_t s[64];
      const uint32_t t_s = tmem + t_lane + TM_S + 128 * b + 64 * g;
      tmem_ld_32x32b_x32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
      tmem_ld_32x32b_x32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
      tmem_ld_wait();
      // mask: j2 in [i - w2 + 1, i] and < seq, valid query row, valid K1 row.
      // Uniform fast path: the tile is inside every row's window.
      const int k0 = (lo + t) * BKV + 64 * g;
      const bool need_mask = ((lo + t) * BKV + BKV - 1 > i0) || ((lo + t) * BKV < i0 + BQ - p.w2) ||
                             ((lo + t) * BKV + BKV > p.seq) || (i0 + BQ > p.seq) || (i0 < d) || !p.scale_pos;
      const bool live = row_live && j1 >= 0;
      if (need_mask) {
        // valid columns [c_lo, c_hi] of this group's 64 as a bit mask: one
        // bit test + select per element instead of two compares + select
        const int c_lo = max(i - p.w2 + 1 - k0, 0);
        const int c_hi = min(min(i, p.seq - 1) - k0, 63);
        uint64_t bits = 0;
        if (live && c_lo <= c_hi) bits = (~0ull >> (63 - c_hi)) & (~0ull << c_lo);
        const uint32_t b_lo = (uint32_t)bits, b_hi = (uint32_t)(bits >> 32);
        if (!p.scale_pos) {  // uniform: scale not folded into the exponent FFMA
#pragma unroll
          for (int c = 0; c < 64; ++c) s[c] = __float_as_uint(__uint_as_float(s[c]) * p.scale_log2);
        }
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          float v = __uint_as_float(s[c]);
          const uint32_t w = c < 32 ? b_lo : b_hi;
          if (!(w & (1u << (c & 31)))) v = -INFINITY;
          s[c] = __float_as_uint(v);
        }
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 64; c += 8) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          m4[e] = fmax3(m4[e], __uint_as_float(s[c + 2 * e]), __uint_as_float(s[c + 2 * e + 1]));
      }
      float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * sl;
      mx = fmaxf(mx, exchange(mx));
      float corr = 1.f;
      bool rescale = false;
      if (mx > m_used + 8.f || (m_used == -INFINITY && mx > -INFINITY)) {
        corr = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
        rescale = m_used != -INFINITY;
        m_used = mx;
      }
      l *= corr;
      const float nm = (m_used == -INFINITY) ? 0.f : -m_used;
      const uint64_t nm2 = f2_pack(nm, nm);
      uint64_t acc2[4] = {0, 0, 0, 0};
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), sl2, nm2);
        const uint64_t p2 = ((e & 7) < EMU) ? ex2_poly2(x2) : ex2_mufu2(x2);
        acc2[e & 3] = f2_add(acc2[e & 3], p2);
        pk[e] = pack_bf16_2(p2);
      }
      {
        float a0, a1, b0, b1;
        f2_unpack(f2_add(acc2[0], acc2[1]), a0, a1);
        f2_unpack(f2_add(acc2[2], acc2[3]), b0, b1);
        l += (a0 + a1) + (b0 + b1);
      }
      // P_n overwrites S buffer b, last read as P_{n-2} by PV(n-2)
      if (n >= 2) wait_pv(n - 2);
      if (__any_sync(0xffffffffu, rescale)) {
        // U (this d's partial sum, or the previous d's complete U_{d-1} still
        // waiting for its fold) and O carry the old max
        if (n >= 1) wait_pv(n - 1);
#pragma unroll 1
        for (int c = 64 * g; c < 64 * g + 64; c += 32) {
          uint32_t o[32];
          if (t > 0 || fold_pending) {
            tmem_ld_32x32b_x32(tmem + t_lane + TM_U + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x16(tmem + t_lane + TM_U + c, *reinterpret_cast<uint32_t(*)[16]>(&o[0]));
            tmem_st_32x32b_x16(tmem + t_lane + TM_U + c + 16, *reinterpret_cast<uint32_t(*)[16]>(&o[16]));
          }
          if (o_live) {
            tmem_ld_32x32b_x32(tmem + t_lane + TM_O + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x16(tmem + t_lane + TM_O + c, *reinterpret_cast<uint32_t(*)[16]>(&o[0]));
            tmem_st_32x32b_x16(tmem + t_lane + TM_O + c + 16, *reinterpret_cast<uint32_t(*)[16]>(&o[16]));
          }
        }
      }
      tmem_st_32x32b_x16(t_s, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
      tmem_st_32x32b_x16(t_s + 16, *reinterpret_cast<uint32_t(*)[16]>(&pk[16]));
      if (fold_pending) {
        // U_{d-1} is complete once PV(n-1) is; folded now, a step late, so
        // the wait overlaps this step's softmax.  P_n is published after it:
        // PV(n) (t == 0) overwrites U.
        wait_pv(n - 1);
        fold(d - 1);
        fold_pending = false;
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full(b));
      if (t == ntile - 1) fold_pending = true;
    }
    if (fold_pending) {
      wait_pv(nsteps - 1);
      fold(nd - 1);
    }
    // ---------------- epilogue: O / l, lse ----------------
    l += exchange(l);  // both groups' partial sums
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    if (g == 0 && row_live && p.lse != nullptr)
      p.lse[(size_t)bh * p.seq + i] = (m_used + __log2f(l)) * (1.0f / LOG2E);
    uint4 *orow = reinterpret_cast<uint4 *>(p.o + ((size_t)bh * p.seq + min(i, p.seq - 1)) * D);
#pragma unroll 1
    for (int c = 64 * g; c < 64 * g + 64; c += 32) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tmem + t_lane + TM_O + c, o);
      tmem_ld_wait();
      if (row_live) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l);
          orow[c / 8 + v] = w;
        }
      }
    }
  }

  TR_END
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace

cudaError_t simplicial_fwd_launch(const SimplicialArgs &a, cudaStream_t stream) {
  const uint64_t bh = (uint64_t)a.bh;
  if (bh == 0 || a.seq == 0) return cudaSuccess;
  CUtensorMap tK2 = make_tmap_3d(a.k2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                 (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tV2 = make_tmap_3d(a.v2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, a.seq, bh, D,
                                 (uint64_t)a.seq * D, 64, BKV, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  Params p;
  p.q = static_cast<const __nv_bfloat16 *>(a.q);
  p.k1 = static_cast<const __nv_bfloat16 *>(a.k1);
  p.v1 = static_cast<const __nv_bfloat16 *>(a.v1);
  p.o = static_cast<__nv_bfloat16 *>(a.o);
  p.lse = a.lse;
  p.seq = (int)a.seq;
  p.w1 = (int)std::min<int64_t>(a.w1, a.seq);
  p.w2 = (int)std::min<int64_t>(a.w2, a.seq);
  p.nqt = (int)((a.seq + BQ - 1) / BQ);
  p.scale_log2 = (float)(a.scale * 1.4426950408889634);
  p.scale_pos = a.scale > 0 ? 1 : 0;
  static const int emu_env = getenv("MIMW_SIMP_EMU") ? atoi(getenv("MIMW_SIMP_EMU")) : 1;  // A/B knob (1: 661, 2: 659, 3: 648 TF measured)
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(bh * p.nqt), NUM_THREADS, SMEM_TOTAL, stream>>>(tK2, tV2, p);
    return cudaGetLastError();
  };
  switch (emu_env) {
    case 1: return go(simplicial_fwd_kernel<1>);
    case 2: return go(simplicial_fwd_kernel<2>);
    case 3: return go(simplicial_fwd_kernel<3>);
    case 4: return go(simplicial_fwd_kernel<4>);
    default: return go(simplicial_fwd_kernel<0>);
  }
}

}  // namespace mimw

// Debug hook (not in the public header): the per-warp cycle buckets of the
// first 4 CTAs when built with -DMIMW_SIMP_TRACE (tools/simp_trace.py).
extern "C" int mimw_b200_debug_simplicial_trace(unsigned long long *host, int n) {
#ifdef MIMW_SIMP_TRACE
  if (n > 4 * 12 * 8) n = 4 * 12 * 8;
  return cudaMemcpyFromSymbol(host, mimw::g_simp_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 3;
#else
  (void)host;
  (void)n;
  return 2;
#endif
}
