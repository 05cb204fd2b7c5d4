// 2-CTA flash-attention forward (included by attention_fwd.cu inside its
// anonymous namespace; same Params / kv_range / work_item).
//
// Why a second design: in the one-CTA kernel two Q tiles share ONE S buffer
// in TMEM (S 128 + P 2x64 + O 2x128 columns = 512), so S_0(j) -> softmax-0
// load -> S_1(j) -> softmax-1 load -> S_0(j+1) is a serial chain of two
// (S-MMA latency + 64 KiB TMEM load) per KV step: ~3130 cycles against 2048 of
// tensor work (profiles/r02/fa_shared_s_events.txt).
//
// Here a CTA pair (cluster of 2) runs tcgen05.mma.cta_group::2 with M = 256:
// CTA rank r owns ONE 128-row Q tile (rows r0 + 128 r ..), so its TMEM holds
//   S_0 [0,128)  S_1 [128,256)  P_0 [256,320)  P_1 [320,384)  O [384,512)
// - S is double-buffered: S(j+1) is issued while the softmax still works on
//   S(j); P is double-buffered, so the softmax of step j only waits for
//   PV(j-2) (and for PV(j-1) only in the rare steps that rescale O).
// - The pair shares every K/V tile: CTA r stages keys [64 r, 64 r + 64) of K
//   and d-columns [64 r, 64 r + 64) of V (half the TMA bytes and half the
//   B-operand smem reads per SM of the one-CTA kernel).
// - Two softmax warpgroups per CTA take alternate KV steps (warpgroup w the
//   steps of parity w, i.e. S_w / P_w), so one warpgroup's TMEM loads and P
//   stores overlap the other's exponentials; the running max is handed from
//   step to step through smem, the row sums are combined at the epilogue.
// - Q is double-buffered in smem, so the next item's Q load overlaps the
//   current item; the epilogue reads O into registers, hands it back, then
//   stores, so the next item's first P.V waits only for that read.
// Roles: warps 0-7 softmax/correction/epilogue, warp 8 TMA producer (both
// CTAs), warp 9 S = Q K^T issuer + TMEM allocator, warp 10 O += P V issuer
// (leader CTA only; tcgen05.mma issue blocks at the pipe rate, so each
// dependency chain gets its own issuer), warp 11 idle.  Work items (one
// 256-row Q block of one head per pair) come from cluster launch control in
// the band / longest-first order of work_item().

constexpr int C2_THREADS = 384;
constexpr int C2_NSLOT = 7;                   // K/V ring slots of 16 KiB (half a tile per CTA)
constexpr int C2_SLOT_BYTES = 64 * D * 2;     // 16 KiB: 64 keys x 128 d (K) or 128 keys x 64 d (V)
constexpr int C2_SMEM_Q = 0;                  // 2 x 32 KiB Q tiles
constexpr int C2_SMEM_KV = 2 * TILE_BYTES;
constexpr int C2_SMEM_O = C2_SMEM_KV + C2_NSLOT * C2_SLOT_BYTES;   // 8 warps x 4 KiB O staging
constexpr int C2_SMEM_RED = C2_SMEM_O + 8 * 4096;                  // per-step max hand-off [2 wg][128] f32
constexpr int C2_SMEM_LRED = C2_SMEM_RED + 2 * 128 * 4;            // epilogue (l, m) exchange [2 wg][2][128] f32
constexpr int C2_SMEM_BAR = C2_SMEM_LRED + 2 * 2 * 128 * 4;
constexpr int C2_BAR_BYTES = 512;
constexpr int C2_SMEM_TOTAL = C2_SMEM_BAR + C2_BAR_BYTES + 1024;
static_assert(C2_SMEM_TOTAL <= 232448, "2-CTA FA smem");
constexpr uint32_t C2_IDESC_S = idesc_bf16(256, BKV, 0, 0);   // Q (K-major) x K (K-major)
constexpr uint32_t C2_IDESC_PV = idesc_bf16(256, D, 0, 1);    // P (TMEM) x V (MN-major)
constexpr uint32_t C2_TM_S = 0, C2_TM_P = 256, C2_TM_O = 384;

template <int EMU>
__global__ void __launch_bounds__(C2_THREADS, 1)
attention_fwd_cg2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + C2_SMEM_BAR;
  // leader-side barriers (arrivals from both CTAs / TMA of both CTAs)
  auto q_full = [&](int b) { return bars + 8 * b; };
  auto kv_full = [&](int s) { return bars + 16 + 8 * s; };
  auto s_free = [&](int b) { return bars + 80 + 8 * b; };
  auto p_full = [&](int b) { return bars + 96 + 8 * b; };
  const uint32_t o_free = bars + 112;
  // local barriers (completed by the leader's multicast commits)
  auto q_empty = [&](int b) { return bars + 120 + 8 * b; };
  auto kv_empty = [&](int s) { return bars + 136 + 8 * s; };
  auto s_full = [&](int b) { return bars + 200 + 8 * b; };
  auto pv_done = [&](int b) { return bars + 216 + 8 * b; };
  // cluster launch control response ring
  constexpr int CLC_SLOTS = 4;
  constexpr uint32_t CLC_CONSUMERS = 2 * (1 + 8) + 2;
  auto clc_resp = [&](int s) { return bars + 256 + 16 * s; };
  auto clc_full = [&](int s) { return bars + 320 + 8 * s; };
  auto clc_empty = [&](int s) { return bars + 352 + 8 * s; };
  const uint32_t tmem_slot = bars + 384;
  const uint32_t *tmem_slot_ptr = reinterpret_cast<const uint32_t *>(smem + C2_SMEM_BAR + 384);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int num_items = (int)nclusters_x();  // one cluster per work item (CLC cancels the rest)
#ifdef MIMW_FA_EVENTS
  // event log of cluster 0 (tools/fa2_events.py), kept in smem during the run
  // (global stores would be waited for by every release.cluster arrive) and
  // copied to p.trace[rank][warp][1024] at the end: (clock64 << 8 | code)
  constexpr int EV_CAP = 128;
  int ev_n = 0;
  unsigned long long *ev_mine = reinterpret_cast<unsigned long long *>(smem_raw + C2_SMEM_TOTAL) +
                                (size_t)warp * EV_CAP;
#define EV2(code)                                                                      \
  do {                                                                                 \
    if (blockIdx.x < 2 && lane == 0 && ev_n < EV_CAP && p.trace)                       \
      ev_mine[ev_n++] = ((unsigned long long)clock64() << 8) | (code);                 \
  } while (0)
#else
#define EV2(code) do {} while (0)
#endif

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    for (int b = 0; b < 2; ++b) {
      mbar_init(q_full(b), 1);
      mbar_init(s_free(b), 8);   // the 4 warps of warpgroup b, both CTAs
      mbar_init(p_full(b), 8);
      mbar_init(q_empty(b), 1);
      mbar_init(s_full(b), 1);
      mbar_init(pv_done(b), 1);
    }
    mbar_init(o_free, 16);
    for (int s = 0; s < C2_NSLOT; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    for (int s = 0; s < CLC_SLOTS; ++s) {
      mbar_init(clc_full(s), 1);
      mbar_init(clc_empty(s), CLC_CONSUMERS);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<2>(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  // u-th response of the CLC ring: the next item (or num_items when done)
  auto next_item = [&](int u, bool arrive) -> int {
    const int slot = u % CLC_SLOTS;
    mbar_wait(clc_full(slot), (uint32_t)(u / CLC_SLOTS) & 1, 12);
    const int x = clc_query(clc_resp(slot));
    if (arrive) mbar_arrive_cluster(map_to_rank(clc_empty(slot), 0));
    return x < 0 ? num_items : x / 2;
  };
  auto pair_range = [&](int qb, int &lo, int &hi) {
    const int r0 = qb * 2 * BQ;
    int lo0, hi0, lo1, hi1;
    kv_range(r0, p, lo0, hi0);
    kv_range(r0 + BQ < p.seq ? r0 + BQ : r0, p, lo1, hi1);
    lo = min(lo0, lo1);
    hi = max(hi0, hi1);
  };

  if (warp >= 8) {
  // control warpgroup gives registers to the two softmax warpgroups
  // (4 x (168 - 88) >= 8 x (208 - 168))
  asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
  if (warp == 8) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      const uint32_t lead_bars = map_to_rank(bars, 0);  // the leader's barrier block
      uint32_t pos = 0;                                  // ring position (2 per KV step)
      int n = 0;
      for (int it = (int)cluster_id_x(); it < num_items; it = next_item(n++, true)) {
        if (leader) {  // ask for the item after this one (response multicast to both CTAs)
          const int slot = n % CLC_SLOTS;
          mbar_wait_cluster(clc_empty(slot), ((uint32_t)(n / CLC_SLOTS) & 1) ^ 1, 13);
          mbar_arrive_expect_tx(clc_full(slot), 16);
          clc_try_cancel_multicast(clc_resp(slot), clc_full(slot));
        } else {
          mbar_arrive_expect_tx(clc_full(n % CLC_SLOTS), 16);
        }
        int bh, qb;
        work_item(it, p, bh, qb);
        int lo, hi;
        pair_range(qb, lo, hi);
        const int qbuf = n & 1;
        mbar_wait(q_empty(qbuf), ((n >> 1) & 1) ^ 1, 10);
        if (leader) mbar_arrive_expect_tx(q_full(qbuf), 2 * TILE_BYTES);
        const uint32_t dq = sbase + C2_SMEM_Q + qbuf * TILE_BYTES;
        const int qrow = qb * 2 * BQ + (int)rank * BQ;
        tma_load_3d_cg2(dq, &tmQ, lead_bars + 8 * qbuf, 0, qrow, bh);
        tma_load_3d_cg2(dq + HALF_BYTES, &tmQ, lead_bars + 8 * qbuf, 64, qrow, bh);
        for (int j = lo; j <= hi; ++j) {
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++pos) {
            const int slot = pos % C2_NSLOT;
            mbar_wait(kv_empty(slot), ((pos / C2_NSLOT) & 1) ^ 1, 11);
            EV2(30 + kv);
            if (leader) mbar_arrive_expect_tx(kv_full(slot), 2 * C2_SLOT_BYTES);
            const uint32_t dst = sbase + C2_SMEM_KV + slot * C2_SLOT_BYTES;
            const uint32_t fb = lead_bars + 16 + 8 * slot;
            if (kv == 0) {  // K: keys [j*128 + 64 r, +64), both 64-d panels
              tma_load_3d_cg2(dst, &tmK, fb, 0, j * BKV + (int)rank * 64, bh);
              tma_load_3d_cg2(dst + C2_SLOT_BYTES / 2, &tmK, fb, 64, j * BKV + (int)rank * 64, bh);
            } else {        // V: keys [j*128, +128), d-columns [64 r, +64)
              tma_load_3d_cg2(dst, &tmV, fb, (int)rank * 64, j * BKV, bh);
            }
          }
        }
      }
    }
  } else if (warp == 9 || warp == 10) {
    // ================= MMA issuers (leader CTA) =================
    if (leader) {
      const bool s_role = warp == 9;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t sb = __shfl_sync(0xffffffffu, sbase, 0);
      constexpr uint32_t HI_KMAJ = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, version, SW128
      constexpr uint32_t LO_KMAJ = (16u >> 4) << 16;
      uint32_t g = 0;    // KV steps issued so far (S / P buffer = g & 1)
      uint32_t pos = 0;  // ring position
      int n = 0;
      for (int it = (int)cluster_id_x(); it < num_items; it = next_item(n++, lane == 0)) {
        int bh, qb;
        work_item(it, p, bh, qb);
        int lo, hi;
        pair_range(qb, lo, hi);
        const int qbuf = n & 1;
        if (s_role) mbar_wait(q_full(qbuf), (n >> 1) & 1, 21);
        for (int j = lo; j <= hi; ++j, ++g, pos += 2) {
          const uint32_t b = g & 1;
          if (s_role) {
            const uint32_t kslot = pos % C2_NSLOT;
            mbar_wait(kv_full(kslot), (pos / C2_NSLOT) & 1, 23);
            EV2(1);
            mbar_wait(s_free(b), ((g >> 1) & 1) ^ 1, 24);
            EV2(2);
            tc_fence_after();
            const uint32_t qa = (sb + C2_SMEM_Q + qbuf * TILE_BYTES) >> 4;
            const uint32_t kb = (sb + C2_SMEM_KV + kslot * C2_SLOT_BYTES) >> 4;
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint32_t oa = ((k >> 2) * HALF_BYTES + (k & 3) * 32) >> 4;
                const uint32_t ob = ((k >> 2) * (C2_SLOT_BYTES / 2) + (k & 3) * 32) >> 4;
                mma_f16_ss<2>(tm + C2_TM_S + b * 128, make_desc(LO_KMAJ | (qa + oa), HI_KMAJ),
                              make_desc(LO_KMAJ | (kb + ob), HI_KMAJ), C2_IDESC_S, k != 0);
              }
              mma_commit_cg2_mc(s_full(b), 0x3);
              mma_commit_cg2_mc(kv_empty(kslot), 0x3);
              if (j == hi) mma_commit_cg2_mc(q_empty(qbuf), 0x3);
            }
            __syncwarp();
            EV2(3);
          } else {
            const uint32_t vslot = (pos + 1) % C2_NSLOT;
            mbar_wait(kv_full(vslot), ((pos + 1) / C2_NSLOT) & 1, 25);
            EV2(4);
            mbar_wait(p_full(b), (g >> 1) & 1, 26);
            if (j == lo) mbar_wait(o_free, (n & 1) ^ 1, 27);  // the previous item's O has been read
            EV2(5);
            tc_fence_after();
            const uint32_t vb = (sb + C2_SMEM_KV + vslot * C2_SLOT_BYTES) >> 4;
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < BKV / 16; ++k)
                mma_f16_ts<2>(tm + C2_TM_O, tm + C2_TM_P + b * 64 + k * 8,
                              make_desc(LO_KMAJ | (vb + k * (2048 >> 4)), HI_KMAJ), C2_IDESC_PV,
                              (j != lo || k != 0) ? 1u : 0u);
              mma_commit_cg2_mc(pv_done(b), 0x3);
              mma_commit_cg2_mc(kv_empty(vslot), 0x3);
            }
            __syncwarp();
            EV2(6);
          }
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    // ================= softmax / correction / epilogue =================
    // Warpgroup wg takes the KV steps of parity wg (global step counter g):
    // its S / P buffers are S_wg / P_wg, and while it works on step g the
    // other warpgroup works on g + 1, so their TMEM loads, exponentials and P
    // stores interleave on every SM sub-partition.  The running max is a
    // chain over steps: each step waits for the previous step's max (smem +
    // named barrier 1 + 4 wg' + q) and publishes its own.
    const int q = warp & 3;   // TMEM lane quarter (rows q*32 ..)
    const int wg = warp >> 2; // step parity handled by this warpgroup
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    const uint32_t lead_bars = map_to_rank(bars, 0);
    const uint32_t mpub_s = sbase + C2_SMEM_RED;                    // [2 wg][128 rows]: max published per step
    float *lred = reinterpret_cast<float *>(smem + C2_SMEM_LRED);  // [2 wg][128 rows]: (l, m) at the epilogue
    const int trow = q * 32 + (int)lane;
    const uint32_t bar_out = 1 + 4 * wg + q, bar_in = 1 + 4 * (wg ^ 1) + q;
    uint32_t g = 0;
    int n = 0;
    for (int it = (int)cluster_id_x(); it < num_items; it = next_item(n++, lane == 0)) {
      int bh, qb;
      work_item(it, p, bh, qb);
      int lo, hi;
      pair_range(qb, lo, hi);
      const int rt = qb * 2 * BQ + (int)rank * BQ;  // first row of this CTA's Q tile
      const int row = rt + trow;
      float m_seen = -INFINITY;  // reference max of this warpgroup's l
      int m_seen_j = -8;         // KV step that set m_seen (this item)
      float m_last = -INFINITY;  // max after the last step of this item seen by this warpgroup
      float l = 0.f;
      const uint32_t g_item = g;
      for (int j = lo; j <= hi; ++j, ++g) {
        if ((int)(g & 1) != wg) continue;
        const uint32_t b = g & 1;
        mbar_wait(s_full(b), (g >> 1) & 1, 30);
        EV2(10);
        tc_fence_after();
        uint32_t s[128];
        const uint32_t t_s = tmem + t_lane + C2_TM_S + b * 128;
        tmem_ld_32x32b_x32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld_32x32b_x32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld_32x32b_x32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
        tmem_ld_32x32b_x32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
        tmem_ld_wait();
        EV2(16);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(lead_bars + 80 + 8 * b);  // s_free(b) on the leader
        EV2(11);
        const int k0 = j * BKV;
        const bool need_mask = (p.causal && ((k0 + BKV - 1 > rt) || (k0 < rt + BQ - p.window))) ||
                               (k0 + BKV > p.seq) || !p.scale_pos;
        if (need_mask) {
          if (!p.scale_pos) {
#pragma unroll
            for (int e = 0; e < 128; ++e) s[e] = __float_as_uint(__uint_as_float(s[e]) * p.scale_log2);
          }
          const int c_lo = p.causal ? row - p.window + 1 - k0 : -k0;
          const int c_hi = (p.causal ? min(row, p.seq - 1) : p.seq - 1) - k0;
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e < c_lo || e > c_hi) s[e] = 0xff800000u;  // -inf
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int e = 0; e < 128; e += 8) {
#pragma unroll
          for (int f = 0; f < 4; ++f)
            m4[f] = fmax3(m4[f], __uint_as_float(s[e + 2 * f]), __uint_as_float(s[e + 2 * f + 1]));
        }
        const float sl = p.scale_pos ? p.scale_log2 : 1.f;
        const float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * sl;
        // Exponentials against a provisional reference: the max rule applied
        // to this warpgroup's own last reference (two steps back).  The true
        // reference needs the previous step's max from the other warpgroup;
        // it is taken after the exponentials, so that hand-off overlaps them,
        // and in the rare step where the two differ P and its sum are rescaled.
        const float m_base = (m_seen_j + 2 == j) ? m_seen : -INFINITY;
        const float m_p = (mx > m_base + 8.f || (m_base == -INFINITY && mx > -INFINITY)) ? mx : m_base;
        const float nm = (m_p == -INFINITY) ? 0.f : -m_p;
        const uint64_t sl2 = f2_pack(sl, sl), nm2 = f2_pack(nm, nm);
        uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), sl2, nm2);
          const uint64_t p2 = ((e & 7) < EMU) ? ex2_poly2(x2) : ex2_mufu2(x2);
          acc[e & 3] = f2_add(acc[e & 3], p2);
          float lo_, hi_;
          f2_unpack(p2, lo_, hi_);
          s[2 * e] = __float_as_uint(lo_);
          s[2 * e + 1] = __float_as_uint(hi_);
        }
        float l_p;
        {
          float a0, a1, b0, b1;
          f2_unpack(f2_add(acc[0], acc[1]), a0, a1);
          f2_unpack(f2_add(acc[2], acc[3]), b0, b1);
          l_p = (a0 + a1) + (b0 + b1);
        }
        EV2(18);
        // the previous step's max (the other warpgroup's), unless this is the item's first step
        float m_prev = -INFINITY;
        if (g > 0) {
          named_bar_sync(bar_in, 64);
          EV2(19);
          if (j != lo) m_prev = ld_shared_f32(mpub_s + (uint32_t)((wg ^ 1) * 128 + trow) * 4);
        }
        float m_used = m_prev;
        if (mx > m_prev + 8.f || (m_prev == -INFINITY && mx > -INFINITY)) m_used = mx;
        st_shared_f32(mpub_s + (uint32_t)(wg * 128 + trow) * 4, m_used);
        named_bar_arrive(bar_out, 64);
        EV2(12);
        if (__any_sync(0xffffffffu, m_used != m_p)) {
          const float f = (m_p == m_used) ? 1.f : ((m_used == -INFINITY) ? 0.f : ex2(m_p - m_used));
#pragma unroll
          for (int e = 0; e < 128; ++e) s[e] = __float_as_uint(__uint_as_float(s[e]) * f);
          l_p *= f;
        }
        if (m_used != m_seen) {
          l *= (m_seen == -INFINITY) ? 0.f : ex2(m_seen - m_used);
          m_seen = m_used;
        }
        m_seen_j = j;
        l += l_p;
        m_last = m_used;
        const bool rescale = (j != lo) && (m_used != m_prev);
        const float corr = (m_prev == -INFINITY) ? 0.f : ex2(m_prev - m_used);
        uint32_t *pk = s;  // P packed to bf16 in place over S
#pragma unroll
        for (int e = 0; e < 64; ++e) pk[e] = pack_bf16(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1]));
        EV2(13);
        // P_b was last read by PV(g - 2)
        if (g >= 2) mbar_wait(pv_done(b), ((g >> 1) & 1) ^ 1, 32);
        EV2(14);
        if (__any_sync(0xffffffffu, rescale)) {
          // O holds PV(.. g - 1) only once PV(g - 1) is done.  PV(g - 2) is
          // done (waited above), so pv_done(b ^ 1) has passed PV(g - 3) and
          // this parity wait cannot alias two phases back.
          mbar_wait(pv_done(b ^ 1), ((g - 1) >> 1) & 1, 33);
          tc_fence_after();
          const uint32_t t_o = tmem + t_lane + C2_TM_O;
#pragma unroll 1
          for (int cc = 0; cc < 128; cc += 32) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + cc, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x16(t_o + cc, *reinterpret_cast<uint32_t(*)[16]>(&o[0]));
            tmem_st_32x32b_x16(t_o + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(&o[16]));
          }
        } else {
          tc_fence_after();
        }
        const uint32_t t_p = tmem + t_lane + C2_TM_P + b * 64;
#pragma unroll
        for (int cc = 0; cc < 64; cc += 16)
          tmem_st_32x32b_x16(t_p + cc, *reinterpret_cast<uint32_t(*)[16]>(&pk[cc]));
        tmem_st_wait();
        EV2(17);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(lead_bars + 96 + 8 * b);  // p_full(b) on the leader
        EV2(15);
      }
      // ---------------- epilogue: O / l, lse (warpgroup wg: O columns 64 wg ..) ----------------
      const uint32_t g_last = g - 1;
      (void)g_item;
      // PV(g_last - 1), then PV(g_last): each wait is at most one phase ahead
      // of its barrier (see the rescale), so the parities cannot alias
      if (g_last >= 1) mbar_wait(pv_done((g_last - 1) & 1), ((g_last - 1) >> 1) & 1, 41);
      mbar_wait(pv_done(g_last & 1), (g_last >> 1) & 1, 40);
      tc_fence_after();
      uint32_t w[32];
      {
        const uint32_t t_o = tmem + t_lane + C2_TM_O + wg * 64;
        uint32_t o[64];
        tmem_ld_32x32b_x32(t_o, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
        tmem_ld_32x32b_x32(t_o + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(lead_bars + 112);  // o_free on the leader
        // combine the two warpgroups' sums: m_final = the larger reference max
        lred[wg * 256 + trow] = l;
        lred[wg * 256 + 128 + trow] = m_seen;
        named_bar_sync(9 + q, 64);
        const float l2 = lred[(wg ^ 1) * 256 + trow], m2 = lred[(wg ^ 1) * 256 + 128 + trow];
        named_bar_sync(9 + q, 64);  // both read before either rewrites (next item)
        const float mf = fmaxf(m_seen, m2);
        const float lt = (m_seen == -INFINITY ? 0.f : l * ex2(m_seen - mf)) + (m2 == -INFINITY ? 0.f : l2 * ex2(m2 - mf));
        const float inv_l = (lt > 0.f) ? 1.f / lt : 0.f;
        if (wg == 0 && row < p.seq && p.lse != nullptr)
          p.lse[(size_t)bh * p.seq + row] = (mf + __log2f(lt)) * (1.0f / LOG2E);
#pragma unroll
        for (int e = 0; e < 32; ++e)
          w[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
        (void)m_last;
      }
      // O / l through this warp's 4 KiB SW128 box (32 rows x 64 columns) and a TMA store
      const uint32_t obuf = sbase + C2_SMEM_O + (uint32_t)warp * 4096;
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        st_shared_v4(obuf + lane * 128 + ((cc ^ (lane & 7)) << 4), w[4 * cc], w[4 * cc + 1], w[4 * cc + 2],
                     w[4 * cc + 3]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0 && p.dbg != 1) {
        tma_store_3d(&tmO, obuf, 64 * wg, rt + q * 32, bh);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync();
#ifdef MIMW_FA_EVENTS
  if (blockIdx.x < 2 && lane == 0 && p.trace)
    for (int e = 0; e < ev_n; ++e) p.trace[(rank * 12 + warp) * 1024 + e] = ev_mine[e];
#endif
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}
