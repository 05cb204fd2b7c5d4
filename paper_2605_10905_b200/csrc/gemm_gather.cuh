// All-gather (K-gathered) multi-device GEMM: the problem policy and the comm
// role of gemm_bf16_kernel (included by gemm_bf16.cu inside its anonymous
// namespace; needs SchedT, TileCoord and the ptx.cuh primitives).
#pragma once

// K-gathered multi-device GEMM (proj/kernels/multi_device_gemm.mimw:1-79,
// oracle_multi_device_gemm oracles.cpp:57-80, generalised from 2 to `world`
// K-splits): device s holds A_s [M, k_s] and B_s [k_s, N]; this rank owns
// C rows [row0, row0 + rows) = sum_s A_s[rows] . B_s.  Two roles:
//   comm agents (the reference's rank-0 "comm" CTA): pull every remote split
//     in 256-column K slabs, box by box, from the peer's HBM (NVLink via the
//     IPC-mapped pointer) through smem into a local landing buffer (TMA load
//     -> TMA store); a signaler thread publishes each slab on a readiness
//     counter (red.release.gpu; the "remote barrier_arrive" of :67).  By
//     default warp 6 of every GEMM CTA is an agent (16 KiB buffer); with
//     comm_clusters > 0, dedicated comm CTA pairs run several agents each.
//   GEMM pairs (the reference's compute CTA): the persistent 2-CTA GEMM over
//     the splits in rotation order q = 0 (local split, no wait), 1, ...; the
//     producer waits on a slab's counter (ld.acquire) before its first TMA
//     load from the landing buffer, so the transfer of split q overlaps the
//     tensor-core work on splits < q tile by tile.
constexpr int MAX_SPLITS = 8;
constexpr int kDefaultCommPairs = -1;  // distributed comm warps (see multi_device_gemm_launch)
constexpr int COMM_SLAB = 256;   // K columns per readiness counter
// comm boxes are {256, R} with 512-byte rows (TMA moves long rows far faster
// than 128-byte ones): A box = one slab's 256 K columns x R rows, B box = 256
// N columns x R K rows.  R = box rows (32 / 64 / 128: 16 / 32 / 64 KiB).
constexpr int COMM_W = 256;
constexpr int COMM_MAX_BUFS = 24;
struct GatherSched : SchedT<1> {
  static constexpr bool kGather = true;
  static constexpr bool kClc = false;  // comm and GEMM CTAs must be co-resident: persistent grid
  CUtensorMap ga[MAX_SPLITS], gb[MAX_SPLITS];          // GEMM operands, rotation order (q = 0 local)
  CUtensorMap src_a[MAX_SPLITS], dst_a[MAX_SPLITS];    // comm: peer A rows -> landing (q >= 1)
  CUtensorMap src_b[MAX_SPLITS], dst_b[MAX_SPLITS];    // comm: peer B -> landing (q >= 1)
  int ks[MAX_SPLITS];
  int nsplit, kblocks, comm_clusters, max_slabs, rbox, nbox;
  int box;                    // comm box rows R (32 / 64 / 128): 16 / 32 / 64 KiB boxes
  int agents;                 // independent TMA copy pipelines per comm CTA (one thread each)
  int lag;                    // stores in flight before a slab signal waits for completion
  int pull;                   // 0: this rank pulls nothing (no rows), barrier only
  uint32_t *ctr;              // [MAX_SPLITS * max_slabs] slab counters + GO + PULLED, zeroed per launch
  uint32_t *pad_local;        // this rank's signal pad: IN[MAX_SPLITS], OUT[MAX_SPLITS]; null = no barrier
  uint32_t *pad_peer[MAX_SPLITS];
  uint32_t epoch;
  uint64_t peer_budget;       // cycles a peer-dependent wait may spin before trapping (0 = forever)
  int rank, world;
  __device__ __forceinline__ int nslabs(int q) const { return (ks[q] + COMM_SLAB - 1) / COMM_SLAB; }
  // B boxes of slab j (K rows of the slab that exist, R at a time)
  __device__ __forceinline__ int bsub(int q, int j) const {
    const int left = ks[q] - j * COMM_SLAB;
    return min(COMM_SLAB / box, (left + box - 1) / box);
  }
  __device__ __forceinline__ uint32_t pieces(int q, int j) const {
    if (j >= nslabs(q)) return 0u;  // empty split
    return (uint32_t)(rbox + bsub(q, j) * nbox);
  }
};

// Position in the rotation-ordered list of comm boxes: split q (>= 1), slab j,
// piece p of that slab's P boxes (the rbox A boxes first, then the B boxes).
// A comm agent walks every nagents-th box.
struct BoxCursor {
  int q, j, p;
  uint32_t P;
  bool live;
  __device__ __forceinline__ void init(const GatherSched &sp, int first) {
    q = 1; j = 0; p = 0;
    live = sp.pull && sp.nsplit > 1;
    P = live ? sp.pieces(1, 0) : 0;
    advance(sp, first);
  }
  __device__ __forceinline__ void advance(const GatherSched &sp, int by) {
    p += by;
    while (live && p >= (int)P) {
      p -= (int)P;
      if (++j >= sp.nslabs(q)) {
        j = 0;
        if (++q >= sp.nsplit) { live = false; break; }
      }
      P = sp.pieces(q, j);
    }
  }
  __device__ __forceinline__ uint32_t *ctr(const GatherSched &sp) const { return sp.ctr + q * sp.max_slabs + j; }
};

// mailbox publish / read as shared-memory atomics (release / acquire at CTA
// scope; atomics also keep compute-sanitizer's racecheck, which does not model
// plain acquire/release flags, out of the message passing)
__device__ __forceinline__ void st_release_cta_shared(uint32_t addr, uint32_t v) {
  asm volatile("{\n\t.reg .b32 prev;\n\tatom.release.cta.shared::cta.exch.b32 prev, [%0], %1;\n\t}" ::"r"(addr), "r"(v)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta_shared(uint32_t addr) {
  uint32_t v;
  asm volatile("atom.acquire.cta.shared::cta.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// One comm agent (a single thread): copies boxes g = agent, agent + nagents,
// ... through `nb` smem buffers — TMA load from the peer into buffer
// i % nb, TMA store into the landing buffer, the buffer refilled once its
// store has read it.  Once a store has fully landed (bulk wait_group, LAG
// stores behind the newest so the agent rarely blocks), the agent publishes
// its landed-box count in its smem mailbox; the CTA's signaler thread turns
// counts into slab-counter releases (a release here would wait for this
// thread's in-flight TMA traffic and serialise the pipeline).
template <int LAG>
__device__ __forceinline__ void gather_agent(const GatherSched &sp, uint32_t buf0, uint32_t bar0,
                                             int nb, int agent, int nagents, uint32_t mbox) {
  const uint32_t box_bytes = (uint32_t)sp.box * COMM_W * 2;
  for (int i = 0; i < nb; ++i) mbar_init(bar0 + 8 * i, 1);
  fence_mbar_init();
  BoxCursor cur;
  cur.init(sp, agent);
  const CUtensorMap *dmap[COMM_MAX_BUFS];
  int dx[COMM_MAX_BUFS], dy[COMM_MAX_BUFS];
  auto issue_load = [&](int idx) {
    const int slot = idx % nb;
    const int k0 = cur.j * COMM_SLAB;
    const CUtensorMap *src;
    int x, y;
    if (cur.p < sp.rbox) {
      src = &sp.src_a[cur.q]; dmap[slot] = &sp.dst_a[cur.q]; x = k0; y = cur.p * sp.box;
    } else {
      const int pb = cur.p - sp.rbox;
      src = &sp.src_b[cur.q]; dmap[slot] = &sp.dst_b[cur.q];
      x = (pb % sp.nbox) * COMM_W; y = k0 + (pb / sp.nbox) * sp.box;
    }
    dx[slot] = x;
    dy[slot] = y;
    const uint32_t bar = bar0 + 8 * slot;
    mbar_arrive_expect_tx(bar, box_bytes);
    tma_load_2d(buf0 + slot * box_bytes, src, bar, x, y);
    cur.advance(sp, nagents);
  };
  // boxes [0, count) have landed: publish the count to the signaler (measured:
  // a red.release.gpu issued here waits for this thread's in-flight TMA
  // traffic and halved the copy rate)
  auto landed = [&](int count) {
    fence_proxy_async_global();
    st_release_cta_shared(mbox, (uint32_t)count);
  };
  int nl = 0;
  while (nl < nb && cur.live) issue_load(nl++);
  int ns = 0;
  for (; ns < nl; ++ns) {
    const int slot = ns % nb;
    mbar_wait(bar0 + 8 * slot, (uint32_t)((ns / nb) & 1), 22);
    tma_store_2d(dmap[slot], buf0 + slot * box_bytes, dx[slot], dy[slot]);
    bulk_commit();
    if (nb == 1) {
      bulk_wait_read<0>();           // single buffer: reload once this store has read it
      if (cur.live) issue_load(nl++);
    } else if (ns >= 1) {
      bulk_wait_read<1>();           // store ns-1 has read its buffer: refill it
      if (cur.live) issue_load(nl++);
    }
    if (ns >= LAG) {
      bulk_wait<LAG>();              // stores <= ns-LAG have landed
      landed(ns - LAG + 1);
    }
  }
  bulk_wait<0>();
  landed(ns);
}

// Signaler thread of a comm CTA: replays each agent's box sequence and, as
// the agents' mailboxes advance, bumps the slab counters with red.release.gpu
// (cumulative over the agents' landed stores it acquired through smem).
__device__ __forceinline__ void gather_signaler(const GatherSched &sp, int agent0, int agents,
                                                int nagents, uint32_t mbox0) {
  BoxCursor cs[6];
  int seen[6];
  for (int a = 0; a < agents; ++a) {
    cs[a].init(sp, agent0 + a);
    seen[a] = 0;
  }
  const uint64_t t0 = clock64();
  while (true) {
    bool any = false;
    for (int a = 0; a < agents; ++a) {
      if (!cs[a].live) continue;
      any = true;
      const int done = (int)ld_acquire_cta_shared(mbox0 + 4 * a);
      uint32_t *c0 = nullptr;
      uint32_t cnt = 0;
      while (seen[a] < done && cs[a].live) {
        uint32_t *c = cs[a].ctr(sp);
        if (c != c0) {
          if (cnt) red_release_gpu_add(c0, cnt);
          c0 = c;
          cnt = 0;
        }
        ++cnt;
        ++seen[a];
        cs[a].advance(sp, nagents);
      }
      if (cnt) red_release_gpu_add(c0, cnt);
    }
    if (!any) break;
    if (clock64() - t0 > MIMW_WATCHDOG_CYCLES) watchdog_trap(mbox0, 0, 26);
  }
}

// Entry barrier: every peer has launched, so its inputs are complete and it
// may read ours ("arrive remote, wait local").  The leader (comm agent 0)
// meets the peers through their signal pads and opens the local GO flag the
// other agents wait on.
__device__ __forceinline__ void gather_entry(const GatherSched &sp, bool leader) {
  if (!sp.pad_local) return;
  uint32_t *go = sp.ctr + MAX_SPLITS * sp.max_slabs;
  if (leader) {
    fence_sc_sys();
    for (int p = 0; p < sp.world; ++p)
      if (p != sp.rank) st_release_sys(sp.pad_peer[p] + sp.rank, sp.epoch);
    for (int p = 0; p < sp.world; ++p)
      if (p != sp.rank) flag_wait_geq<true>(sp.pad_local + p, sp.epoch, 20, sp.peer_budget);
    st_release_gpu(go, 1u);
  } else {
    flag_wait_geq<false>(go, 1u, 21, sp.peer_budget);
  }
}

// Exit barrier: no rank returns (and lets its caller overwrite A_s / B_s)
// before every peer has finished pulling from it.  Every agent counts itself
// out; the leader waits for all `nparts`, then meets the peers.
__device__ __forceinline__ void gather_exit(const GatherSched &sp, bool leader, uint32_t nparts) {
  if (!sp.pad_local) return;
  uint32_t *pulled = sp.ctr + MAX_SPLITS * sp.max_slabs + 1;
  red_release_gpu_add(pulled, 1u);
  if (!leader) return;
  flag_wait_geq<false>(pulled, nparts, 23);
  fence_sc_sys();
  for (int p = 0; p < sp.world; ++p)
    if (p != sp.rank) st_release_sys(sp.pad_peer[p] + MAX_SPLITS + sp.rank, sp.epoch);
  for (int p = 0; p < sp.world; ++p)
    if (p != sp.rank) flag_wait_geq<true>(sp.pad_local + MAX_SPLITS + p, sp.epoch, 24, sp.peer_budget);
}

__device__ __forceinline__ void gather_agent_lag(const GatherSched &sp, uint32_t buf0, uint32_t bar0,
                                                 int nb, int agent, int nagents, uint32_t mbox) {
  switch (sp.lag) {
    case 1: gather_agent<1>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
    case 2: gather_agent<2>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
    case 4: gather_agent<4>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
    case 6: gather_agent<6>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
    case 12: gather_agent<12>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
    default: gather_agent<8>(sp, buf0, bar0, nb, agent, nagents, mbox); break;
  }
}

// Dedicated comm CTA (comm_clusters > 0; the reference's rank-0 comm CTA,
// multi_device_gemm.mimw:23-49): `agents` copy pipelines over the CTA's
// whole smem ring, warp 7 the signaler.
__device__ __forceinline__ void gather_comm_cta(const GatherSched &sp, uint32_t ring, uint32_t ring_bytes,
                                                uint32_t bars, uint32_t mbox0, int ci, int ncomm) {
  const int warp = threadIdx.x / 32;
  const bool lane0 = (threadIdx.x % 32) == 0;
  if (threadIdx.x == 0) gather_entry(sp, ci == 0);
  __syncthreads();
  const int nagents = ncomm * sp.agents;
  if (lane0 && warp < sp.agents) {
    const uint32_t box_bytes = (uint32_t)sp.box * COMM_W * 2;
    const int nbuf = min((int)(ring_bytes / box_bytes), COMM_MAX_BUFS);
    const int nb = nbuf / sp.agents;
    gather_agent_lag(sp, ring + warp * nb * box_bytes, bars + 8 * warp * nb, nb,
                     ci * sp.agents + warp, nagents, mbox0 + 4 * warp);
  } else if (lane0 && warp == 7) {
    gather_signaler(sp, ci * sp.agents, sp.agents, nagents, mbox0);
  }
  __syncthreads();
  if (threadIdx.x == 0) gather_exit(sp, ci == 0, (uint32_t)ncomm);
}
