// Hardware-contract self-test of the mbarrier primitives every kernel relies
// on (ptx.cuh): the B200 analogue of the reference's mbarrier unit tests
// (proj/tests/test_sync.cpp:10-85, MbarrierState in core/include/mimw/sync.hpp:
// 16-45, phase flips iff pending == 0 and tx == 0).  One CTA runs each
// scenario and records what the hardware did; tests/test_selftest_gpu.py
// checks the pattern.  Exported as a test hook (not in the public header).
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace mimw {

namespace {

enum : int {
  kFreshParity0Open = 0,    // try_wait(0) on a fresh barrier: phase 0 not complete
  kFreshParity1Done,        // try_wait(1): the "previous" phase counts as complete ("full of emptiness")
  kOneArrivalFlips,         // count 1: one arrive completes phase 0
  kAfterFlipParity1Open,    // ... and phase 1 is then open
  kTwoArrivalsFirstOpen,    // count 2: one arrive leaves the phase open
  kTwoArrivalsSecondDone,   // ... the second completes it
  kTxCompletes,             // expect 16 + a 16-byte bulk copy (complete_tx 16) completes the phase
  kTxData,                  // ... and the copied bytes are visible after the wait
  kTxTwoPartials,           // expect 32 + two 16-byte copies complete it
  kExpectZero,              // arrive.expect_tx(0) completes immediately
  kParityAlternates,        // four phases in a row alternate parity 0,1,0,1
  kRemoteArriveCluster,     // an arrive from the peer CTA of a 2-CTA cluster completes a local phase
  kNumChecks
};

__global__ void __cluster_dims__(2, 1, 1) mbar_selftest_kernel(int *out, const uint4 *src) {
  __shared__ alignas(8) uint64_t bars[8];
  __shared__ alignas(16) uint4 buf[2];
  const uint32_t rank = cluster_ctarank();
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  if (threadIdx.x == 0) {
    mbar_init(bar(0), 1);
    mbar_init(bar(1), 2);
    mbar_init(bar(2), 1);
    mbar_init(bar(3), 1);
    mbar_init(bar(4), 1);
    mbar_init(bar(5), 1);
    mbar_init(bar(6), 1);  // remote-arrive target
    fence_mbar_init();
  }
  cluster_sync();
  if (rank == 0 && threadIdx.x == 0) {
    out[kFreshParity0Open] = !mbar_test_wait(bar(0), 0);
    out[kFreshParity1Done] = mbar_test_wait(bar(0), 1);
    mbar_arrive(bar(0));
    out[kOneArrivalFlips] = mbar_test_wait(bar(0), 0);
    out[kAfterFlipParity1Open] = !mbar_test_wait(bar(0), 1);

    mbar_arrive(bar(1));
    out[kTwoArrivalsFirstOpen] = !mbar_test_wait(bar(1), 0);
    mbar_arrive(bar(1));
    out[kTwoArrivalsSecondDone] = mbar_test_wait(bar(1), 0);

    mbar_arrive_expect_tx(bar(2), 16);
    bulk_load(smem_u32(&buf[0]), src, 16, bar(2));
    mbar_wait(bar(2), 0, 90);
    out[kTxCompletes] = 1;
    out[kTxData] = buf[0].x == src[0].x && buf[0].y == src[0].y && buf[0].z == src[0].z && buf[0].w == src[0].w;

    mbar_arrive_expect_tx(bar(3), 32);
    bulk_load(smem_u32(&buf[0]), src, 16, bar(3));
    bulk_load(smem_u32(&buf[1]), src + 1, 16, bar(3));
    mbar_wait(bar(3), 0, 91);
    out[kTxTwoPartials] = buf[1].x == src[1].x;

    mbar_arrive_expect_tx(bar(4), 0);
    out[kExpectZero] = mbar_test_wait(bar(4), 0);

    int alt = 1;
    for (int ph = 0; ph < 4; ++ph) {
      alt &= !mbar_test_wait(bar(5), ph & 1);
      mbar_arrive(bar(5));
      alt &= mbar_test_wait(bar(5), ph & 1);
    }
    out[kParityAlternates] = alt;
  }
  if (rank == 1 && threadIdx.x == 0) mbar_arrive_cluster(map_to_rank(bar(6), 0));
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait_cluster(bar(6), 0, 92);
    out[kRemoteArriveCluster] = 1;
  }
  cluster_sync();
}


// CLC exactly-once (the reference's test_clc.cpp:25-92 on the hardware): a
// grid of `ntiles` clusters in which every running cluster keeps cancelling
// not-yet-launched clusters and doing their tile, with the same response ring
// the GEMM uses (2 slots; per slot a full barrier completed by the 16-byte
// response and an empty barrier on the leader released by every consumer of
// both CTAs).  count[t] = times tile t was done; ran[c] = tiles cluster c did.
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) clc_selftest_kernel(int *count, int *ran, int spin) {
  __shared__ alignas(16) uint4 resp[2];
  __shared__ alignas(8) uint64_t full[2], empty[2];
  const uint32_t crank = CS > 1 ? cluster_ctarank() : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 2 * CS);
    }
    fence_mbar_init();
  }
  if (CS > 1) cluster_sync(); else __syncthreads();
  const int first = (int)cluster_id_x();
  if (lane == 0 && warp < 2) {
    int t = first;
    for (int u = 0; t >= 0; ++u) {
      const int slot = u & 1;
      const uint32_t ph = (uint32_t)(u >> 1) & 1;
      const uint32_t fb = smem_u32(&full[slot]), rs = smem_u32(&resp[slot]);
      if (warp == 0) {  // requester, one tile ahead of the response it reads
        if (crank == 0) {
          mbar_wait_cluster(smem_u32(&empty[slot]), ph ^ 1, 70);
          mbar_arrive_expect_tx(fb, 16);
          if (CS > 1) clc_try_cancel_multicast(rs, fb); else clc_try_cancel(rs, fb);
          atomicAdd(&count[t], 1);
          atomicAdd(&ran[first], 1);
        } else {
          mbar_arrive_expect_tx(fb, 16);
        }
      }
      const long long t0 = clock64();
      while (clock64() - t0 < spin) {
      }
      mbar_wait(fb, ph, 71);
      const int x = clc_query(rs);
      t = x < 0 ? -1 : x / CS;
      if (CS > 1) mbar_arrive_cluster(map_to_rank(smem_u32(&empty[slot]), 0));
      else mbar_arrive(smem_u32(&empty[slot]));
    }
  }
  if (CS > 1) cluster_sync(); else __syncthreads();  // no remote arrive targets an exited CTA
}

}  // namespace

}  // namespace mimw

extern "C" int mimw_b200_selftest_mbarrier(int *host_out, int n) {
  using namespace mimw;
  if (!host_out || n < kNumChecks) return 4;
  int *d = nullptr;
  uint4 *src = nullptr;
  const uint4 h_src[2] = {{0x01020304u, 0x05060708u, 0x090a0b0cu, 0x0d0e0f10u}, {0xdeadbeefu, 1u, 2u, 3u}};
  if (cudaMalloc(&d, sizeof(int) * kNumChecks) != cudaSuccess) return 3;
  if (cudaMalloc(&src, sizeof(h_src)) != cudaSuccess) return 3;
  cudaMemset(d, 0, sizeof(int) * kNumChecks);
  cudaMemcpy(src, h_src, sizeof(h_src), cudaMemcpyHostToDevice);
  mbar_selftest_kernel<<<2, 32>>>(d, src);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(host_out, d, sizeof(int) * kNumChecks, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(src);
  return e == cudaSuccess ? kNumChecks : 3;
}

// out[0] = tiles not done exactly once, out[1] = clusters that did >= 2 tiles
// (work was stolen), out[2] = most tiles done by one cluster.  Returns 0, or a
// CUDA error code.
extern "C" int mimw_b200_selftest_clc(int ntiles, int cluster, int spin, int *out) {
  using namespace mimw;
  if (ntiles <= 0 || !out || (cluster != 1 && cluster != 2)) return -1;
  int *d = nullptr;
  if (cudaMalloc(&d, sizeof(int) * 2 * ntiles) != cudaSuccess) return 2;
  cudaMemset(d, 0, sizeof(int) * 2 * ntiles);
  if (cluster == 2) clc_selftest_kernel<2><<<2 * ntiles, 64>>>(d, d + ntiles, spin);
  else clc_selftest_kernel<1><<<ntiles, 64>>>(d, d + ntiles, spin);
  cudaError_t e = cudaDeviceSynchronize();
  int *h = new int[2 * (size_t)ntiles];
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(int) * 2 * ntiles, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e == cudaSuccess) {
    out[0] = out[1] = out[2] = 0;
    for (int i = 0; i < ntiles; ++i) {
      out[0] += h[i] != 1;
      out[1] += h[ntiles + i] >= 2;
      out[2] = h[ntiles + i] > out[2] ? h[ntiles + i] : out[2];
    }
  }
  delete[] h;
  return (int)e;
}
