"""The mbarrier contract every kernel relies on, checked on the hardware: the
B200 analogue of the reference's MbarrierState unit tests
(proj/tests/test_sync.cpp:10-85; sync.hpp:16-45: a phase flips iff no
arrivals and no transaction bytes are pending; try_wait(p) <=> phase != p).
csrc/selftest.cu runs each scenario in one 2-CTA cluster."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu

CHECKS = ["fresh barrier: phase 0 open", "fresh barrier: parity 1 counts as complete (full of emptiness)",
          "count 1: one arrive completes the phase", "after the flip, phase 1 is open",
          "count 2: one arrive leaves it open", "count 2: the second arrive completes it",
          "expect_tx 16 + 16-byte bulk copy completes", "bulk-copied bytes visible after the wait",
          "expect_tx 32 + two 16-byte copies complete", "arrive.expect_tx(0) completes at once",
          "four phases alternate parity", "remote arrive from the peer CTA (cluster) completes a phase"]


def test_mbarrier_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    out = (ctypes.c_int * len(CHECKS))()
    n = P.lib().mimw_b200_selftest_mbarrier(out, len(CHECKS))
    assert n == len(CHECKS)
    failed = [c for c, v in zip(CHECKS, out) if v != 1]
    assert not failed, failed


@pytest.mark.parametrize("cluster", [1, 2])
@pytest.mark.parametrize("ntiles,spin", [(1, 0), (148, 0), (5000, 0), (3000, 20000)])
def test_clc_exactly_once(cluster, ntiles, spin):
    """Cluster launch control on the hardware (the reference's test_clc.cpp:
    25-92: every tile dispatched exactly once, then the -1 sentinel): a grid of
    ntiles clusters whose running clusters cancel pending ones and do their
    tiles, with the response ring the grouped GEMM uses."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    out = (ctypes.c_int * 3)()
    assert P.lib().mimw_b200_selftest_clc(ntiles, cluster, spin, out) == 0
    assert out[0] == 0, f"{out[0]} tiles not done exactly once"
    if ntiles >= 3000:
        assert out[1] > 0 and out[2] > 1, "no cluster cancelled another (no work stealing)"
