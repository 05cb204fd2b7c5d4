"""Schedule independence: the B200 analogue of the reference's 100-seed
schedule-robustness criterion (acceptance.cpp:428-486, test_kernels.cpp:37-61)
and of CLC exactly-once (test_clc.cpp:25-92).  The kernels hand out work
through different paths: hardware cluster launch control (GEMM and grouped
GEMM by default, max_clusters=0), persistent static striding (max_clusters > 0)
or the atomic work counter published through a 2-slot mbarrier ring with a -1
sentinel (attention forward).  Every tile must be
computed exactly once, in the same arithmetic order, whatever the CTA count,
so the results must be bit-identical across grid sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def test_gemm_bitwise_across_cluster_counts(P):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    a = (torch.rand((1000, 520), device="cuda", generator=g) * 2 - 1).bfloat16()
    b = (torch.rand((520, 1288), device="cuda", generator=g) * 2 - 1).bfloat16()
    ref = P.gemm(a, b, out_dtype=torch.float32)
    for mc in (1, 3, 7, 40, 0):
        for rg in (1, 8):
            c = P.gemm(a, b, out_dtype=torch.float32, max_clusters=mc, raster_group=rg)
            assert torch.equal(c, ref), (mc, rg)


def test_grouped_gemm_bitwise_across_cluster_counts(P):
    import torch
    g = torch.Generator(device="cuda").manual_seed(4)
    offs = np.array([0, 300, 300, 301, 900, 1000], np.int64)
    x = (torch.rand((1000, 256), device="cuda", generator=g) * 2 - 1).bfloat16()
    w = (torch.rand((5, 256, 520), device="cuda", generator=g) * 2 - 1).bfloat16()
    ref = P.grouped_gemm(x, offs, w)
    for mc in (1, 2, 5, 17):
        assert torch.equal(P.grouped_gemm(x, offs, w, max_clusters=mc), ref), mc


@pytest.mark.parametrize("causal", [True, False])
def test_attention_bitwise_across_cta_counts(P, causal):
    """The dynamic scheduler (atomic counter + mbarrier ring + -1 sentinel):
    1 CTA does every item, 148 race for them; the output may not change."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = ((torch.rand((2, 3, 1100, 128), device="cuda", generator=g) * 2 - 1).bfloat16()
               for _ in range(3))
    ref_o, ref_l = P.attention_fwd(q, k, v, causal=causal)
    for ctas in (1, 2, 5, 13, 0):
        o, l = P.attention_fwd(q, k, v, causal=causal, max_ctas=ctas)
        assert torch.equal(o, ref_o) and torch.equal(l, ref_l), ctas


def test_multi_device_gemm_bitwise_across_comm_modes(P):
    """The all-gather GEMM: where the comm agents run (every GEMM CTA, or 1-8
    dedicated pairs) changes the transfer schedule, never the result."""
    import torch
    from paper_2605_10905_b200 import multi_device as MD
    g = torch.Generator(device="cuda").manual_seed(6)
    ks = [256, 136, 64]
    a = [(torch.rand((700, k), device="cuda", generator=g) * 2 - 1).bfloat16() for k in ks]
    b = [(torch.rand((k, 520), device="cuda", generator=g) * 2 - 1).bfloat16() for k in ks]
    ref = MD.emulated_multi_device_gemm(a, b)
    for cp in (-1, 1, 3, 8):
        for conc in (False, True):
            out = MD.emulated_multi_device_gemm(a, b, comm_pairs=cp, concurrent=conc)
            assert torch.equal(out, ref), (cp, conc)


def test_attention_concurrent_streams_bitwise(P):
    """Two forward launches in flight on different streams (the host entries
    run one stream per calling thread): each launch's work counter is its own
    stream-ordered scratch, so both outputs equal their one-at-a-time runs."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    qs = [[(torch.rand((1, 8, 2048, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3)]
          for _ in range(2)]
    ref = [P.attention_fwd(*t)[0].clone() for t in qs]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            o1 = P.attention_fwd(*qs[0])[0]  # current stream = s1
        with torch.cuda.stream(s2):
            o2 = P.attention_fwd(*qs[1])[0]  # current stream = s2
        outs.append((o1, o2))
    torch.cuda.synchronize()
    for o1, o2 in outs:
        assert torch.equal(o1, ref[0]) and torch.equal(o2, ref[1])
