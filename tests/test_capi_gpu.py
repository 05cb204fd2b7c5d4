"""GPU tests of the boundary's library hygiene and argument validation
(ADVICE r01):

* scratch comes from a library-private memory pool: the device's default pool
  (the host application's cudaMallocAsync) keeps its release threshold;
* the FA scheduler counter ring self-resets (many more launches than slots,
  two streams) and results stay bitwise identical;
* the batched host attention entry equals per-head reference-signature calls
  bitwise and matches oracle_attention (oracles.cpp:119-145);
* the torch wrappers reject mis-shaped / mis-typed operands before launching.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def _default_pool_threshold():
    from cuda.bindings import runtime as rt
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    assert err == rt.cudaError_t.cudaSuccess
    err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert err == rt.cudaError_t.cudaSuccess
    return int(v)


def test_default_mempool_untouched(P):
    import torch
    before = _default_pool_threshold()
    q, k, v, do = ((torch.rand((1, 2, 512, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(4))
    o, lse = P.attention_fwd(q, k, v)
    P.attention_bwd(q, k, v, o, do, lse)
    a = oracle.random_tile([300, 200], 1)
    b = oracle.random_tile([200, 136], 2)
    P.oracle_gemm(a, b)
    P.oracle_attention(oracle.random_tile([100, 64], 3), oracle.random_tile([100, 64], 4),
                       oracle.random_tile([100, 64], 5), 100, 0.125)
    torch.cuda.synchronize()
    assert _default_pool_threshold() == before
    P.trim_pool()


def test_fa_counter_ring_self_resets(P):
    """1100 launches (> the 1024-slot ring) on two alternating streams: every
    output equals the first, so no launch saw a stale counter."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = ((torch.rand((2, 3, 700, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3))
    ref, ref_lse = P.attention_fwd(q, k, v)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty_like(ref) for _ in range(2)]
    lses = [torch.empty_like(ref_lse) for _ in range(2)]
    for it in range(1100):
        i = it & 1
        with torch.cuda.stream(streams[i]):
            P.attention_fwd(q, k, v, out=outs[i], lse=lses[i], stream=streams[i].cuda_stream)
        if it % 97 == 0 or it >= 1098:
            streams[i].synchronize()
            assert torch.equal(outs[i], ref) and torch.equal(lses[i], ref_lse), it
    torch.cuda.synchronize()


@pytest.mark.parametrize("heads,s,d,w", [(5, 300, 64, 300), (3, 1000, 128, 257), (1, 8192, 128, 8192)])
def test_attention_heads_entry(P, heads, s, d, w):
    q, k, v = (oracle.round_bf16(oracle.random_tile([heads, s, d], oracle.input_seed(17 + s, i)))
               for i in range(3))
    o, lse = P.oracle_attention_heads(q, k, v, w, d ** -0.5, with_lse=True)
    for h in range(heads):
        o1, l1 = P.oracle_attention(q[h], k[h], v[h], w, d ** -0.5, with_lse=True)
        np.testing.assert_array_equal(o[h], o1)
        np.testing.assert_array_equal(lse[h], l1)
    rows = sorted({0, 1, s // 2, s - 1})
    for h in range(heads):
        want, wl = oracle.oracle_attention_rows(q[h], k[h], v[h], w, d ** -0.5, rows[0], rows[-1] + 1)
        got = o[h][rows[0]:rows[-1] + 1]
        assert oracle.rel_error_rows(got[[r - rows[0] for r in rows]], want[[r - rows[0] for r in rows]]) <= 1e-2
        assert np.max(np.abs(lse[h][rows[0]:rows[-1] + 1] - wl)) <= 1e-2


def test_attention_heads_f32_precision(P):
    q, k, v = (oracle.random_tile([2, 64, 32], oracle.input_seed(9, i)) for i in range(3))
    o = P.oracle_attention_heads(q, k, v, 16, 0.25, precision=P.PREC_F32)
    for h in range(2):
        assert oracle.rel_error(o[h], oracle.oracle_attention(q[h], k[h], v[h], 16, 0.25)) <= 1e-4


def test_wrapper_validation(P):
    import torch
    a = torch.zeros((64, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(P.MimwError) as e:
        P.gemm(a, torch.zeros((64, 32), device="cuda", dtype=torch.bfloat16))  # K mismatch
    assert e.value.code == P.ERR_SHAPE
    with pytest.raises(P.MimwError) as e:
        P.gemm(a.float(), torch.zeros((128, 32), device="cuda", dtype=torch.bfloat16))  # dtype
    assert e.value.code == P.ERR_UNSUPPORTED
    with pytest.raises(P.MimwError) as e:
        P.gemm(a, torch.zeros((32, 64), device="cuda", dtype=torch.bfloat16), b_layout=P.B_NK)
    assert e.value.code == P.ERR_SHAPE
    q = torch.zeros((1, 2, 256, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(P.MimwError) as e:
        P.attention_fwd(q, torch.zeros((1, 1, 256, 128), device="cuda", dtype=torch.bfloat16), q)  # GQA shape
    assert e.value.code == P.ERR_SHAPE
    with pytest.raises(P.MimwError):
        P.attention_fwd(q.float(), q, q)
    x = torch.zeros((4, 1024), device="cuda")
    with pytest.raises(P.MimwError) as e:
        P.layernorm(x, torch.zeros(512, device="cuda"), torch.zeros(1024, device="cuda"))
    assert e.value.code == P.ERR_SHAPE
    # the C hooks check alignment / extents too
    L = P.lib()
    base = q.data_ptr()
    r = L.mimw_b200_attention_fwd_ex(base + 2, base, base, base, None, 1, 1, 256, 256, 0.1, -1, 0, None, 1, None)
    assert r == P.ERR_UNSUPPORTED and b"aligned" in L.mimw_b200_last_error()
    r = L.mimw_b200_gemm_bf16_ex(a.data_ptr(), a.data_ptr(), a.data_ptr(), 64, 64, 128, 100, 64, 64, 0, 1, 2, 0,
                                 0, 0, None)
    assert r == P.ERR_SHAPE or r == P.ERR_UNSUPPORTED


def test_wrapper_validation_other_kernels(P):
    """gemm_mxfp8, grouped_gemm, simplicial_attention_fwd and attention_bwd
    reject mis-typed / mis-shaped operands before any launch (the C side
    builds its tensor maps from one operand's extents)."""
    import torch
    cu = dict(device="cuda")
    qa = torch.zeros((128, 256), dtype=torch.uint8, **cu).view(torch.float8_e4m3fn)
    sf = torch.zeros((128, 8), dtype=torch.uint8, **cu)
    P.gemm_mxfp8(qa, sf, qa, sf)  # well-formed
    bad = [
        lambda: P.gemm_mxfp8(qa, sf[:, :4].contiguous(), qa, sf),                 # sfa too small
        lambda: P.gemm_mxfp8(qa, sf, qa[:, :128].contiguous(), sf),               # K mismatch
        lambda: P.gemm_mxfp8(qa.view(torch.uint8).bfloat16(), sf, qa, sf),        # dtype
    ]
    x = torch.zeros((40, 64), dtype=torch.bfloat16, **cu)
    w = torch.zeros((2, 64, 96), dtype=torch.bfloat16, **cu)
    P.grouped_gemm(x, [0, 10, 40], w)
    bad += [
        lambda: P.grouped_gemm(x.float(), [0, 10, 40], w),                        # dtype
        lambda: P.grouped_gemm(x, [0, 10, 40], w[:, :32].contiguous()),           # K mismatch
        lambda: P.grouped_gemm(x, [0, 10, 40], w, out=torch.zeros((40, 64), dtype=torch.bfloat16, **cu)),
    ]
    t = torch.zeros((1, 64, 128), dtype=torch.bfloat16, **cu)
    P.simplicial_attention_fwd(t, t, t, t, t, 2, 16)
    bad += [
        lambda: P.simplicial_attention_fwd(t, t, t.float(), t, t, 2, 16),         # dtype
        lambda: P.simplicial_attention_fwd(t, t, t, t[:, :32].contiguous(), t, 2, 16),  # shape
    ]
    q = torch.zeros((1, 1, 64, 128), dtype=torch.bfloat16, **cu)
    lse = torch.zeros((1, 1, 64), **cu)
    P.attention_bwd(q, q, q, q, q, lse)
    bad += [
        lambda: P.attention_bwd(q, q, q, q, q, lse[:, :, :32].contiguous()),      # lse shape
        lambda: P.attention_bwd(q, q[:, :, :32].contiguous(), q, q, q, lse),      # k shape
        lambda: P.attention_bwd(q, q, q, q, q.float(), lse),                      # dtype
    ]
    for i, f in enumerate(bad):
        with pytest.raises(P.MimwError):
            f()
    torch.cuda.synchronize()


def test_run_oracle_simplicial_defaults(P):
    """run_oracle uses the reference's scalar defaults sc("w1", 2), sc("w2", 16),
    sc("scale", 1.0) (oracles.cpp:190-193)."""
    xs = {n: oracle.random_tile([32, 16], oracle.input_seed(31, i))
          for i, n in enumerate(["q", "k1", "v1", "k2", "v2"])}
    got = P.run_oracle("simplicial_attention", xs, {}, precision=P.PREC_F32)
    want_o, want_l = oracle.oracle_simplicial_attention(xs["q"], xs["k1"], xs["v1"], xs["k2"], xs["v2"],
                                                        2, 16, 1.0)
    assert oracle.rel_error(got["o"], want_o) <= 1e-3
