"""GPU parity of the non-causal attention forward and the attention backward
(PAPER.md:702-716 AFN / ABC rows).

Neither has a reference oracle (the reference's attention is causal and
forward-only, oracles.cpp:119-145).  The oracles are restatements in
oracle/oracle.c: ``oracle_attention_full`` (the reference's arithmetic with
the key range widened to every key) and ``oracle_attention_bwd`` (the
standard gradients, in f64); both are checked against torch f64 autograd in
tests/test_oracle.py.  At sizes the CPU oracle cannot finish, a torch fp32
autograd reference on the same bf16 inputs is the check.

Tolerances (max-norm rel_error, case.cpp:94-104):
  forward  1e-2 (north_star bf16)
  backward 2e-2: P and dS are rounded to bf16 before the dV / dK / dQ MMAs
           (as every bf16 flash-attention backward does) and o is the
           kernel's bf16 output, so the error is ~2 bf16 roundings of O(1)
           terms, accumulated over the keys.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-2
BWD_TOL = 2e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def _heads(bh, s, seed):
    return [oracle.round_bf16(oracle.random_tile([bh, s, 128], oracle.input_seed(seed, i)))
            for i in range(4)]


def _dev(x, b, h):
    import torch
    s = x.shape[1]
    return torch.from_numpy(x).cuda().bfloat16().view(b, h, s, 128).contiguous()


@pytest.mark.parametrize("s", [64, 200, 300, 1000])
def test_noncausal_forward(P, s):
    import torch
    q, k, v, _ = _heads(2, s, 41)
    o, lse = P.attention_fwd(_dev(q, 1, 2), _dev(k, 1, 2), _dev(v, 1, 2), causal=False)
    torch.cuda.synchronize()
    o = o.float().cpu().numpy().reshape(2, s, 128)
    lse = lse.cpu().numpy().reshape(2, s)
    for hd in range(2):
        want, wl = oracle.oracle_attention_full(q[hd], k[hd], v[hd], 128 ** -0.5)
        assert oracle.rel_error(o[hd], want) <= FWD_TOL
        assert oracle.rel_error_rows(o[hd], want) <= FWD_TOL
        assert np.abs(lse[hd] - wl).max() <= 1e-3 * max(1.0, np.abs(wl).max())


@pytest.mark.parametrize("s,causal,w", [
    (128, False, None), (200, False, None), (300, False, None),
    (128, True, None), (300, True, None), (256, True, 77), (1000, True, None), (1000, False, None),
])
def test_backward_vs_oracle(P, s, causal, w):
    import torch
    b, h = 1, 2
    q, k, v, do = _heads(b * h, s, 57 + s)
    tq, tk, tv, tdo = (_dev(x, b, h) for x in (q, k, v, do))
    window = (w if w is not None else s) if causal else None
    o, lse = P.attention_fwd(tq, tk, tv, window=window, causal=causal)
    dq, dk, dv = P.attention_bwd(tq, tk, tv, o, tdo, lse, window=window, causal=causal)
    torch.cuda.synchronize()
    got = [t.float().cpu().numpy().reshape(b * h, s, 128) for t in (dq, dk, dv)]
    for hd in range(b * h):
        want = oracle.oracle_attention_bwd(q[hd], k[hd], v[hd], do[hd], 128 ** -0.5, causal=causal,
                                           w=w)
        for name, g, wnt in zip(("dq", "dk", "dv"), got, want):
            e = oracle.rel_error(g[hd], wnt)
            assert np.isfinite(g[hd]).all(), name
            assert e <= BWD_TOL, (name, hd, e)


def _torch_ref(q, k, v, do, causal, scale):
    import torch
    qf, kf, vf = (t.float().detach().requires_grad_(True) for t in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, is_causal=causal, scale=scale)
    return torch.autograd.grad(o, (qf, kf, vf), do.float())


@pytest.mark.parametrize("causal", [False, True])
def test_backward_long_sequence_vs_torch_fp32(P, causal):
    """S = 4096, B*H = 4 (the ABC3 shape scaled down in heads): torch fp32
    autograd on the same bf16 inputs as the reference check."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(11)
    b, h, s = 2, 2, 4096
    q, k, v, do = ((torch.rand((b, h, s, 128), device="cuda", generator=g) * 2 - 1).bfloat16()
                   for _ in range(4))
    o, lse = P.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = P.attention_bwd(q, k, v, o, do, lse, causal=causal)
    ref = _torch_ref(q, k, v, do, causal, 128 ** -0.5)
    torch.cuda.synchronize()
    for name, got, want in zip(("dq", "dk", "dv"), (dq, dk, dv), ref):
        e = float((got.float() - want).abs().max() / want.abs().max())
        assert e <= BWD_TOL, (name, e)


def test_backward_arguments(P):
    import torch
    q = torch.zeros((1, 1, 130, 128), device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros((1, 1, 130), device="cuda")
    with pytest.raises(P.MimwError):  # negative window
        P.attention_bwd(q, q, q, q, q, lse, window=-3)
