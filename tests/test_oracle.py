"""CPU tests: pin the oracle restatement (oracle/oracle.c) to the reference.

1. against the committed golden fixtures produced by the UNMODIFIED
   reference (tests/golden/make_golden.py) — bit-exact for GEMM (fixed
   ascending-k float sums, oracles.cpp:17-23) and random_tile;
2. live against oracle/_ref (the reference compiled from its own sources)
   on fresh seeds and odd shapes, when _ref is present.
"""
import numpy as np
import pytest

import oracle
from golden_util import case_inputs, case_outputs


def run_restatement(case, xs):
    o = case["oracle"]
    sc = case.get("scalars", {})
    if o == "gemm":
        return {"c": oracle.oracle_gemm(xs["a"], xs["b"])}
    if o == "multi_device_gemm":
        return {"c": oracle.oracle_multi_device_gemm(xs["a0"], xs["a1"], xs["b0"], xs["b1"])}
    if o == "simplicial_attention":
        ov, lse = oracle.oracle_simplicial_attention(xs["q"], xs["k1"], xs["v1"], xs["k2"],
                                                     xs["v2"], int(sc["w1"]), int(sc["w2"]),
                                                     sc["scale"])
        return {"o": ov, "lse": lse}
    if o == "attention":
        m = case["map"]
        return {"o": oracle.oracle_attention(xs[m["q"]], xs[m["k"]], xs[m["v"]], int(sc["w"]),
                                             sc["scale"])}
    if o == "layernorm":
        return {"y": oracle.oracle_layernorm(xs["x"], xs["w"], xs["b"], sc["eps"])[0]}
    if o == "random_tile":
        return {"x": xs["x"]}
    raise KeyError(o)


def test_manifest_covers_reference_pins(golden):
    for name in ("gemm_pipeline", "gemm_clc", "multi_device_gemm", "simplicial_attention",
                 "attention_degeneration", "collective_dot", "layernorm_cluster",
                 "random_tile_9"):
        assert name in golden


@pytest.mark.parametrize("name", [
    "gemm_pipeline", "gemm_clc", "multi_device_gemm", "collective_dot", "random_tile_9",
    "gemm_bf16_256x320x384", "gemm_bf16_ragged_200x136x72",
])
def test_restatement_bit_exact_vs_golden(golden, name):
    case = golden[name]
    got = run_restatement(case, case_inputs(case))
    for k, want in case_outputs(case).items():
        assert got[k].shape == want.shape
        assert np.array_equal(got[k].view(np.uint32), want.view(np.uint32)), (name, k)


@pytest.mark.parametrize("name", [
    "simplicial_attention", "attention_degeneration", "layernorm_cluster",
    "attention_bf16_causal_s256", "attention_bf16_window_s320_w100",
])
def test_restatement_vs_golden_float(golden, name):
    # Same operation order as the reference; libm exp/log may differ in the
    # last ulp across hosts, so these are checked at 1e-6 (far below every
    # kernel tolerance) rather than bitwise.
    case = golden[name]
    got = run_restatement(case, case_inputs(case))
    for k, want in case_outputs(case).items():
        assert oracle.rel_error(got[k], want) <= 1e-6, (name, k)


def test_golden_tolerances_hold_against_each_other(golden):
    # the reference's own degeneration property (test_kernels.cpp:93-104)
    case = golden["simplicial_attention"]
    xs = case_inputs(case)
    ones = np.ones((32, 16), np.float32)
    o1, _ = oracle.oracle_simplicial_attention(xs["q"], ones, ones, xs["k2"], xs["v2"], 1, 16,
                                               0.25)
    o2 = oracle.oracle_attention(xs["q"], xs["k2"], xs["v2"], 16, 0.25)
    assert oracle.rel_error(o1, o2) <= 1e-4


def test_random_tile_deterministic_and_bounded():
    a, b, c = oracle.random_tile([64], 9), oracle.random_tile([64], 9), oracle.random_tile([64], 10)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.all(np.abs(a) <= 1.0)


def test_rel_error_matches_reference_definition():
    a = np.array([1.0, 2.0, 3.0], np.float32)
    b = np.array([1.0, 2.5, 2.0], np.float32)
    assert oracle.rel_error(a, b) == pytest.approx(1.0 / 2.5)
    assert oracle.rel_error(np.zeros(3, np.float32), np.zeros(3, np.float32)) == 0.0
    assert oracle.rel_error(a, b[:2]) == float("inf")


def test_round_bf16_matches_torch():
    torch = pytest.importorskip("torch")
    x = oracle.random_tile([4096], 123) * 37.0
    x[:4] = [0.0, -0.0, 1e-40, 3.0e38]
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(oracle.round_bf16(x).view(np.uint32), want.view(np.uint32))


def test_e4m3_decode_matches_torch():
    torch = pytest.importorskip("torch")
    codes = np.arange(256, dtype=np.uint8)
    sf = np.full((1, 8), 127, np.uint8)
    got = oracle.mx_dequant(codes.reshape(1, 256), sf).ravel()
    want = torch.from_numpy(codes).view(torch.float8_e4m3fn).float().numpy()
    finite = np.isfinite(want)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(got[finite], want[finite])


def test_row_sampled_gemm_is_exact():
    a = oracle.round_bf16(oracle.random_tile([96, 80], 3))
    b = oracle.round_bf16(oracle.random_tile([80, 40], 4))
    full = oracle.oracle_gemm(a, b)
    part = oracle.oracle_gemm(a, b, rows=(17, 53))
    assert np.array_equal(full[17:53], part)


ref = pytest.mark.skipif(oracle.REF is None, reason="oracle/_ref not built (needs /root/reference)")


@ref
@pytest.mark.parametrize("shape,seed", [([7, 13], 1), ([1000], 2), ([3, 5, 8], 1234567)])
def test_random_tile_live_vs_reference(shape, seed):
    import ctypes
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    oracle.REF.ref_random_tile((ctypes.c_int64 * len(shape))(*shape), len(shape), seed, out)
    assert np.array_equal(out.reshape(shape), oracle.random_tile(shape, seed))


@ref
@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (33, 17, 9), (128, 96, 64)])
def test_gemm_live_vs_reference(m, k, n):
    a = oracle.random_tile([m, k], m * 7 + 1)
    b = oracle.random_tile([k, n], n * 5 + 2)
    want = np.empty((m, n), np.float32)
    oracle.REF.ref_oracle_gemm(a, b, want, m, n, k)
    assert np.array_equal(oracle.oracle_gemm(a, b).view(np.uint32), want.view(np.uint32))
    mt = np.empty((m, n), np.float32)
    oracle.REF.ref_oracle_gemm_mt(a, b, mt, m, n, k, 3)
    assert np.array_equal(mt, want)


@ref
@pytest.mark.parametrize("s,d,w", [(1, 8, 1), (40, 16, 40), (64, 32, 7)])
def test_attention_live_vs_reference(s, d, w):
    q, k, v = (oracle.random_tile([s, d], 100 + i) for i in range(3))
    want = np.empty((s, d), np.float32)
    oracle.REF.ref_oracle_attention(q, k, v, want, s, d, w, 0.3)
    assert oracle.rel_error(oracle.oracle_attention(q, k, v, w, 0.3), want) <= 1e-6


def test_attention_rows_matches_full():
    q, k, v = (oracle.random_tile([70, 24], 200 + i) for i in range(3))
    o, lse = oracle.oracle_attention(q, k, v, 30, 0.2, with_lse=True)
    orow, lrow = oracle.oracle_attention_rows(q, k, v, 30, 0.2, 33, 61)
    assert np.array_equal(orow, o[33:61]) and np.array_equal(lrow, lse[33:61])


# ---------------------------------------------------------------------------
# restated oracles without a reference counterpart:
# pinned against torch float64 autograd instead
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("causal,w", [(False, None), (True, None), (True, 7)])
def test_attention_bwd_oracle_matches_torch_f64(causal, w):
    import torch
    s, d, scale = 37, 16, 0.3
    q, k, v, do = (oracle.random_tile([s, d], 900 + i) for i in range(4))
    Q, K, V = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    S = (Q @ K.T) * scale
    if causal:
        i = torch.arange(s)
        ww = w if w is not None else s
        bad = (i[None, :] > i[:, None]) | (i[:, None] - i[None, :] >= ww)
        S = S.masked_fill(bad, -float("inf"))
    O = torch.softmax(S, -1) @ V
    want = torch.autograd.grad(O, (Q, K, V), torch.tensor(do, dtype=torch.float64))
    got = oracle.oracle_attention_bwd(q, k, v, do, scale, causal=causal, w=w)
    for g, t in zip(got, want):
        np.testing.assert_allclose(g, t.numpy(), rtol=1e-5, atol=1e-6)
    if not causal:
        o, lse = oracle.oracle_attention_full(q, k, v, scale)
        np.testing.assert_allclose(o, O.detach().numpy(), rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(lse, torch.logsumexp(S, -1).detach().numpy(), rtol=1e-5)
    else:
        # the causal mode of the restatement is the reference's oracle_attention
        o_ref = oracle.oracle_attention(q, k, v, w if w is not None else s, scale)
        np.testing.assert_allclose(o_ref, O.detach().numpy(), rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------------------
# config-scale checkers, pinned to the unmodified reference
# ---------------------------------------------------------------------------
@ref
@pytest.mark.parametrize("r,k,n,threads", [(1, 1, 1, 1), (37, 300, 200, 3), (17, 1000, 1030, 8)])
def test_gemm_rowlist_bit_exact_vs_reference(r, k, n, threads):
    """The threaded k-outer restatement used by the config-scale tests gives
    the reference's float sums bit for bit (oracles.cpp:17-23)."""
    a = oracle.random_tile([r, k], 31 * r + k)
    b = oracle.round_bf16(oracle.random_tile([k, n], 7 * n + 1))
    want = np.empty((r, n), np.float32)
    oracle.REF.ref_oracle_gemm(a, b, want, r, n, k)
    got = oracle.oracle_gemm_rowlist(a, b, threads=threads)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_attention_rowlist_matches_rows():
    q, k, v = (oracle.random_tile([300, 64], 40 + i) for i in range(3))
    rows = [299, 0, 150, 7, 128]
    o, lse = oracle.oracle_attention_rowlist(q, k, v, 100, 0.125, rows, threads=3)
    for i, r in enumerate(rows):
        want, wl = oracle.oracle_attention_rows(q, k, v, 100, 0.125, r, r + 1)
        assert np.array_equal(o[i], want[0]) and lse[i] == wl[0]


@ref
@pytest.mark.parametrize("s,d,w1,w2", [(32, 16, 2, 16), (50, 8, 5, 50), (40, 12, 40, 3)])
def test_simplicial_rows_vs_reference(s, d, w1, w2):
    """oracle.oracle_simplicial_rows (the f64 numpy checker of every device
    simplicial test) against the unmodified oracle_simplicial_attention
    (oracles.cpp:82-117) through oracle/_ref: every row, o at 1e-5 (the
    reference accumulates o in f32), lse at 1e-6."""
    xs = [oracle.random_tile([s, d], oracle.input_seed(31 + s, i)) for i in range(5)]
    want_o = np.empty((s, d), np.float32)
    want_l = np.empty(s, np.float32)
    oracle.REF.ref_oracle_simplicial_attention(*xs, want_o, want_l, s, d, w1, w2, 0.25)
    got_o, got_l = oracle.oracle_simplicial_rows(*xs, w1, w2, 0.25, list(range(s)))
    assert oracle.rel_error(got_o, want_o) <= 1e-5
    assert oracle.rel_error_rows(got_o, want_o) <= 1e-5
    np.testing.assert_allclose(got_l, want_l, rtol=1e-6, atol=1e-6)
    # and the C restatement (the full-oracle checker) bit for bit in lse, f32-close in o
    c_o, c_l = oracle.oracle_simplicial_attention(*xs, w1, w2, 0.25)
    assert oracle.rel_error(c_o, want_o) <= 1e-6
    assert np.array_equal(c_l, want_l)


def _ref_attention(q, k, v, w, scale):
    s, d = q.shape
    out = np.empty((s, d), np.float32)
    oracle.REF.ref_oracle_attention(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(k, np.float32),
                                    np.ascontiguousarray(v, np.float32), out, s, d, w, scale)
    return out


def _ref_noncausal(q, k, v, scale):
    """Non-causal attention from the REFERENCE's causal oracle_attention by the
    last-row trick: with w >= S, row S-1 attends every key, so putting query i
    in the last row gives non-causal row i (oracles.cpp:123-126)."""
    s, d = q.shape
    out = np.empty((s, d), np.float32)
    for i in range(s):
        qi = q.copy()
        qi[s - 1] = q[i]
        out[i] = _ref_attention(qi, k, v, s, scale)[s - 1]
    return out


@ref
@pytest.mark.parametrize("s,d", [(1, 8), (33, 16), (64, 32)])
def test_noncausal_rows_pinned_to_reference(s, d):
    """orc_attention_mode_rows(causal=0) (the checker of every non-causal
    device test) equals the reference's own oracle row bit for bit."""
    q, k, v = (oracle.random_tile([s, d], 500 + s + i) for i in range(3))
    got, _ = oracle.oracle_attention_full(q, k, v, 0.3)
    want = _ref_noncausal(q, k, v, 0.3)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@ref
@pytest.mark.parametrize("causal,w", [(True, None), (True, 9), (False, None)])
def test_attention_bwd_pinned_to_reference_finite_differences(causal, w):
    """orc_attention_bwd (the f64 checker of the device backward) against
    central differences of the REFERENCE's oracle_attention (through _ref; the
    non-causal forward by the last-row trick): for L = <dO, O(q, k, v)>,
    <dX, delta> ~= (L(X + eps delta) - L(X - eps delta)) / (2 eps) for random
    directions delta in q, k and v."""
    s, d, scale, eps = 24, 16, 0.3, 1e-2
    rng = np.random.default_rng(17 + int(causal) + (w or 0))
    q, k, v, do = (oracle.random_tile([s, d], 700 + i).astype(np.float64) for i in range(4))
    ww = w if w is not None else s

    def fwd(q_, k_, v_):
        if causal:
            return _ref_attention(q_, k_, v_, ww, scale).astype(np.float64)
        return _ref_noncausal(q_.astype(np.float32), k_.astype(np.float32), v_.astype(np.float32),
                              scale).astype(np.float64)

    grads = oracle.oracle_attention_bwd(q, k, v, do, scale, causal=causal, w=w)
    for which in range(3):
        for _ in range(3):
            delta = rng.standard_normal((s, d))
            args_p = [q, k, v]
            args_m = [q, k, v]
            args_p = [x + eps * delta if i == which else x for i, x in enumerate(args_p)]
            args_m = [x - eps * delta if i == which else x for i, x in enumerate(args_m)]
            fd = (np.sum(do * fwd(*args_p)) - np.sum(do * fwd(*args_m))) / (2 * eps)
            an = float(np.sum(grads[which].astype(np.float64) * delta))
            assert abs(fd - an) <= 5e-4 * max(1.0, abs(an)), (which, fd, an)  # measured ~1e-5
