"""GPU parity: 2-simplicial attention forward vs
oracle_simplicial_attention (oracles.cpp:82-117).

Tolerance: the kernel computes in bf16 with fp32 accumulation (north_star
"bf16 within rel-err 1e-2"), so bf16-rounded inputs are compared at 1e-2
(reference rel_error, case.cpp:94-104) whole-tensor and per row; the
reference case's own 1e-3 is an f32 tolerance."""
import numpy as np
import pytest

import oracle
from golden_util import case_inputs, case_outputs

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def test_reference_case_through_reference_signature(P, golden):
    case = golden["simplicial_attention"]
    xs = case_inputs(case)
    sc = case["scalars"]
    want = case_outputs(case)
    o, lse = P.oracle_simplicial_attention(xs["q"], xs["k1"], xs["v1"], xs["k2"], xs["v2"],
                                           int(sc["w1"]), int(sc["w2"]), sc["scale"])
    assert oracle.rel_error(o, want["o"]) <= TOL
    assert oracle.rel_error(lse, want["lse"]) <= TOL
    out = P.run_oracle("simplicial_attention", xs, sc)
    assert oracle.rel_error(out["o"], want["o"]) <= TOL


def test_degenerates_to_attention(P):
    """w1 = 1, k1 = v1 = 1: plain windowed causal attention (the reference's
    own degeneration check, acceptance.cpp:333-355 / test_kernels.cpp:93-104)."""
    s, d = 200, 64
    q, k, v = (oracle.round_bf16(oracle.random_tile([s, d], oracle.input_seed(31, i))) for i in range(3))
    one = np.ones((s, d), np.float32)
    o, lse = P.oracle_simplicial_attention(q, one, one, k, v, 1, 77, 0.125)
    want, wl = oracle.oracle_attention(q, k, v, 77, 0.125, with_lse=True)
    assert oracle.rel_error(o, want) <= TOL and oracle.rel_error_rows(o, want) <= TOL
    assert oracle.rel_error(lse, wl) <= TOL


def _dev_case(bh, s, seed):
    import torch
    xs = [oracle.round_bf16(oracle.random_tile([bh, s, 128], oracle.input_seed(seed, i)))
          for i in range(5)]
    return xs, [torch.from_numpy(x).cuda().bfloat16() for x in xs]


@pytest.mark.parametrize("s,w1,w2", [(128, 1, 128), (300, 3, 200), (300, 8, 16), (1000, 16, 300),
                                     (130, 40, 1000)])
def test_device_vs_oracle(P, s, w1, w2):
    import torch
    bh = 2
    xs, ts = _dev_case(bh, s, s + w1 + w2)
    scale = 128 ** -0.5
    o, lse = P.simplicial_attention_fwd(*ts, w1=w1, w2=w2, scale=scale)
    torch.cuda.synchronize()
    o = o.float().cpu().numpy()
    lse = lse.cpu().numpy()
    for b in range(bh):
        rows = sorted({0, 1, s // 3, s // 2, s - 2, s - 1} | set(range(0, s, max(1, s // 16))))
        wo, wl = oracle.oracle_simplicial_rows(*(x[b] for x in xs), w1, w2, scale, rows)
        assert oracle.rel_error(o[b][rows], wo) <= TOL, b
        assert oracle.rel_error_rows(o[b][rows], wo) <= 2 * TOL, b
        assert np.max(np.abs(lse[b][rows] - wl)) <= 1e-2 * max(1.0, np.max(np.abs(wl)))


def test_device_full_oracle_small(P):
    """Every row of a small case against the C restatement of the oracle."""
    import torch
    s, w1, w2 = 256, 4, 100
    xs, ts = _dev_case(1, s, 5)
    o, lse = P.simplicial_attention_fwd(*ts, w1=w1, w2=w2, scale=0.1)
    torch.cuda.synchronize()
    wo, wl = oracle.oracle_simplicial_attention(*(x[0] for x in xs), w1, w2, 0.1)
    assert oracle.rel_error(o[0].float().cpu().numpy(), wo) <= TOL
    assert oracle.rel_error(lse[0].cpu().numpy(), wl) <= TOL


def test_reference_precision_case(P, golden):
    """MIMW_PREC_F32: the reference case at its own 1e-3 (simplicial_attention.case)."""
    case = golden["simplicial_attention"]
    xs = case_inputs(case)
    sc = case["scalars"]
    o, lse = P.oracle_simplicial_attention(xs["q"], xs["k1"], xs["v1"], xs["k2"], xs["v2"],
                                           int(sc["w1"]), int(sc["w2"]), sc["scale"],
                                           precision=P.PREC_F32)
    outs = case_outputs(case)
    assert oracle.rel_error(o, outs["o"]) <= case["tolerance"]
    assert oracle.rel_error(lse, outs["lse"]) <= case["tolerance"]
    out = P.run_oracle("simplicial_attention", xs, sc, precision=P.PREC_F32)
    assert oracle.rel_error(out["o"], outs["o"]) <= case["tolerance"]
