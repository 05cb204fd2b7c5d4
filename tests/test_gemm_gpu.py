"""GPU parity: the sm_100a persistent warp-specialized GEMM vs the oracle.

Tolerances (metric = reference rel_error, case.cpp:94-104):
  * bf16 inputs, fp32 accumulate            rel_error <= 1e-2  (north_star)
  * reference f32 cases via MIMW_PREC_F32_BF16X3  <= the case's own 1e-4
"""
import numpy as np
import pytest

import oracle
from golden_util import case_inputs, case_outputs

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


@pytest.mark.parametrize("name", ["gemm_pipeline", "gemm_clc", "collective_dot"])
def test_reference_f32_cases_at_reference_tolerance(P, golden, name):
    case = golden[name]
    xs = case_inputs(case)
    want = case_outputs(case)["c"]
    got = P.oracle_gemm(xs["a"], xs["b"], precision=P.PREC_F32_BF16X3)
    assert oracle.rel_error(got, want) <= case["tolerance"]  # 1e-4
    got16 = P.oracle_gemm(xs["a"], xs["b"])  # bf16 rounding: north-star tolerance
    assert oracle.rel_error(got16, want) <= BF16_TOL


def test_multi_device_gemm_case(P, golden):
    case = golden["multi_device_gemm"]
    xs = case_inputs(case)
    want = case_outputs(case)["c"]
    got = P.oracle_multi_device_gemm(xs["a0"], xs["a1"], xs["b0"], xs["b1"],
                                     precision=P.PREC_F32_BF16X3)
    assert oracle.rel_error(got, want) <= case["tolerance"]


@pytest.mark.parametrize("name", ["gemm_bf16_256x320x384", "gemm_bf16_ragged_200x136x72"])
def test_bf16_golden(P, golden, name):
    case = golden[name]
    xs = case_inputs(case)
    want = case_outputs(case)["c"]
    got = P.oracle_gemm(xs["a"], xs["b"])
    assert oracle.rel_error(got, want) <= BF16_TOL
    assert oracle.rel_error_rows(got, want) <= BF16_TOL


def _dev_case(m, k, n, seed):
    import torch
    a = oracle.round_bf16(oracle.random_tile([m, k], oracle.input_seed(seed, 0)))
    b = oracle.round_bf16(oracle.random_tile([k, n], oracle.input_seed(seed, 1)))
    ta = torch.from_numpy(a).cuda().to(torch.bfloat16)
    tb = torch.from_numpy(b).cuda().to(torch.bfloat16)
    return a, b, ta, tb


@pytest.mark.parametrize("cta_group", [1, 2, 4])
@pytest.mark.parametrize("b_layout", ["kn", "nk"])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_device_gemm_1024_full_oracle(P, cta_group, b_layout, out):
    """configs[0]: bf16 GEMM 1024^3 fp32 accumulate against the full oracle."""
    import torch
    a, b, ta, tb = _dev_case(1024, 1024, 1024, 7)
    want = _full_oracle_1024(a, b)
    bl = P.B_KN if b_layout == "kn" else P.B_NK
    tbb = tb if b_layout == "kn" else tb.t().contiguous()
    c = P.gemm(ta, tbb, b_layout=bl, cta_group=cta_group,
               out_dtype=torch.float32 if out == "f32" else torch.bfloat16)
    torch.cuda.synchronize()
    got = c.float().cpu().numpy()
    assert np.isfinite(got).all()
    tol = BF16_TOL
    assert oracle.rel_error(got, want) <= tol
    assert oracle.rel_error_rows(got, want) <= tol
    if out == "f32":
        # fp32 accumulate of exact bf16 products: far tighter than the bf16 budget
        assert oracle.rel_error(got, want) <= 1e-5


_CACHE = {}


def _full_oracle_1024(a, b):
    if "c" not in _CACHE:
        _CACHE["c"] = oracle.oracle_gemm(a, b)
    return _CACHE["c"]


@pytest.mark.parametrize("m,k,n", [(1, 8, 8), (130, 72, 264), (384, 1000, 520), (257, 4104, 136),
                                   (2048, 64, 2048)])
@pytest.mark.parametrize("cta_group", [1, 2, 4])
def test_device_gemm_ragged(P, m, k, n, cta_group):
    import torch
    a, b, ta, tb = _dev_case(m, k, n, m + n + k)
    want = oracle.oracle_gemm(a, b)
    got = P.gemm(ta, tb, out_dtype=torch.float32, cta_group=cta_group).cpu().numpy()
    assert oracle.rel_error(got, want) <= 1e-5


@pytest.mark.parametrize("b_layout", ["kn", "nk"])
@pytest.mark.parametrize("m,k,n", [(1024, 1024, 1024), (1, 8, 8), (130, 72, 264), (300, 136, 1000),
                                   (257, 4104, 600), (513, 64, 1544), (2048, 192, 2056)])
def test_device_gemm_wide_tiles(P, b_layout, m, k, n):
    """256 x 512 pair tiles (gemm_wide.cuh): vs the oracle at the bf16 budget,
    and bit-identical to the 256 x 256 kernel (same fp32 K order per element)."""
    import torch
    a, b, ta, tb = _dev_case(m, k, n, 3 * m + n + k)
    want = oracle.oracle_gemm(a, b)
    bl = P.B_KN if b_layout == "kn" else P.B_NK
    tbb = tb if b_layout == "kn" else tb.t().contiguous()
    guard = torch.full((m + 1, n), 3.0, device="cuda", dtype=torch.bfloat16)  # row m: must stay untouched
    wide = P.gemm(ta, tbb, b_layout=bl, tile_n=512, out=guard[:m])
    narrow = P.gemm(ta, tbb, b_layout=bl, tile_n=256)
    torch.cuda.synchronize()
    got = wide.float().cpu().numpy()
    assert oracle.rel_error(got, want) <= BF16_TOL
    assert oracle.rel_error_rows(got, want) <= BF16_TOL
    assert torch.equal(wide, narrow)
    assert torch.all(guard[m] == 3.0)


def test_device_gemm_8192_sampled_rows(P):
    """configs[1] size: 8192^3 bf16, row-sampled exact oracle."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    ta = (torch.rand((8192, 8192), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    tb = (torch.rand((8192, 8192), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c = P.gemm(ta, tb)
    torch.cuda.synchronize()
    rows = [0, 1, 255, 256, 4095, 5000, 8191]
    a = ta[rows].float().cpu().numpy()
    b = tb.float().cpu().numpy()
    want = oracle.oracle_gemm(a, b)
    got = c[rows].float().cpu().numpy()
    assert oracle.rel_error(got, want) <= BF16_TOL
    # whole-tensor property: column sums == (1^T A) B  (linearity)
    ones = torch.ones((1, 8192), device="cuda", dtype=torch.float32)
    lhs = (ones @ c.float()).double()
    rhs = ((ones @ ta.float()).double() @ tb.double())
    assert torch.max(torch.abs(lhs - rhs)) / torch.max(torch.abs(rhs)) < 1e-2


def test_k_zero_gives_zeros(P):
    import torch
    ta = torch.zeros((64, 0), device="cuda", dtype=torch.bfloat16)
    tb = torch.zeros((0, 64), device="cuda", dtype=torch.bfloat16)
    out = torch.full((64, 64), 7.0, device="cuda")
    P.gemm(ta, tb, out=out)
    assert torch.count_nonzero(out).item() == 0


@pytest.mark.parametrize("m,k,n", [(2000, 300, 264), (1537, 72, 40)])
def test_host_path_pipelined_chunks(P, m, k, n):
    """The host-f32 entry pipelines row chunks of 512+ rows over three
    streams; results equal the oracle in both precisions."""
    a = oracle.random_tile([m, k], oracle.input_seed(3, 0))
    b = oracle.random_tile([k, n], oracle.input_seed(3, 1))
    want = oracle.oracle_gemm(a, b)
    assert oracle.rel_error(P.oracle_gemm(a, b, precision=P.PREC_F32_BF16X3), want) <= 1e-4
    assert oracle.rel_error(P.oracle_gemm(a, b), want) <= BF16_TOL
    a1 = oracle.random_tile([m, 40], oracle.input_seed(3, 2))
    b1 = oracle.random_tile([40, n], oracle.input_seed(3, 3))
    want = oracle.oracle_multi_device_gemm(a, a1, b, b1)
    got = P.oracle_multi_device_gemm(a, a1, b, b1, precision=P.PREC_F32_BF16X3)
    assert oracle.rel_error(got, want) <= 1e-4
