"""GPU parity: block-scaled FP8 (MXFP8) GEMM vs oracle_gemm on the dequantised
inputs (the reference has no FP8; oracle semantics defined in
SURVEY.md §8a row a14).  Tolerance (north_star "fp8 within a stated looser
tolerance"): rel_error <= 2e-2 against the dequantised
oracle; in practice only the bf16 rounding of C remains (~4e-3)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def _mx_operand(rows, k, seed):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 256, size=(rows, k), dtype=np.uint8)
    q[(q & 0x7F) == 0x7F] = 0x38  # no NaN codes
    sf = rng.integers(118, 136, size=(rows, k // 32), dtype=np.uint8)
    return q, sf


@pytest.mark.parametrize("m,n,k", [(128, 224, 128), (256, 448, 512), (300, 504, 1056), (1, 8, 32),
                                   (1024, 1024, 1024), (520, 8192, 160)])
@pytest.mark.parametrize("cta_group", [1, 2, 3])  # 3: 2-CTA, 256 x 448 tiles
def test_mxfp8_vs_dequant_oracle(P, m, n, k, cta_group):
    import torch
    qa, sfa = _mx_operand(m, k, m + k)
    qb, sfb = _mx_operand(n, k, n + 3 * k)
    ta, tb = torch.from_numpy(qa).cuda(), torch.from_numpy(qb).cuda()
    tsa, tsb = torch.from_numpy(sfa).cuda(), torch.from_numpy(sfb).cuda()
    c = P.gemm_mxfp8(ta.view(torch.float8_e4m3fn), tsa, tb.view(torch.float8_e4m3fn), tsb,
                     cta_group=cta_group)
    torch.cuda.synchronize()
    got = c.float().cpu().numpy()
    assert np.isfinite(got).all()
    a = oracle.mx_dequant(qa, sfa)
    b = oracle.mx_dequant(qb, sfb)
    want = oracle.oracle_gemm(a, np.ascontiguousarray(b.T))
    assert oracle.rel_error(got, want) <= TOL
    assert oracle.rel_error_rows(got, want) <= TOL


@pytest.mark.parametrize("cta_group", [2, 3])
def test_mxfp8_8192_sampled_rows(P, cta_group):
    """configs[2] size (8192^3): row-sampled exact oracle on dequantised inputs
    (cta_group 3: 256 x 448 tiles, whose last column tile is 128 wide)."""
    import torch
    m = n = k = 8192
    g = torch.Generator(device="cuda").manual_seed(3)
    qa = torch.randint(0, 256, (m, k), device="cuda", dtype=torch.uint8, generator=g)
    qb = torch.randint(0, 256, (n, k), device="cuda", dtype=torch.uint8, generator=g)
    qa[(qa & 0x7F) == 0x7F] = 0x38
    qb[(qb & 0x7F) == 0x7F] = 0x38
    sfa = torch.randint(120, 134, (m, k // 32), device="cuda", dtype=torch.uint8, generator=g)
    sfb = torch.randint(120, 134, (n, k // 32), device="cuda", dtype=torch.uint8, generator=g)
    c = P.gemm_mxfp8(qa.view(torch.float8_e4m3fn), sfa, qb.view(torch.float8_e4m3fn), sfb, cta_group=cta_group)
    torch.cuda.synchronize()
    rows = [0, 127, 128, 4097, 8191]
    a = oracle.mx_dequant(qa[rows].cpu().numpy(), sfa[rows].cpu().numpy())
    b = oracle.mx_dequant(qb.cpu().numpy(), sfb.cpu().numpy())
    want = oracle.oracle_gemm(a, np.ascontiguousarray(b.T))
    got = c[rows].float().cpu().numpy()
    assert oracle.rel_error(got, want) <= TOL
