"""GPU parity: cluster LayerNorm vs oracle_layernorm
(oracles.cpp:28-55, restated in oracle/oracle.c orc_layernorm).  Tolerance:
the reference case's own 1e-5 (kernels/layernorm_cluster.case:6)."""
import numpy as np
import pytest

import oracle
from golden_util import case_inputs, case_outputs

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def test_reference_case_through_reference_signature(P, golden):
    case = golden["layernorm_cluster"]
    xs = case_inputs(case)
    want = case_outputs(case)["y"]
    y, mean, rstd = P.oracle_layernorm(xs["x"], xs["w"], xs["b"], case["scalars"]["eps"])
    assert oracle.rel_error(y, want) <= case["tolerance"]
    ry, rm, rr = oracle.oracle_layernorm(xs["x"], xs["w"], xs["b"], case["scalars"]["eps"])
    assert oracle.rel_error(mean, rm) <= TOL and oracle.rel_error(rstd, rr) <= TOL
    out = P.run_oracle("layernorm", xs, case["scalars"])
    assert oracle.rel_error(out["y"], want) <= case["tolerance"]


@pytest.mark.parametrize("rows,n", [(1, 1), (3, 7), (4, 1024), (5, 1000), (2, 4099), (7, 65536),
                                    (2, 262144), (300, 2048)])
@pytest.mark.parametrize("cluster", [0, 1, 4, 16])
def test_device_layernorm_vs_oracle(P, rows, n, cluster):
    import torch
    if cluster and (n + cluster - 1) // cluster > 16384:
        pytest.skip("cluster size does not fit this row length")
    rng = np.random.default_rng(rows * 7 + n)
    x = (rng.standard_normal((rows, n)) * 3 + 1.5).astype(np.float32)
    w = rng.standard_normal(n).astype(np.float32)
    b = rng.standard_normal(n).astype(np.float32)
    tx, tw, tb = (torch.from_numpy(a).cuda() for a in (x, w, b))
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    y = P.layernorm(tx, tw, tb, 1e-5, mean=mean, rstd=rstd, cluster=cluster)
    torch.cuda.synchronize()
    ry, rm, rr = oracle.oracle_layernorm(x, w, b, 1e-5)
    assert oracle.rel_error(y.cpu().numpy(), ry) <= TOL
    assert oracle.rel_error(mean.cpu().numpy(), rm) <= TOL
    assert oracle.rel_error(rstd.cpu().numpy(), rr) <= TOL


def test_layernorm_paper_shape_ln6_sampled(P):
    """PAPER.md:736 LN6 (1152 x 65536): sampled rows vs the oracle plus
    per-row mean 0 / variance 1 of the normalised output (w=1, b=0)."""
    import torch
    rows, n = 1152, 65536
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((rows, n), device="cuda", generator=g) * 2 + 0.5
    w = torch.ones(n, device="cuda")
    b = torch.zeros(n, device="cuda")
    y = P.layernorm(x, w, b, 1e-5)
    torch.cuda.synchronize()
    idx = [0, 1, 577, 1151]
    ry, _, _ = oracle.oracle_layernorm(x[idx].cpu().numpy(), w.cpu().numpy(), b.cpu().numpy(), 1e-5)
    assert oracle.rel_error(y[idx].cpu().numpy(), ry) <= TOL
    yd = y.double()
    assert yd.mean(dim=1).abs().max().item() < 1e-5
    assert (yd.var(dim=1, unbiased=False) - 1).abs().max().item() < 1e-4
