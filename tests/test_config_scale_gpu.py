"""Config-scale parity: EVERY work item of the BASELINE configs checked
against the oracle.

The schedulers hand out work per output tile (GEMM: cluster launch control
over 256x256 tiles; grouped MoE: per-expert tiles + swapped tails) or per item
(FA: a head's 256-row query block, band-LPT order).  A scheduler or tail bug
hits whole tiles / items, so each test samples rows such that every tile (both
CTAs of each pair, i.e. both 128-row halves) / every item is covered, and
compares every 256-column segment of those rows with the oracle:

* configs[1] 8192^3 bf16 GEMM: 2 rows per 256-row M tile (one per CTA of the
  pair) x all 8192 columns = every one of the 1024 output tiles;
* configs[3] causal FA B4 H32 S8192 D128: one row per (head, 256-row block) =
  4096 rows, alternating between the item's two 128-row Q tiles;
* configs[4] grouped MoE 64 x 4096 x 14336, Dirichlet routing: 1-2 rows per
  256-row tile of every non-empty expert (incl. each swapped tail tile);
* the 2-simplicial bench shape BH16 S8192 w1=32 w2=512: 8 rows per head.

Oracles: oracle_gemm rows (oracles.cpp:14-26, exact per row; the threaded
restatement is pinned bit-exact to oracle/_ref in test_oracle.py), oracle
attention rows (oracles.cpp:119-145), oracle_simplicial rows (oracles.cpp:
82-117, pinned to _ref in test_oracle.py).  Tolerance: bf16 1e-2 (north
star) per row and per 256-column segment of a row.
"""
import numpy as np
import pytest

import oracle

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


def _segments_ok(got, want, seg=256, tol=TOL):
    """rel_error of every (row, seg-column block), normalised by that row's
    max |want| (the per-row metric restricted to one output tile's columns)."""
    bad = []
    for r in range(want.shape[0]):
        scale = max(float(np.max(np.abs(want[r]))), 1e-30)
        for c0 in range(0, want.shape[1], seg):
            e = float(np.max(np.abs(got[r, c0:c0 + seg] - want[r, c0:c0 + seg]))) / scale
            if not np.isfinite(e) or e > tol:
                bad.append((r, c0, e))
    return bad


def test_gemm_configs1_every_tile(P):
    import torch
    m = n = k = 8192
    g = torch.Generator(device="cuda").manual_seed(7)
    ta = (torch.rand((m, k), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    tb = (torch.rand((k, n), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c = P.gemm(ta, tb)  # bf16 out, the bench's configuration
    torch.cuda.synchronize()
    rows = []
    for t in range(m // 256):
        rows += [256 * t + (37 * t) % 128, 256 * t + 128 + (59 * t) % 128]
    a = ta[rows].float().cpu().numpy()
    b = tb.float().cpu().numpy()
    want = oracle.oracle_gemm_rowlist(a, b)
    got = c[rows].float().cpu().numpy()
    assert np.isfinite(got).all()
    assert oracle.rel_error_rows(got, want) <= TOL
    bad = _segments_ok(got, want)
    assert not bad, bad[:10]


def test_attention_configs3_every_item(P):
    import torch
    b, h, s, d = 4, 32, 8192, 128
    g = torch.Generator(device="cuda").manual_seed(31)
    q, k, v = ((torch.rand((b, h, s, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
               for _ in range(3))
    o, lse = P.attention_fwd(q, k, v)
    torch.cuda.synchronize()
    scale = d ** -0.5
    nqb = s // 256
    o = o.reshape(b * h, s, d)
    lse = lse.reshape(b * h, s)
    q, k, v = (t.reshape(b * h, s, d) for t in (q, k, v))
    worst, worst_l = 0.0, 0.0
    for bh in range(b * h):
        rows = np.array([256 * qb + (37 * qb + 11 * bh) % 256 for qb in range(nqb)], np.int64)
        qh, kh, vh = (t[bh].float().cpu().numpy() for t in (q, k, v))
        want, wl = oracle.oracle_attention_rowlist(qh, kh, vh, s, scale, rows)
        got = o[bh][torch.from_numpy(rows).cuda()].float().cpu().numpy()
        gl = lse[bh][torch.from_numpy(rows).cuda()].cpu().numpy()
        e = oracle.rel_error_rows(got, want)
        el = float(np.max(np.abs(gl - wl) / np.maximum(1.0, np.abs(wl))))
        assert e <= TOL, (bh, e)
        assert el <= 1e-3, (bh, el)
        worst, worst_l = max(worst, e), max(worst_l, el)
    print(f"configs[3] 4096 item rows: worst per-row rel {worst:.2e}, worst lse {worst_l:.2e}")


def _moe_counts(seed=5, experts=64, rows=32768):
    """bench.py moe_counts: Dirichlet(1) expert probabilities, multinomial
    assignment of tokens * top_k rows."""
    rng = np.random.default_rng(seed)
    p = rng.dirichlet(np.ones(experts))
    return rng.multinomial(rows, p)


def test_grouped_moe_configs4_every_tile(P):
    import torch
    E, K, N = 64, 4096, 14336
    counts = _moe_counts()
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    g = torch.Generator(device="cuda").manual_seed(5)
    w = torch.empty((E, K, N), device="cuda", dtype=torch.bfloat16)
    for e in range(E):
        w[e] = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
    x = (torch.rand((int(offs[-1]), K), device="cuda", generator=g) * 2 - 1).bfloat16()
    y = P.grouped_gemm(x, offs, w)
    torch.cuda.synchronize()
    checked = 0
    for e in range(E):
        m = int(counts[e])
        if m == 0:
            continue
        local = []
        for t in range((m + 255) // 256):
            span = min(256, m - 256 * t)
            local.append(256 * t + (37 * t + 13 * e) % min(128, span))
            if span > 128:
                local.append(256 * t + 128 + (59 * t + 7 * e) % (span - 128))
        rows = [int(offs[e]) + r for r in local]
        idx = torch.tensor(rows, device="cuda")
        a = x[idx].float().cpu().numpy()
        want = oracle.oracle_gemm_rowlist(a, w[e].float().cpu().numpy())
        got = y[idx].float().cpu().numpy()
        assert np.isfinite(got).all(), e
        assert oracle.rel_error_rows(got, want) <= TOL, e
        bad = _segments_ok(got, want)
        assert not bad, (e, bad[:5])
        checked += len(rows)
    # rows outside every group are never written (none here: offs[-1] == rows)
    assert checked >= int(np.sum((counts + 255) // 256))


def test_simplicial_bench_config(P):
    """BH16 S8192 w1=32 w2=512 (bench.py's §8f rank 2 line), 8 rows per head
    incl. the window edges, against the oracle rows."""
    import torch
    bh, s, w1, w2 = 16, 8192, 32, 512
    g = torch.Generator(device="cuda").manual_seed(31)
    ts = [((torch.rand((bh, s, 128), device="cuda", generator=g) * 2 - 1).bfloat16()) for _ in range(5)]
    scale = 128 ** -0.5
    o, lse = P.simplicial_attention_fwd(*ts, w1=w1, w2=w2, scale=scale)
    torch.cuda.synchronize()
    for hh in range(bh):
        rows = sorted({0, 31, 32, 511, 512, 8191, (977 * hh + 100) % s, (3001 * hh + 4000) % s})
        xs = [t[hh].float().cpu().numpy() for t in ts]
        wo, wl = oracle.oracle_simplicial_rows(*xs, w1, w2, scale, rows)
        got = o[hh][rows].float().cpu().numpy()
        gl = lse[hh][rows].cpu().numpy()
        assert oracle.rel_error_rows(got, wo) <= TOL, hh
        assert np.max(np.abs(gl - wl)) <= 1e-2 * max(1.0, float(np.max(np.abs(wl)))), hh
