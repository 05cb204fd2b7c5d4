"""GPU parity of the all-gather (K-gathered) multi-device GEMM, SURVEY §8f rank 1.

Oracle: oracle_multi_device_gemm (oracles.cpp:57-80) for the reference's own
two-device case (multi_device_gemm.case, seed 23), and oracle_gemm on the
K-concatenated operands for `world` > 2 (the same function the reference's
oracle reduces to, oracles.cpp:79).  Every "device" is emulated on the one
GPU: rank r's kernel pulls the other ranks' splits from their buffers exactly
as it would through IPC-mapped peer pointers over NVLink.  With
``concurrent=True`` the ranks' kernels run side by side on separate streams
and meet in the device-side entry/exit barrier.

Tolerance: bf16 inputs, fp32 accumulation, bf16 output -> rel_error <= 1e-2
(north_star); in practice one bf16 output rounding (<= 2^-8 per element).
"""
import numpy as np
import pytest

import oracle
from golden_util import case_inputs, case_outputs

pytestmark = pytest.mark.gpu

TOL = 1e-2


@pytest.fixture(scope="module")
def MD():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_10905_b200 import multi_device as MD
    MD._lib()
    return MD


def _splits(m, ks, n, seed):
    a = [oracle.round_bf16(oracle.random_tile([m, k], oracle.input_seed(seed, 2 * i)))
         for i, k in enumerate(ks)]
    b = [oracle.round_bf16(oracle.random_tile([k, n], oracle.input_seed(seed, 2 * i + 1)))
         for i, k in enumerate(ks)]
    return a, b


def _dev(xs):
    import torch
    return [torch.from_numpy(x).cuda().bfloat16().contiguous() for x in xs]


def _want(a, b, rows=None):
    return oracle.oracle_gemm(np.concatenate(a, axis=1), np.concatenate(b, axis=0), rows=rows)


def test_reference_two_device_case(MD, golden):
    """multi_device_gemm.case: a0,a1 [64,64], b0,b1 [64,32]; each device owns
    32 rows of c, as the reference program's two clusters (:6-7,21)."""
    import torch
    case = golden["multi_device_gemm"]
    xs = {k: oracle.round_bf16(v) for k, v in case_inputs(case).items()}
    a, b = [xs["a0"], xs["a1"]], [xs["b0"], xs["b1"]]
    for concurrent in (False, True):
        c = MD.emulated_multi_device_gemm(_dev(a), _dev(b), row_ranges=[(0, 32), (32, 64)],
                                          concurrent=concurrent)
        torch.cuda.synchronize()
        got = c.float().cpu().numpy()
        want = oracle.oracle_multi_device_gemm(*a, *b)
        assert oracle.rel_error(got, want) <= 2 ** -8
        # and against the reference's own f32 output (bf16 input rounding on top)
        assert oracle.rel_error(got, case_outputs(case)["c"]) <= TOL


@pytest.mark.parametrize("ks,m,n", [
    ([64, 64], 600, 264),
    ([200, 8, 136], 515, 96),          # ragged K splits (TMA zero-fills each split's tail)
    ([256, 0, 320, 72], 300, 1032),    # an empty split
    ([64] * 8, 1100, 520),             # 8 devices
])
@pytest.mark.parametrize("concurrent", [False, True])
@pytest.mark.parametrize("comm_pairs", [-1, 2])  # comm warps in every GEMM CTA / dedicated comm pairs
def test_ragged_world(MD, ks, m, n, concurrent, comm_pairs):
    import torch
    a, b = _splits(m, ks, n, 101 + len(ks))
    c = MD.emulated_multi_device_gemm(_dev(a), _dev(b), concurrent=concurrent, comm_pairs=comm_pairs)
    torch.cuda.synchronize()
    got = c.float().cpu().numpy()
    want = _want(a, b)
    assert oracle.rel_error(got, want) <= TOL
    assert oracle.rel_error_rows(got, want) <= TOL


def test_uneven_row_ownership(MD):
    """Row blocks that are not tile-aligned, one device owning no rows."""
    import torch
    ks, m, n = [128, 192], 700, 256
    a, b = _splits(m, ks, n, 77)
    ranges = [(0, 0), (0, 700)]
    c = MD.emulated_multi_device_gemm(_dev(a), _dev(b), row_ranges=ranges)
    ranges = [(0, 333), (333, 700)]
    c2 = MD.emulated_multi_device_gemm(_dev(a), _dev(b), row_ranges=ranges, concurrent=True)
    torch.cuda.synchronize()
    want = _want(a, b)
    for x in (c, c2):
        assert oracle.rel_error(x.float().cpu().numpy(), want) <= TOL


def test_repeated_epochs_reuse_pads_and_workspace(MD):
    """Several calls through one set of signal pads (epoch 1, 2, 3) and
    workspaces, inputs changed between calls: no stale slab is consumed."""
    import torch
    world, m, n, ks = 2, 512, 512, [512, 512]
    rows = [(0, 256), (256, 512)]
    pads = torch.zeros(world * 16, device="cuda", dtype=torch.int32)
    pad_ptrs = [pads.data_ptr() + 64 * p for p in range(world)]
    wss = [torch.empty(MD.workspace_bytes(r, world, ks, 256, n) + 1024, device="cuda",
                       dtype=torch.uint8) for r in range(world)]
    out = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    streams = [torch.cuda.Stream() for _ in range(world)]
    for epoch in (1, 2, 3):
        a, b = _splits(m, ks, n, 300 + epoch)
        da, db = _dev(a), _dev(b)
        torch.cuda.synchronize()
        for r, (lo, hi) in enumerate(rows):
            wp = (wss[r].data_ptr() + 1023) & ~1023
            MD.multi_device_gemm(r, world, [t.data_ptr() for t in da], [t.data_ptr() for t in db],
                                 ks, m, n, lo, hi - lo, out.data_ptr() + lo * n * 2, n, wp,
                                 wss[r].numel() - 1024, pads=pad_ptrs, epoch=epoch, comm_pairs=2,
                                 max_pairs=30, stream=streams[r].cuda_stream)
        torch.cuda.synchronize()
        assert oracle.rel_error(out.float().cpu().numpy(), _want(a, b)) <= TOL
    # every pad slot saw the last epoch: IN[p] and OUT[p] for each peer p != r
    pv = pads.cpu().numpy().reshape(world, 16)
    assert pv[0, 1] == 3 and pv[0, 9] == 3 and pv[1, 0] == 3 and pv[1, 8] == 3


def test_paper_shape_sampled_rows(MD):
    """PAPER.md:751 GD1-like shape (2 devices, M=8192, N=2048, K=16384) scaled
    to K=8192: the full kernel, oracle on sampled rows of both row blocks."""
    import torch
    world, m, n = 2, 4096, 2048
    ks = [4096, 4096]
    g = torch.Generator(device="cuda").manual_seed(5)
    a = [(torch.rand((m, k), device="cuda", generator=g) * 2 - 1).bfloat16() for k in ks]
    b = [(torch.rand((k, n), device="cuda", generator=g) * 2 - 1).bfloat16() for k in ks]
    c = MD.emulated_multi_device_gemm(a, b, concurrent=True)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 255, 256, 2047, 2048, 2049, 3000, 4095])
    an = [x.float().cpu().numpy() for x in a]
    bn = [x.float().cpu().numpy() for x in b]
    want = oracle.oracle_gemm(np.concatenate(an, axis=1)[rows], np.concatenate(bn, axis=0))
    got = c.float().cpu().numpy()[rows]
    assert oracle.rel_error(got, want) <= TOL
    # full-size linearity check: column sums of C vs (1^T A) . B
    colsum = c.float().sum(0)
    ref = sum((x.float().sum(0, keepdim=True) @ y.float()) for x, y in zip(a, b))[0]
    assert torch.allclose(colsum, ref, rtol=2e-3, atol=2e-3 * float(ref.abs().max()))


def test_arguments_rejected(MD):
    import torch
    from paper_2605_10905_b200 import MimwError
    a = torch.zeros((64, 60), device="cuda", dtype=torch.bfloat16)  # K not a multiple of 8 ... 60 % 8 != 0
    b = torch.zeros((60, 64), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(MimwError):
        MD.emulated_multi_device_gemm([a, a], [b, b])
