"""The torch.distributed form of the all-gather GEMM (AllGatherGemm) across
two PROCESSES sharing the one GPU: CUDA IPC allocation, handle exchange over a
gloo group, peer buffers mapped with cudaIpcOpenMemHandle and read by the
kernel's TMA through those mappings.  Kernels of different processes do not
run concurrently on one GPU, so the device-side barrier is replaced by host
barriers here (device_barrier=False); the barrier itself is covered by the
concurrent-streams tests in test_multi_device_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, ks, n, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_10905_b200 import multi_device as MD
        ag = MD.AllGatherGemm(m, ks, n, device=torch.device("cuda", 0))
        a = oracle.round_bf16(oracle.random_tile([m, ks[rank]], oracle.input_seed(61, 2 * rank)))
        b = oracle.round_bf16(oracle.random_tile([ks[rank], n], oracle.input_seed(61, 2 * rank + 1)))
        ag.a_local.copy_(torch.from_numpy(a).cuda().bfloat16())
        ag.b_local.copy_(torch.from_numpy(b).cuda().bfloat16())
        torch.cuda.synchronize()
        dist.barrier()  # every split written before any rank pulls
        c = ag(device_barrier=False)
        torch.cuda.synchronize()
        dist.barrier()  # every rank done pulling before any buffer is freed
        q.put((rank, ag.row0, c.float().cpu().numpy()))
        ag.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ks,m,n", [(2, [128, 192], 600, 264), (3, [64, 8, 256], 300, 128)])
def test_all_gather_gemm_across_processes(world, ks, m, n):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, ks, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a = [oracle.round_bf16(oracle.random_tile([m, k], oracle.input_seed(61, 2 * r))) for r, k in enumerate(ks)]
    b = [oracle.round_bf16(oracle.random_tile([k, n], oracle.input_seed(61, 2 * r + 1))) for r, k in enumerate(ks)]
    want = oracle.oracle_gemm(np.concatenate(a, axis=1), np.concatenate(b, axis=0))
    got = np.zeros_like(want)
    for _, row0, c in res:
        got[row0:row0 + c.shape[0]] = c
    assert oracle.rel_error(got, want) <= 1e-2
    assert oracle.rel_error_rows(got, want) <= 1e-2
