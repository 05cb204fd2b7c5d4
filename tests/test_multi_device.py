"""CPU tests of the all-gather multi-device GEMM host side:
the workspace plan and argument validation of the C-ABI (host-only code, no
kernel launch), and AllGatherGemm's symmetric-buffer / IPC-handle exchange
over a world-2 gloo process group with a fake IPC backend (the CUDA IPC calls
need a GPU; the bookkeeping around them does not)."""
import ctypes
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_10905_b200 import MimwError, multi_device as MD


@pytest.fixture(scope="module")
def L():
    from paper_2605_10905_b200 import build
    build.build()
    return MD._lib()


def test_workspace_plan(L):
    # counters (8 splits x max slabs + 4 words, 1 KiB aligned) + landing A/B of the remote splits
    ks, rows, n = [512, 256], 300, 128
    nb = MD.workspace_bytes(0, 2, ks, rows, n)
    al = lambda x: (x + 1023) & ~1023  # noqa: E731
    ctr = al(4 * (8 * 2 + 4))
    assert nb == al(al(ctr + rows * 256 * 2) + 256 * n * 2)
    nb1 = MD.workspace_bytes(1, 2, ks, rows, n)
    assert nb1 == al(al(ctr + rows * 512 * 2) + 512 * n * 2)
    assert MD.workspace_bytes(0, 1, [4096], 256, 256) == al(4 * (8 + 4))  # no peers: counters only
    with pytest.raises(MimwError):
        MD.workspace_bytes(2, 2, ks, rows, n)


def _call(L, rank=0, world=2, ks=(64, 64), m=64, n=64, row0=0, rows=32, pads=None, epoch=0):
    a = (ctypes.c_void_p * world)(*([16] * world))
    b = (ctypes.c_void_p * world)(*([16] * world))
    k = (ctypes.c_int64 * world)(*ks)
    return L.mimw_b200_multi_device_gemm(rank, world, ctypes.cast(a, ctypes.c_void_p),
                                         ctypes.cast(b, ctypes.c_void_p),
                                         ctypes.cast(k, ctypes.c_void_p), m, n, row0, rows, 1024,
                                         n, 1024, 1 << 20, pads, epoch, 0, 0, None)


def test_argument_validation_before_device_work(L):
    assert _call(L, world=9, ks=(64,) * 9) == 4
    assert _call(L, rank=2) == 4
    assert _call(L, row0=40, rows=32) == 1 and b"row range" in L.mimw_b200_last_error()
    assert _call(L, ks=(64, 60)) == 2 and b"multiple of 8" in L.mimw_b200_last_error()
    assert _call(L, n=60) == 2
    pads = (ctypes.c_void_p * 2)(64, None)
    assert _call(L, pads=ctypes.cast(pads, ctypes.c_void_p), epoch=1) == 4
    pads = (ctypes.c_void_p * 2)(64, 128)
    assert _call(L, pads=ctypes.cast(pads, ctypes.c_void_p), epoch=0) == 4
    assert b"epoch" in L.mimw_b200_last_error()


def test_symmetric_layout_aligned():
    for r in range(4):
        lay = MD.symmetric_layout(1000, [64, 128, 8, 0], 520, r)
        assert lay["pad"] == 0 and lay["a"] % 1024 == 0 and lay["b"] % 1024 == 0
        assert lay["b"] - lay["a"] >= 1000 * [64, 128, 8, 0][r] * 2
        assert lay["total"] >= lay["b"] + [64, 128, 8, 0][r] * 520 * 2


class FakeIpc:
    """Stands in for CUDA IPC: 'device pointers' are integers, a handle names
    the owner's allocation; open/close are recorded."""

    def __init__(self, rank):
        self.rank = rank
        self.opened, self.closed, self.freed = [], [], []

    def alloc(self, nbytes):
        base = (self.rank + 1) << 40
        return base, f"h{self.rank}:{base}:{nbytes}".encode().ljust(64, b"\0")

    def open(self, handle):
        owner, base, _ = handle.rstrip(b"\0").decode()[1:].split(":")
        self.opened.append(int(owner))
        return int(base) + (1 << 50)  # a different VA in this process, as IPC gives

    def close(self, ptr):
        self.closed.append(ptr)

    def free(self, ptr):
        self.freed.append(ptr)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ipc = FakeIpc(rank)
        ks = [256, 512]
        g = MD.AllGatherGemm(1000, ks, 384, ipc=ipc)
        res = dict(rank=g.rank, world=g.world, row0=g.row0, nrows=g.nrows, bases=g.bases,
                   a_ptrs=g.a_ptrs, b_ptrs=g.b_ptrs, pads=g.pad_ptrs, opened=list(ipc.opened),
                   ws=g.ws_bytes)
        g.close()
        res.update(closed=ipc.closed, freed=ipc.freed)
        q.put(res)
    finally:
        dist.destroy_process_group()


def test_all_gather_gemm_handle_exchange_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r = q.get(timeout=120)
        out[r["rank"]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # row panels of 1000 rows over 2 devices, 256-aligned
    assert (out[0]["row0"], out[0]["nrows"]) == (0, 512)
    assert (out[1]["row0"], out[1]["nrows"]) == (512, 488)
    for r in range(world):
        o = out[r]
        peer = 1 - r
        assert o["opened"] == [peer]                           # mapped exactly the peer's buffer
        assert o["bases"][r] == (r + 1) << 40                   # own allocation in place
        assert o["bases"][peer] == ((peer + 1) << 40) + (1 << 50)
        lay = [MD.symmetric_layout(1000, [256, 512], 384, s) for s in range(world)]
        assert o["a_ptrs"] == [o["bases"][s] + lay[s]["a"] for s in range(world)]
        assert o["b_ptrs"] == [o["bases"][s] + lay[s]["b"] for s in range(world)]
        assert o["pads"] == [o["bases"][s] for s in range(world)]
        assert o["closed"] == [o["bases"][peer]] and o["freed"] == [o["bases"][r]]
    # workspace: landing buffers for the one remote split
    assert out[0]["ws"] > 512 * 512 * 2 + 512 * 384 * 2
