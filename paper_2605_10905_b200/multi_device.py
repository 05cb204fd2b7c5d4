"""All-gather (K-gathered) multi-device GEMM — SURVEY.md §8f rank 1.

The reference's multi-device program (proj/kernels/multi_device_gemm.mimw:1-79,
oracle ``oracle_multi_device_gemm``, oracles.cpp:57-80) computes
``C = [a0 | a1] . [b0 ; b1]``: every device holds one K-split of A and B, owns
a row block of C, and a "comm" CTA streams the other device's K chunks into
the compute CTA's shared-memory ring while it accumulates.  On B200 the same
program is one kernel per GPU (``mimw_b200_multi_device_gemm``): comm CTA
pairs pull the peers' splits over NVLink (CUDA IPC mappings of the peers'
HBM) into a local landing buffer, slab by slab, and the GEMM CTA pairs wait on
a slab's readiness counter only right before its first TMA load — so the
transfer overlaps the tensor-core work tile by tile.

Three layers:

* ``multi_device_gemm(...)``  — one rank's launch on explicit pointers
  (local or IPC-mapped), the C-ABI call 1:1;
* ``emulated_multi_device_gemm(...)``  — every "device" on one GPU (the
  reference's own setting: its devices are clusters of one grid); with
  ``concurrent=True`` the per-rank kernels run side by side on separate
  streams and meet in the device-side entry/exit barrier;
* ``AllGatherGemm``  — the torch.distributed form: one process per GPU,
  symmetric IPC buffers exchanged through the process group, one call per
  step.  The IPC backend is injectable so the host logic runs on CPU (gloo).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import MimwError, ERR_ARG, ERR_SHAPE, _check, _stream, lib
from .shard import row_panels

MAX_DEVICES = 8
IPC_HANDLE_BYTES = 64
SIGNAL_PAD_BYTES = 64

_SIGS = {
    "mimw_b200_multi_device_gemm_workspace_bytes": ([C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                                     C.c_int64], C.c_int64),
    "mimw_b200_multi_device_gemm": ([C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
                                    + [C.c_int64] * 4 + [C.c_void_p, C.c_int64, C.c_void_p,
                                                         C.c_int64, C.c_void_p, C.c_uint32,
                                                         C.c_int32, C.c_int32, C.c_void_p], C.c_int),
    "mimw_b200_multi_device_gemm_ex": ([C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
                                       + [C.c_int64] * 4 + [C.c_void_p, C.c_int64, C.c_void_p,
                                                            C.c_int64, C.c_void_p, C.c_uint32]
                                       + [C.c_int32] * 5 + [C.c_void_p], C.c_int),
    "mimw_b200_ipc_alloc": ([C.c_int64, C.POINTER(C.c_void_p), C.c_void_p], C.c_int),
    "mimw_b200_ipc_open": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "mimw_b200_ipc_close": ([C.c_void_p], C.c_int),
    "mimw_b200_ipc_free": ([C.c_void_p], C.c_int),
}


def _lib():
    L = lib()
    for name, (args, res) in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


def _arr(ctype, vals):
    return (ctype * len(vals))(*vals)


def workspace_bytes(rank: int, world: int, k_splits: Sequence[int], rows: int, n: int) -> int:
    """Landing buffers for the world-1 remote splits + slab counters."""
    ks = _arr(C.c_int64, [int(k) for k in k_splits])
    r = _lib().mimw_b200_multi_device_gemm_workspace_bytes(rank, world, C.cast(ks, C.c_void_p),
                                                           rows, n)
    if r < 0:
        raise MimwError(ERR_ARG, "bad rank/world/k_splits")
    return int(r)


def multi_device_gemm(rank: int, world: int, a_ptrs: Sequence[int], b_ptrs: Sequence[int],
                      k_splits: Sequence[int], m: int, n: int, row0: int, rows: int, c_ptr: int,
                      ldc: int, ws_ptr: int, ws_bytes: int, pads: Optional[Sequence[int]] = None,
                      epoch: int = 0, comm_pairs: int = 0, max_pairs: int = 0, stream=None,
                      comm_box: int = 0, comm_agents: int = 0, comm_lag: int = 0) -> None:
    """One rank's launch (``mimw_b200_multi_device_gemm``) on raw device pointers.
    ``comm_box`` / ``comm_agents`` / ``comm_lag`` tune the comm CTAs' copy
    pipelines (0 = library defaults)."""
    if len(a_ptrs) != world or len(b_ptrs) != world or len(k_splits) != world:
        raise MimwError(ERR_ARG, "one a/b pointer and one K per device")
    a = _arr(C.c_void_p, list(a_ptrs))
    b = _arr(C.c_void_p, list(b_ptrs))
    ks = _arr(C.c_int64, [int(k) for k in k_splits])
    p = _arr(C.c_void_p, list(pads)) if pads is not None else None
    _check(_lib().mimw_b200_multi_device_gemm_ex(
        rank, world, C.cast(a, C.c_void_p), C.cast(b, C.c_void_p), C.cast(ks, C.c_void_p), m, n,
        row0, rows, c_ptr, ldc, ws_ptr, ws_bytes, C.cast(p, C.c_void_p) if p is not None else None,
        epoch, comm_pairs, max_pairs, comm_box, comm_agents, comm_lag, _stream(stream)))


def _check_splits(a_splits, b_splits):
    world = len(a_splits)
    if world < 1 or world > MAX_DEVICES or len(b_splits) != world:
        raise MimwError(ERR_ARG, f"1..{MAX_DEVICES} devices, one A and one B split each")
    m = a_splits[0].shape[0]
    n = b_splits[0].shape[1]
    for a, b in zip(a_splits, b_splits):
        if a.shape[0] != m or b.shape[1] != n or a.shape[1] != b.shape[0]:
            raise MimwError(ERR_SHAPE, "multi_device_gemm: inconsistent split shapes")
    return world, m, n


def emulated_multi_device_gemm(a_splits, b_splits, row_ranges: Optional[List[Tuple[int, int]]] = None,
                               concurrent: bool = False, comm_pairs: int = 0, out=None):
    """All ``world`` devices emulated on the current GPU: rank r's kernel reads
    the other ranks' splits in place (they stand in for the IPC-mapped peer
    buffers) and writes C rows ``row_ranges[r]``.  ``concurrent=True`` runs the
    ranks side by side on their own streams (each with a share of the SMs)
    with the device-side entry/exit barrier over signal pads in local memory;
    otherwise the ranks run one after another without the barrier.
    Returns bf16 C [m, n]."""
    import torch
    world, m, n = _check_splits(a_splits, b_splits)
    ks = [int(a.shape[1]) for a in a_splits]
    if row_ranges is None:
        row_ranges = row_panels(m, world)
    dev = a_splits[0].device
    if out is None:
        out = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
    a_ptrs = [a.data_ptr() for a in a_splits]
    b_ptrs = [b.data_ptr() for b in b_splits]
    wss = []
    for r, (lo, hi) in enumerate(row_ranges):
        nb = workspace_bytes(r, world, ks, hi - lo, n)
        wss.append(torch.empty(nb + 1024, device=dev, dtype=torch.uint8))
    if not concurrent:
        for r, (lo, hi) in enumerate(row_ranges):
            ws = wss[r]
            wp = (ws.data_ptr() + 1023) & ~1023
            multi_device_gemm(r, world, a_ptrs, b_ptrs, ks, m, n, lo, hi - lo,
                              out.data_ptr() + lo * n * 2, n, wp, ws.numel() - (wp - ws.data_ptr()),
                              comm_pairs=comm_pairs)
        return out
    # concurrent ranks: one stream each, SMs shared out so all kernels are co-resident
    pads = torch.zeros(world * SIGNAL_PAD_BYTES // 4, device=dev, dtype=torch.int32)
    pad_ptrs = [pads.data_ptr() + SIGNAL_PAD_BYTES * p for p in range(world)]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cp = comm_pairs
    # margin: GPC packing may strand a few SMs; a rank without rows still runs one comm pair
    pairs = max(1, sms // 2 // world - max(cp, 1) - 2)
    cur = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    for s in streams:
        s.wait_stream(cur)
    for r, (lo, hi) in enumerate(row_ranges):
        ws = wss[r]
        wp = (ws.data_ptr() + 1023) & ~1023
        multi_device_gemm(r, world, a_ptrs, b_ptrs, ks, m, n, lo, hi - lo,
                          out.data_ptr() + lo * n * 2, n, wp, ws.numel() - (wp - ws.data_ptr()),
                          pads=pad_ptrs, epoch=1, comm_pairs=cp, max_pairs=pairs,
                          stream=streams[r].cuda_stream)
    for s in streams:
        cur.wait_stream(s)
    return out


# ---------------------------------------------------------------------------
# torch.distributed form: one process per GPU, symmetric IPC buffers
# ---------------------------------------------------------------------------
class CudaIpc:
    """libmimw_b200's CUDA IPC entries (the injectable backend of AllGatherGemm)."""

    def alloc(self, nbytes: int) -> Tuple[int, bytes]:
        ptr = C.c_void_p()
        h = (C.c_uint8 * IPC_HANDLE_BYTES)()
        _check(_lib().mimw_b200_ipc_alloc(nbytes, C.byref(ptr), C.cast(h, C.c_void_p)))
        return int(ptr.value), bytes(h)

    def open(self, handle: bytes) -> int:
        ptr = C.c_void_p()
        h = (C.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(handle)
        _check(_lib().mimw_b200_ipc_open(C.cast(h, C.c_void_p), C.byref(ptr)))
        return int(ptr.value)

    def close(self, ptr: int) -> None:
        _check(_lib().mimw_b200_ipc_close(ptr))

    def free(self, ptr: int) -> None:
        _check(_lib().mimw_b200_ipc_free(ptr))


def symmetric_layout(m: int, k_splits: Sequence[int], n: int, rank: int) -> dict:
    """Byte offsets inside rank's symmetric buffer: signal pad, A split
    [m, k_rank], B split [k_rank, n] (each 1 KiB aligned)."""
    al = lambda x: (x + 1023) & ~1023  # noqa: E731
    k = int(k_splits[rank])
    pad = 0
    a = al(SIGNAL_PAD_BYTES)
    b = al(a + m * k * 2)
    return {"pad": pad, "a": a, "b": b, "total": al(b + k * n * 2)}


class _DevView:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class AllGatherGemm:
    """``C = [a_0 | ... | a_{W-1}] . [b_0 ; ... ; b_{W-1}]`` with split s on
    GPU s, C rows partitioned over the GPUs (256-row aligned panels).

    Each rank allocates one symmetric buffer (signal pad + its A/B split),
    exchanges IPC handles through ``group`` (all_gather_object) and maps the
    peers' buffers.  Write the local split into ``a_local`` / ``b_local`` (bf16
    torch views of the symmetric buffer), then call the object: one fused
    gather+GEMM kernel, with the device-side entry/exit barrier, returns this
    rank's C rows.  ``gather_output=True`` also all-gathers C (NCCL) to every
    rank."""

    def __init__(self, m: int, k_splits: Sequence[int], n: int, group=None, ipc=None,
                 comm_pairs: int = 0, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if len(k_splits) != self.world:
            raise MimwError(ERR_ARG, "one K split per rank")
        if self.world > MAX_DEVICES:
            raise MimwError(ERR_ARG, f"at most {MAX_DEVICES} devices")
        self.m, self.n, self.k_splits = int(m), int(n), [int(k) for k in k_splits]
        self.rows = row_panels(self.m, self.world)
        self.row0, hi = self.rows[self.rank]
        self.nrows = hi - self.row0
        self.ipc = ipc if ipc is not None else CudaIpc()
        self.comm_pairs = comm_pairs
        self.device = device
        self.epoch = 0
        self.layouts = [symmetric_layout(self.m, self.k_splits, self.n, r) for r in range(self.world)]
        self.base, handle = self.ipc.alloc(self.layouts[self.rank]["total"])
        handles = [None] * self.world
        dist.all_gather_object(handles, handle, group=group)
        self.bases = []
        for r, h in enumerate(handles):
            self.bases.append(self.base if r == self.rank else self.ipc.open(h))
        self.a_ptrs = [b + L["a"] for b, L in zip(self.bases, self.layouts)]
        self.b_ptrs = [b + L["b"] for b, L in zip(self.bases, self.layouts)]
        self.pad_ptrs = [b + L["pad"] for b, L in zip(self.bases, self.layouts)]
        self.ws_bytes = workspace_bytes(self.rank, self.world, self.k_splits, self.nrows, self.n)
        self._ws = None
        self._out = None

    # -- local split views (bf16) --
    def _view(self, off: int, shape):
        import torch
        return torch.as_tensor(_DevView(self.base + off, shape, "<u2"), device=self.device).view(
            torch.bfloat16)

    @property
    def a_local(self):
        return self._view(self.layouts[self.rank]["a"], (self.m, self.k_splits[self.rank]))

    @property
    def b_local(self):
        return self._view(self.layouts[self.rank]["b"], (self.k_splits[self.rank], self.n))

    def __call__(self, out=None, gather_output: bool = False, stream=None,
                 device_barrier: bool = True):
        """One fused gather+GEMM step; returns this rank's C rows (or all of C
        with ``gather_output``).  ``device_barrier=False`` skips the kernel's
        entry/exit barrier: the caller then orders the ranks itself (e.g. a
        host barrier before and after), as on one GPU shared by several
        processes, where the ranks' kernels cannot be co-resident."""
        import torch
        if self._ws is None:
            self._ws = torch.empty(self.ws_bytes + 1024, dtype=torch.uint8, device=self.device)
        if out is None:
            if self._out is None:
                self._out = torch.empty((self.nrows, self.n), dtype=torch.bfloat16, device=self.device)
            out = self._out
        self.epoch += 1
        wp = (self._ws.data_ptr() + 1023) & ~1023
        multi_device_gemm(self.rank, self.world, self.a_ptrs, self.b_ptrs, self.k_splits, self.m,
                          self.n, self.row0, self.nrows, out.data_ptr(), self.n, wp,
                          self._ws.numel() - (wp - self._ws.data_ptr()),
                          pads=self.pad_ptrs if device_barrier else None,
                          epoch=self.epoch if device_barrier else 0, comm_pairs=self.comm_pairs,
                          stream=stream)
        if not gather_output:
            return out
        from .shard import all_gather_rows
        return all_gather_rows(out, self.rows, group=self.group)

    def close(self) -> None:
        for r, b in enumerate(self.bases):
            if r != self.rank:
                self.ipc.close(b)
        self.ipc.free(self.base)
        self.bases = []
