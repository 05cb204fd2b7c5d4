"""Multi-GPU sharding of the hot path: one process per GPU,
independent shards, NCCL all-gather over NVLink only to reassemble outputs.

The reference has no real multi-device code: its "devices" are 2-CTA clusters
inside one simulated grid (proj/kernels/multi_device_gemm.mimw:2-6,
oracles.cpp:57-80).  Here the path partitions cleanly:

* GEMM  — C row panels (B replicated), aligned to the 256-row cluster tile;
* FA    — the B*H (batch, head) pairs;
* MoE   — contiguous expert ranges balanced by padded MMA tiles.

Each ``sharded_*`` function computes the local shard with the B200 kernels
(``compute`` is injectable only so the CPU gloo tests can exercise the plan
and the reassembly without a GPU) and then ``all_gather``s the pieces.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

Range = Tuple[int, int]


def split_even(n: int, world: int, align: int = 1) -> List[Range]:
    """Contiguous [lo, hi) ranges covering [0, n), sizes multiples of ``align``
    (except the last non-empty one), as equal as the alignment allows."""
    if world <= 0:
        raise ValueError("world must be >= 1")
    units = -(-n // align) if n else 0
    out, lo_u = [], 0
    for r in range(world):
        cnt = units // world + (1 if r < units % world else 0)
        lo, hi = min(n, lo_u * align), min(n, (lo_u + cnt) * align)
        out.append((lo, hi))
        lo_u += cnt
    return out


def row_panels(m: int, world: int, tile: int = 256) -> List[Range]:
    """GEMM C row panels aligned to the cluster tile (no tile straddles two GPUs)."""
    return split_even(m, world, tile)


def head_shards(bh: int, world: int) -> List[Range]:
    """(batch*head) ranges for the attention forward."""
    return split_even(bh, world, 1)


def expert_shards(counts: Sequence[int], world: int, tile: int = 256) -> List[Range]:
    """Contiguous expert ranges minimising the largest per-GPU MMA work
    (sum of ceil(m_e / tile) padded tiles; rows are packed by expert so each
    shard's rows are contiguous).  Exact min-max partition by binary search
    on the bottleneck + greedy fill."""
    cost = [-(-int(c) // tile) + 1e-9 * int(c) for c in counts]  # tiles, ties by rows
    e = len(cost)
    if e == 0:
        return [(0, 0)] * world

    def fill(cap):
        out, lo, acc = [], 0, 0.0
        for i, c in enumerate(cost):
            if acc + c > cap and i > lo:
                out.append((lo, i))
                lo, acc = i, 0.0
            acc += c
        out.append((lo, e))
        return out

    lo_c, hi_c = max(cost), sum(cost)
    for _ in range(64):
        mid = (lo_c + hi_c) / 2
        if len(fill(mid)) <= world:
            hi_c = mid
        else:
            lo_c = mid
    parts = fill(hi_c)
    while len(parts) < world:
        parts.append((e, e))
    return parts


def group_rows(offsets: Sequence[int], r: Range) -> Range:
    """Row range of experts [r[0], r[1]) given the packed row offsets."""
    return int(offsets[r[0]]), int(offsets[r[1]])


# ---------------------------------------------------------------------------
# reassembly
# ---------------------------------------------------------------------------
def all_gather_rows(local, ranges: Sequence[Range], group=None):
    """Reassemble a tensor split by leading-dim ranges (ragged allowed):
    every rank contributes ``local`` (rows ranges[rank]); returns the full
    tensor on every rank.  Uneven shards are padded to the largest one for
    the collective (NCCL all_gather needs equal sizes) and compacted after."""
    import torch
    import torch.distributed as dist
    world = len(ranges)
    if world == 1:
        return local
    rows = [hi - lo for lo, hi in ranges]
    pad = max(rows)
    shape = tuple(local.shape[1:])
    buf = local
    if local.shape[0] != pad:
        buf = torch.zeros((pad,) + shape, dtype=local.dtype, device=local.device)
        buf[:local.shape[0]] = local
    out = torch.empty((world * pad,) + shape, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    if all(r == pad for r in rows):
        return out
    return torch.cat([out[i * pad:i * pad + rows[i]] for i in range(world)], dim=0)


# ---------------------------------------------------------------------------
# sharded hot-path calls
# ---------------------------------------------------------------------------
def sharded_gemm(a, b, rank: int, world: int, group=None, compute: Callable | None = None,
                 gather: bool = True):
    """C = A.B with C row panels per GPU (A, B replicated on every rank)."""
    r0, r1 = row_panels(a.shape[0], world)[rank]
    if compute is None:
        from . import gemm
        compute = gemm
    local = compute(a[r0:r1], b)
    return all_gather_rows(local, row_panels(a.shape[0], world), group) if gather else local


def sharded_attention(q, k, v, rank: int, world: int, group=None, compute: Callable | None = None,
                      gather: bool = True):
    """Causal attention forward with the (batch, head) pairs split across GPUs.
    q, k, v: [B, H, S, D]; returns (o, lse) reassembled on every rank."""
    b, h, s, d = q.shape
    ranges = head_shards(b * h, world)
    lo, hi = ranges[rank]
    flat = lambda t: t.reshape(b * h, 1, s, d)
    if compute is None:
        from . import attention_fwd
        compute = attention_fwd
    o, lse = compute(flat(q)[lo:hi], flat(k)[lo:hi], flat(v)[lo:hi])
    if not gather:
        return o, lse
    o = all_gather_rows(o, ranges, group).reshape(b, h, s, d)
    lse = all_gather_rows(lse, ranges, group).reshape(b, h, s)
    return o, lse


def sharded_grouped_gemm(x, m_offsets, w_local, rank: int, world: int, counts: Sequence[int],
                         group=None, compute: Callable | None = None, gather: bool = True):
    """MoE grouped GEMM sharded by expert: this rank holds only its experts'
    weights ``w_local`` ([E_r, K, N]) and computes their (contiguous) rows."""
    ranges = expert_shards(counts, world)
    e0, e1 = ranges[rank]
    if w_local.shape[0] != e1 - e0:
        raise ValueError(f"rank {rank} owns experts [{e0}, {e1}) but w_local has {w_local.shape[0]}")
    r0, r1 = group_rows(m_offsets, (e0, e1))
    local_offs = np.asarray(m_offsets[e0:e1 + 1], dtype=np.int64) - r0
    if compute is None:
        from . import grouped_gemm
        compute = grouped_gemm
    y = compute(x[r0:r1], local_offs, w_local)
    if not gather:
        return y
    row_ranges = [group_rows(m_offsets, r) for r in ranges]
    return all_gather_rows(y, row_ranges, group)
