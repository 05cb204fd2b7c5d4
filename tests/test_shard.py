"""CPU tests of the multi-GPU path: shard plans and the
all-gather reassembly, world_size 2 over gloo.  The per-shard compute is the
CPU oracle here (test infrastructure); on the GPU box it is the B200 kernels
and the collective is NCCL — the host logic under test is the same."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_10905_b200 import shard


def test_split_even_covers_and_aligns():
    for n in (0, 1, 255, 256, 8192, 8193):
        for world in (1, 2, 3, 8):
            r = shard.split_even(n, world, 256)
            assert len(r) == world
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all(lo % 256 == 0 for lo, _ in r if lo < n)
    assert shard.row_panels(8192, 8) == [(i * 1024, (i + 1) * 1024) for i in range(8)]
    assert shard.head_shards(128, 8)[3] == (48, 64)


def test_expert_shards_are_contiguous_and_balanced():
    rng = np.random.default_rng(5)
    counts = rng.multinomial(32768, rng.dirichlet(np.ones(64)))
    for world in (1, 2, 4, 8):
        parts = shard.expert_shards(counts, world)
        assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == 64
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        tiles = [sum(-(-int(c) // 256) for c in counts[lo:hi]) for lo, hi in parts]
        total = sum(-(-int(c) // 256) for c in counts)
        # contiguous min-max partition: bottleneck within one expert of the ideal
        assert max(tiles) <= total / world + max(-(-int(c) // 256) for c in counts)
    assert shard.expert_shards([], 3) == [(0, 0)] * 3
    assert shard.expert_shards([5, 0, 0], 4)[-1] == (3, 3)


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
        res = {}
        # GEMM row panels: C = A.B, uneven M (last panel short)
        a = oracle.round_bf16(oracle.random_tile([600, 48], 7))
        b = oracle.round_bf16(oracle.random_tile([48, 40], 8))
        f = lambda x, y: torch.from_numpy(oracle.oracle_gemm(x.numpy(), y.numpy()))
        c = shard.sharded_gemm(torch.from_numpy(a), torch.from_numpy(b), rank, world, compute=f)
        res["gemm"] = float(np.max(np.abs(c.numpy() - oracle.oracle_gemm(a, b))))
        # attention: (batch, head) pairs split, o and lse reassembled
        bq, h, s, d = 1, 3, 20, 8
        qkv = [oracle.random_tile([bq, h, s, d], 31 + i) for i in range(3)]

        def fa(q_, k_, v_):
            os_, ls_ = [], []
            for i in range(q_.shape[0]):
                o, l = oracle.oracle_attention(q_[i, 0].numpy(), k_[i, 0].numpy(),
                                               v_[i, 0].numpy(), s, d ** -0.5, with_lse=True)
                os_.append(o[None])
                ls_.append(l[None])
            return (torch.from_numpy(np.stack(os_)) if os_ else torch.zeros((0, 1, s, d)),
                    torch.from_numpy(np.stack(ls_)) if ls_ else torch.zeros((0, 1, s)))

        o, lse = shard.sharded_attention(*(torch.from_numpy(t) for t in qkv), rank, world,
                                         compute=fa)
        want = [oracle.oracle_attention(qkv[0][0, j], qkv[1][0, j], qkv[2][0, j], s, d ** -0.5,
                                        with_lse=True) for j in range(h)]
        res["attn"] = max(float(np.max(np.abs(o[0, j].numpy() - want[j][0]))) for j in range(h))
        res["lse"] = max(float(np.max(np.abs(lse[0, j].numpy() - want[j][1]))) for j in range(h))
        # MoE: experts split (ragged rows, an empty expert), weights local only
        counts = [5, 0, 17, 3, 9]
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        x = oracle.random_tile([int(offs[-1]), 16], 3)
        w = oracle.random_tile([5, 16, 24], 4)
        e0, e1 = shard.expert_shards(counts, world)[rank]

        def gg(x_, offs_, w_):
            ys = oracle.oracle_grouped_gemm(x_.numpy(), offs_, w_.numpy())
            return torch.from_numpy(np.concatenate(ys, 0) if ys else np.zeros((0, 24), np.float32))

        y = shard.sharded_grouped_gemm(torch.from_numpy(x), offs, torch.from_numpy(w[e0:e1]),
                                       rank, world, counts, compute=gg)
        want = np.concatenate(oracle.oracle_grouped_gemm(x, offs, w), 0)
        res["moe"] = float(np.max(np.abs(y.numpy() - want)))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_paths_reassemble_exactly_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank in range(world):
        for k, v in out[rank].items():
            assert v == 0.0, (rank, k, v)  # same oracle per shard: bit-exact reassembly
