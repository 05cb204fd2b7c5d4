"""GPU: the sharded entry points run the B200 kernels by
default and, at world size 1, equal the unsharded kernels bit for bit; each
shard of a multi-GPU plan computed alone equals the same rows of the full
result (shards are independent, so N GPUs reassemble the N=1 answer)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2605_10905_b200 as P
    P.lib()
    return P


def test_gemm_panels_equal_full(P):
    import torch
    from paper_2605_10905_b200 import shard
    g = torch.Generator(device="cuda").manual_seed(1)
    a = (torch.rand((2000, 512), device="cuda", generator=g) - 0.5).bfloat16()
    b = (torch.rand((512, 768), device="cuda", generator=g) - 0.5).bfloat16()
    full = P.gemm(a, b)
    assert torch.equal(shard.sharded_gemm(a, b, 0, 1), full)
    for world in (2, 8):
        parts = [shard.sharded_gemm(a, b, r, world, gather=False) for r in range(world)]
        assert torch.equal(torch.cat(parts, 0), full)


def test_attention_heads_equal_full(P):
    import torch
    from paper_2605_10905_b200 import shard
    g = torch.Generator(device="cuda").manual_seed(2)
    q, k, v = ((torch.rand((2, 3, 384, 128), device="cuda", generator=g) * 2 - 1).bfloat16()
               for _ in range(3))
    o, lse = P.attention_fwd(q, k, v)
    o1, l1 = shard.sharded_attention(q, k, v, 0, 1)
    assert torch.equal(o1.reshape(o.shape), o) and torch.equal(l1.reshape(lse.shape), lse)
    parts = [shard.sharded_attention(q, k, v, r, 4, gather=False) for r in range(4)]
    assert torch.equal(torch.cat([p[0] for p in parts], 0).reshape(o.shape), o)


def test_moe_experts_equal_full(P):
    import torch
    from paper_2605_10905_b200 import shard
    counts = [300, 0, 17, 256, 129, 64, 1, 500]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.rand((int(offs[-1]), 256), device="cuda", generator=g) - 0.5).bfloat16()
    w = (torch.rand((8, 256, 384), device="cuda", generator=g) - 0.5).bfloat16()
    full = P.grouped_gemm(x, offs, w)
    for world in (1, 2, 3):
        parts = shard.expert_shards(counts, world)
        ys = [shard.sharded_grouped_gemm(x, offs, w[e0:e1], r, world, counts, gather=False)
              for r, (e0, e1) in enumerate(parts)]
        assert torch.equal(torch.cat(ys, 0), full)
