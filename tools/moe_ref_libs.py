"""Same-box library reference for the grouped MoE GEMM (configs[4]):
torch._grouped_mm (CUTLASS grouped GEMM inside PyTorch) on the bench's
operands, beside ours, arms alternated.  Context only, not a product path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402
import bench  # noqa: E402

E, K, N = bench.MOE_E, bench.MOE_K, bench.MOE_N
counts = bench.moe_counts()
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
g = torch.Generator(device="cuda").manual_seed(5)
x = (torch.rand((int(offs[-1]), K), device="cuda", generator=g) * 2 - 1).bfloat16()
w = torch.empty((E, K, N), device="cuda", dtype=torch.bfloat16)
for e in range(E):
    w[e] = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
flop = 2.0 * offs[-1] * K * N
offs_dev = torch.from_numpy(offs[1:].astype(np.int32)).cuda()
arms = {"mimw": lambda: P.grouped_gemm(x, offs, w, out=y),
        "torch._grouped_mm": lambda: torch._grouped_mm(x, w, offs=offs_dev)}


def timed(f, n=10):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ours = arms["mimw"]()
try:
    ref = arms["torch._grouped_mm"]()
    torch.cuda.synchronize()
    err = ((ref.float() - y.float()).abs().max() / y.float().abs().max()).item()
    print(f"torch._grouped_mm vs ours: max abs diff / max {err:.2e}")
except Exception as e:  # noqa: BLE001
    print("torch._grouped_mm unavailable:", type(e).__name__, str(e)[:300])
    arms.pop("torch._grouped_mm")
for rep in range(3):
    for name, f in arms.items():
        ms = timed(f)
        print(f"rep {rep} {name:18s} {ms:.3f} ms {flop / ms / 1e9:.0f} TFLOPS", flush=True)
