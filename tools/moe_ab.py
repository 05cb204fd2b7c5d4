"""configs[4] grouped MoE GEMM: tile / tail-mode arms alternated in one
process (identical inputs, checksums compared):
    python tools/moe_ab.py [reps] [steps] [idle seconds before each arm]"""
import os
import sys
import time

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
arms = {"narrow-swap": dict(tile_n=256, swap_tails=True), "wide-padded": dict(tile_n=512, swap_tails=False),
        "wide-swap": dict(tile_n=512, swap_tails=True)}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
gap = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0  # seconds idle before each arm (cool start)
res = {a: [] for a in arms}
for r in range(reps):
    for name, kw in arms.items():
        f = lambda: P.grouped_gemm(x, offs, w, out=y, **kw)
        if gap:
            torch.cuda.synchronize()
            time.sleep(gap)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[name].append(ms)
        print(f"rep {r} {name:12s} {ms:.3f} ms {flop / ms / 1e9:.0f} TFLOPS  sum {float(y[::97].float().sum()):.6e}",
              flush=True)
for name, v in res.items():
    print(f"{name:12s} median {np.median(v):.3f} ms {flop / np.median(v) / 1e9:.0f} TFLOPS")
