"""Cluster LayerNorm bandwidth over forced cluster sizes (debug aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

for rows, n in ((1152, 16384), (1152, 65536), (1152, 131072), (4, 65536)):
    x = torch.randn((rows, n), device="cuda")
    w = torch.randn(n, device="cuda")
    b = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    for cl in (0, 1, 2, 4, 8, 16):
        if cl and (n + cl - 1) // cl > 16384:
            continue
        f = lambda: P.layernorm(x, w, b, out=y, cluster=cl)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{rows}x{n} cluster {cl}: {ms * 1e3:.1f} us {8 * rows * n / ms / 1e6:.0f} GB/s")
