"""GEMM 8192^3 timing over rasterisation group sizes (debug aid).
Each config: 3 warm-ups, then 50 launches; configs interleaved twice to
expose power-cap drift."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
groups = [int(x) for x in sys.argv[1:]] or [8, 4, 16, 32, 2]
for rep in range(3):
    for gsz in groups:
        if gsz == 0:  # cuBLAS through torch, same operands (B as [K,N] row-major)
            f = lambda: torch.mm(a, b, out=c)
        elif gsz < 0:  # two CTA pairs per cluster sharing B (multicast), raster group -gsz
            f = lambda: P.gemm(a, b, out=c, raster_group=-gsz, cta_group=4)
        else:
            f = lambda: P.gemm(a, b, out=c, raster_group=gsz)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 200
        print(f"rep {rep} group {gsz}: {ms:.4f} ms {2 * n ** 3 / ms / 1e9:.0f} TFLOPS")
