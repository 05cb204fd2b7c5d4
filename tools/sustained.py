"""Sustained (seconds-long) throughput of the bf16 GEMM 8192^3 vs cuBLAS on the
same operands: N back-to-back launches per arm, arms alternated, so the
~1 kW power cap has settled (the default bench measures the burst regime)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
arms = {"mimw": lambda: P.gemm(a, b, out=c), "cublas": lambda: torch.mm(a, b, out=c),
        "mimw-pairs": lambda: P.gemm(a, b, out=c, cta_group=4),
        "mimw-r16": lambda: P.gemm(a, b, out=c, raster_group=16)}
if os.environ.get("ARMS"):
    arms = {k: arms[k] for k in os.environ["ARMS"].split(",")}
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
for rep in range(2):
    for name, f in arms.items():
        for _ in range(20):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"rep {rep} {name:6s} {ms:.4f} ms  {2 * n ** 3 / ms / 1e9:.0f} TFLOPS over {ms * iters / 1e3:.1f} s")
        time.sleep(1)
