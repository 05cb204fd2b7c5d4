"""A/B of library builds on the configs[4] grouped MoE GEMM and the 8192^3
dense GEMM, alternating builds in one process (identical inputs):
    python tools/lib_ab_moe.py <lib_a.so> <lib_b.so> [...] [rounds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402
import bench  # noqa: E402

libs = [a for a in sys.argv[1:] if a.endswith(".so")]
rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
rounds = int(rest[0]) if rest else 3
E, K, N = bench.MOE_E, bench.MOE_K, bench.MOE_N
counts = bench.moe_counts()
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
x = (torch.rand((int(offs[-1]), K), device="cuda") * 2 - 1).bfloat16()
w = (torch.rand((E, K, N), device="cuda") * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
a = (torch.rand((8192, 8192), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((8192, 8192), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((8192, 8192), device="cuda", dtype=torch.bfloat16)
handles = []
for path in libs:
    P._lib = None
    P.LIB_PATH = path
    handles.append(P.lib())


def t(f, iters):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for r in range(rounds):
    order = list(zip(libs, handles)) if r % 2 == 0 else list(zip(libs, handles))[::-1]
    for path, L in order:
        P._lib = L
        time.sleep(1.0)
        ms_moe = t(lambda: P.grouped_gemm(x, offs, w, out=y), 10)
        time.sleep(1.0)
        ms_g = t(lambda: P.gemm(a, b, out=c), 20)
        print(r, os.path.relpath(path), "moe", round(2.0 * offs[-1] * K * N / ms_moe / 1e9, 1),
              "gemm", round(2.0 * 8192 ** 3 / ms_g / 1e9, 1), flush=True)
