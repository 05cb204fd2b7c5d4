"""Grouped MoE GEMM (configs[4]) timing: cta_group 1 vs 2 (debug aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

rng = np.random.default_rng(5)
counts = rng.multinomial(32768, rng.dirichlet(np.ones(64)))
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
K, N = 4096, 14336
x = (torch.rand((int(offs[-1]), K), device="cuda") * 2 - 1).bfloat16()
w = torch.empty((64, K, N), device="cuda", dtype=torch.bfloat16)
for e in range(64):
    w[e] = (torch.rand((K, N), device="cuda") * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
flop = 2.0 * offs[-1] * K * N
for cg in [int(a) for a in sys.argv[1:]] or [2, 3, 2, 3]:  # 3 = cta_group 2 without swapped tails
    f = lambda: P.grouped_gemm(x, offs, w, out=y, cta_group=min(cg, 2), swap_tails=cg != 3)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cta_group {cg}: {ms:.3f} ms {flop / ms / 1e9:.0f} TFLOPS")
