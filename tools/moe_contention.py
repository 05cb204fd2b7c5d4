"""Is the grouped MoE GEMM's weight streaming limited per SM or by DRAM?
Uniform routing (512 rows per expert, configs[4] K/N): time per 256x512 tile
with 74 / 48 / 37 / 24 CTA pairs (expert weights streamed from DRAM), and
the same FLOPs as one dense GEMM (weight L2-resident).  If the per-tile time falls as
fewer pairs stream at once, DRAM is the shared limit; if it stays, each
pair's own fetch pipeline is.
    python tools/moe_contention.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

E, K, N, M = 64, 4096, 14336, 512
offs = np.arange(E + 1, dtype=np.int64) * M
x = (torch.rand((E * M, K), device="cuda") * 2 - 1).bfloat16()
w = (torch.rand((E, K, N), device="cuda") * 2 - 1).bfloat16()
y = torch.empty((E * M, N), device="cuda", dtype=torch.bfloat16)
tiles = E * (M // 256) * ((N + 511) // 512)
flop = 2.0 * E * M * K * N


def run(wt, mc, reps=5):
    for _ in range(2):
        P.grouped_gemm(x, offs, wt, out=y, max_clusters=mc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.grouped_gemm(x, offs, wt, out=y, max_clusters=mc)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for mc in (74, 48, 37, 24):
    ms_d = run(w, mc)
    print(f"pairs {mc:3d}: distinct weights {ms_d:6.3f} ms  {ms_d * 1e3 * mc / tiles:6.1f} us/tile  "
          f"{flop / ms_d / 1e9:6.0f} TFLOPS  weight stream {E * K * N * 2 / ms_d / 1e6:6.0f} GB/s", flush=True)
wd = w[0].contiguous()
for _ in range(2):
    P.gemm(x, wd, out=y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    P.gemm(x, wd, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"dense (one weight): {ms:6.3f} ms  {ms * 1e3 * 74 / tiles:6.1f} us/tile  {flop / ms / 1e9:6.0f} TFLOPS")
