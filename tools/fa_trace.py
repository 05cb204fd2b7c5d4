"""Per-role cycle accounting of the attention kernel (debug aid, not a bench).

    python tools/fa_trace.py [--emu E]
Prints, averaged over CTAs, what the softmax warps and the MMA warp spend
their cycles on (clock64 deltas recorded by attention_fwd.cu when a trace
buffer is passed)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--emu", type=int, default=-1)
ap.add_argument("--bh", type=int, default=128)
ap.add_argument("--seq", type=int, default=8192)
a = ap.parse_args()
q, k, v = (torch.rand((a.bh, 1, a.seq, 128), device="cuda").to(torch.bfloat16) for _ in range(3))
tr = torch.zeros((148, 12, 8), dtype=torch.int64, device="cuda")
for _ in range(2):
    P.attention_fwd(q, k, v, emu=a.emu)
tr.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
P.attention_fwd(q, k, v, emu=a.emu, trace=tr)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
t = tr.cpu().double()
sm = t[:, :8, :].mean(dim=(0, 1))
mma = t[:, 9, :].mean(dim=0)
n = sm[4].item()
print(f"kernel {ms:.3f} ms (traced)")
print(f"softmax warp per tile (n={n:.0f}/warp): wait_S {sm[0]/n:.0f}  ld_S {sm[1]/n:.0f}  "
      f"max+exp {sm[2]/n:.0f}  wait_PV+rescale {sm[3]/n:.0f}  P store+arrive {sm[5]/n:.0f} cycles")
nm = mma[4].item()
print(f"MMA warp per KV step (n={nm:.0f}): wait_P0 {mma[0]/nm:.0f}  wait_P1 {mma[1]/nm:.0f}  "
      f"wait_KV {mma[2]/nm:.0f}  wait_Sfree {mma[3]/nm:.0f}  wait_Q {mma[6]/nm:.0f} cycles")
print(f"cycles per KV step (kernel time x 1.9 GHz / steps per CTA): "
      f"{ms * 1e-3 * 1.9e9 / nm:.0f} (MMA ideal 2048)")
