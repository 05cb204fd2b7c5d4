"""FA forward timing, one-CTA kernel vs the 2-CTA kernel (cta_group=2) over
the exp2-emulation split, in alternating order on one box:
    python tools/fa_cg2_sweep.py [rounds]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2
arms = [(1, -1), (2, 0), (2, 1), (2, 2), (2, 3), (2, 4)]
q, k, v = ((torch.rand((4, 32, 8192, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty((4, 32, 8192), device="cuda", dtype=torch.float32)
flop = 4.0 * 128 * 128 * 8192 * 8192 / 2
ref = None
for r in range(rounds):
    for cg, emu in (arms if r % 2 == 0 else arms[::-1]):
        time.sleep(1.0)
        for _ in range(3):
            P.attention_fwd(q, k, v, out=o, lse=lse, cta_group=cg, emu=emu)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            P.attention_fwd(q, k, v, out=o, lse=lse, cta_group=cg, emu=emu)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        if ref is None:
            ref = o.float().clone()
        err = (o.float() - ref).abs().max().item()
        print(f"round {r} cta_group {cg} emu {emu:2d}: {ms:.3f} ms {flop / ms / 1e9:7.1f} TFLOPS  max|o-o_1cta| {err:.2e}",
              flush=True)
