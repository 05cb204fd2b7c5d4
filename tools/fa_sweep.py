"""Untraced FA-forward timing over the exp2-emulation split (debug aid)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P
bh, s = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 8192
q, k, v = ((torch.rand((bh, 1, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
flop = 4.0 * bh * 128 * s * s / 2
for emu in [int(x) for x in sys.argv[2:]] or (2, 0, 1, 2, 0, 1, 3, 2):
    for _ in range(3):
        P.attention_fwd(q, k, v, emu=emu)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        P.attention_fwd(q, k, v, emu=emu)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"emu {emu}: {ms:.3f} ms  {flop / ms / 1e9:.0f} TFLOPS")
