"""A/B timing of the FA forward between builds of the library on one box:
    python tools/fa_ab.py <lib_a.so> <lib_b.so> [<lib_c.so> ...] [rounds] [launches]"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

libs = [a for a in sys.argv[1:] if a.endswith(".so")]
rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
rounds = int(rest[0]) if rest else 3
iters = int(rest[1]) if len(rest) > 1 else 10  # launches per measurement (200+: the power-capped regime)
q, k, v = ((torch.rand((4, 32, 8192, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
flop = 4.0 * 128 * 128 * 8192 * 8192 / 2
handles = []
for path in libs:
    P._lib = None
    P.LIB_PATH = path
    handles.append(P.lib())
import time
for r in range(rounds):
    order = list(zip(libs, handles)) if r % 2 == 0 else list(zip(libs, handles))[::-1]
    for path, L in order:
        time.sleep(1.5)  # let the power state settle between measurements
        P._lib = L
        o, lse = P.attention_fwd(q, k, v)
        for _ in range(3):
            P.attention_fwd(q, k, v, out=o, lse=lse)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            P.attention_fwd(q, k, v, out=o, lse=lse)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(r, os.path.relpath(path), round(flop / ms / 1e9, 1), flush=True)
