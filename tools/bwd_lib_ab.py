"""A/B of library builds on the ABC4 attention backward (B4 H48 S8192 non-causal),
alternating builds in one process:  python tools/bwd_lib_ab.py <lib_a.so> <lib_b.so> [...]"""
import os, sys, time, torch
sys.path.insert(0, ".")
import paper_2605_10905_b200 as P
libs = [a for a in sys.argv[1:] if a.endswith(".so")]
hs = []
for path in libs:
    P._lib = None; P.LIB_PATH = path; hs.append(P.lib())
b, h, s = 4, 48, 8192
q, k, v, do = ((torch.rand((b, h, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(4))
P._lib = hs[0]
o, lse = P.attention_fwd(q, k, v, causal=False)
ref = None
for r in range(4):
    for path, L in (list(zip(libs, hs)) if r % 2 == 0 else list(zip(libs, hs))[::-1]):
        P._lib = L
        time.sleep(1.0)
        out = P.attention_bwd(q, k, v, o, do, lse, causal=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): out = P.attention_bwd(q, k, v, o, do, lse, causal=False)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        dq = out[0].float()
        if ref is None: ref = dq.clone()
        print(r, path, round(ms, 3), "ms", round(2.5 * 4 * b * h * s * s * 128 / ms / 1e9, 1), "TF", "max|dq-ref|", (dq - ref).abs().max().item(), flush=True)
