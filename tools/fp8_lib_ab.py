"""A/B of library builds on the MXFP8 8192^3 GEMM (cta_group 2), alternating
builds in one process:  python tools/fp8_lib_ab.py <lib_a.so> <lib_b.so> [...] [iters] [reps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

libs = [a for a in sys.argv[1:] if a.endswith(".so")]
rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
iters = int(rest[0]) if rest else 50
reps = int(rest[1]) if len(rest) > 1 else 4
hs = []
for path in libs:
    P._lib = None
    P.LIB_PATH = path
    hs.append(P.lib())
m = n = k = 8192
qa = torch.randint(0, 120, (m, k), device="cuda", dtype=torch.uint8).view(torch.float8_e4m3fn)
qb = torch.randint(0, 120, (n, k), device="cuda", dtype=torch.uint8).view(torch.float8_e4m3fn)
sfa = torch.randint(120, 134, (m, k // 32), device="cuda", dtype=torch.uint8)
sfb = torch.randint(120, 134, (n, k // 32), device="cuda", dtype=torch.uint8)
c = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
for r in range(reps):
    for path, L in (list(zip(libs, hs)) if r % 2 == 0 else list(zip(libs, hs))[::-1]):
        P._lib = L
        time.sleep(1.0)
        for _ in range(3):
            P.gemm_mxfp8(qa, sfa, qb, sfb, out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            P.gemm_mxfp8(qa, sfa, qb, sfb, out=c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(r, os.path.relpath(path), round(2.0 * m * n * k / ms / 1e9, 1), "TFLOPS", round(ms * 1e3, 1), "us",
              flush=True)
