"""MXFP8 8192^3: the 256 x 224 (cta_group 2) and 256 x 448 (cta_group 3)
kernels alternated in one process, blocks of `iters` launches, plus cuBLAS
MXFP8 when torch exposes it:  python tools/fp8_ab.py [iters] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = n = k = 8192
qa = torch.randint(0, 120, (m, k), device="cuda", dtype=torch.uint8).view(torch.float8_e4m3fn)
qb = torch.randint(0, 120, (n, k), device="cuda", dtype=torch.uint8).view(torch.float8_e4m3fn)
sfa = torch.randint(120, 134, (m, k // 32), device="cuda", dtype=torch.uint8)
sfb = torch.randint(120, 134, (n, k // 32), device="cuda", dtype=torch.uint8)
c = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
arms = {cg: (lambda cg=cg: P.gemm_mxfp8(qa, sfa, qb, sfb, out=c, cta_group=cg)) for cg in (2, 3)}
ref = {}
for cg, f in arms.items():
    f()
    torch.cuda.synchronize()
    ref[cg] = c.clone()
print("identical outputs:", torch.equal(ref[2], ref[3]))
for r in range(reps):
    for cg, f in arms.items():
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"rep {r} cta_group {cg}: {ms:.4f} ms {2 * m * n * k / ms / 1e9:.0f} TFLOPS", flush=True)
