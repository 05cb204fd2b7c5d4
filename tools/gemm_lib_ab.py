"""8192^3 bf16 GEMM: two or more builds of the library (MIMW_B200_LIB-style
paths) alternated in blocks of `iters` launches in ONE process, plus cuBLAS:
    python tools/gemm_lib_ab.py lib_a.so lib_b.so [iters] [reps]"""
import ctypes
import os
import sys

import torch

libs = [a for a in sys.argv[1:] if a.endswith(".so")]
rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
iters = int(rest[0]) if rest else 300
reps = int(rest[1]) if len(rest) > 1 else 3
n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
handles = []
for p in libs:
    L = ctypes.CDLL(os.path.abspath(p))
    L.mimw_b200_gemm_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 6 + [ctypes.c_int32] * 2 + [
        ctypes.c_void_p]
    handles.append((p, L))
s = torch.cuda.current_stream().cuda_stream
arms = [(p, (lambda L=L: L.mimw_b200_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, 0, 1, s)))
        for p, L in handles] + [("cublas", lambda: torch.mm(a, b, out=c))]
for r in range(reps):
    for name, f in arms:
        for _ in range(10):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"rep {r} {os.path.basename(name):14s} {ms:.4f} ms {2 * n ** 3 / ms / 1e9:7.1f} TFLOPS", flush=True)
