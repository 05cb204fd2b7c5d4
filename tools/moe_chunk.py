"""Grouped MoE GEMM (configs[4]) timing over MIMW_MOE_CHUNK values, one
process per value (the knob is read once per process).  Debug aid."""
import os
import subprocess
import sys

CODE = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_10905_b200 as P
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
f = lambda: P.grouped_gemm(x, offs, w, out=y)
for _ in range(3):
    f()
ref = y.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"chunk {os.environ.get('MIMW_MOE_CHUNK')}: {ms:.3f} ms {flop / ms / 1e9:.0f} TFLOPS  sum {float(y.float().sum()):.6e}")
'''
for c in (sys.argv[1:] or ["1", "2", "4", "8", "16", "64"]):
    subprocess.run([sys.executable, "-c", CODE], env={**os.environ, "MIMW_MOE_CHUNK": c}, check=False)
