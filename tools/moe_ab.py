"""A/B of the grouped MoE GEMM (configs[4]) between environment settings,
alternating fresh processes (each knob is read once per process) and reporting
the median.  Usage: python tools/moe_ab.py "MIMW_GEMM_CLC=1" "MIMW_GEMM_CLC=0" [reps]"""
import os
import statistics
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
g = torch.Generator(device="cuda").manual_seed(1)
x = (torch.rand((int(offs[-1]), K), device="cuda", generator=g) * 2 - 1).bfloat16()
w = torch.empty((64, K, N), device="cuda", dtype=torch.bfloat16)
for e in range(64):
    w[e] = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
cg = int(os.environ.get("AB_CG", "2"))
f = lambda: P.grouped_gemm(x, offs, w, out=y, cta_group=cg)
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
print(e0.elapsed_time(e1) / 10, float(y[::97, ::13].float().sum()))
'''
a, b = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
flop = 2.0 * 32768 * 4096 * 14336
res = {a: [], b: []}
sums = {a: set(), b: set()}
for _ in range(reps):
    for arm in (a, b):
        env = dict(os.environ)
        for kv in arm.split():
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True).stdout.split()
        res[arm].append(float(out[0]))
        sums[arm].add(out[1])
for arm in (a, b):
    ms = statistics.median(res[arm])
    print(f"{arm:40s} median {ms:.3f} ms {flop / ms / 1e9:.0f} TFLOPS  all {['%.3f' % v for v in res[arm]]} checksum {sums[arm]}")
