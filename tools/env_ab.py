"""A/B of one workload between environment settings (knobs read once per
process), alternating fresh processes, median of the reps.
    python tools/env_ab.py simp "MIMW_SIMP_EMU=0" "MIMW_SIMP_EMU=2" [reps]
Workloads: simp (BH16 S8192 w1=32 w2=512), moe (configs[4]), fa (B4 H32 S8192
causal), bwd (B4 H48 S8192 non-causal), ln (1152 x 65536)."""
import os
import statistics
import subprocess
import sys

SETUP = {
    "simp": r'''
bh, s, w1, w2 = 16, 8192, 32, 512
t = [((torch.rand((bh, s, 128), device="cuda", generator=g) * 2 - 1).bfloat16()) for _ in range(5)]
f = lambda: P.simplicial_attention_fwd(*t, w1=w1, w2=w2)
tri = sum(min(w1, i + 1) * min(w2, i + 1) for i in range(s))
flop = 4.0 * 128 * tri * bh
out = lambda: f()[0]
''',
    "moe": r'''
rng = np.random.default_rng(5)
counts = rng.multinomial(32768, rng.dirichlet(np.ones(64)))
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
K, N = 4096, 14336
x = (torch.rand((int(offs[-1]), K), device="cuda", generator=g) * 2 - 1).bfloat16()
w = torch.empty((64, K, N), device="cuda", dtype=torch.bfloat16)
for e in range(64):
    w[e] = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
f = lambda: P.grouped_gemm(x, offs, w, out=y)
flop = 2.0 * offs[-1] * K * N
out = lambda: (f(), y)[1]
''',
    "fa": r'''
q, k, v = ((torch.rand((4, 32, 8192, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3))
f = lambda: P.attention_fwd(q, k, v)
flop = 4.0 * 128 * 4 * 32 * 8192 * 8193 / 2
out = lambda: f()[0]
''',
    "fa_emu": r'''
q, k, v = ((torch.rand((4, 32, 8192, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3))
f = lambda: P.attention_fwd(q, k, v, emu=int(os.environ.get("AB_EMU", "-1")))
flop = 4.0 * 128 * 4 * 32 * 8192 * 8193 / 2
out = lambda: f()[0]
''',
    "fa1k": r'''
q, k, v = ((torch.rand((1, 8192, 1024, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3))
f = lambda: P.attention_fwd(q, k, v)
flop = 4.0 * 128 * 8192 * 1024 * 1025 / 2
out = lambda: f()[0]
''',
    "bwd": r'''
q, k, v, do = ((torch.rand((4, 48, 8192, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(4))
o, lse = P.attention_fwd(q, k, v, causal=False)
f = lambda: P.attention_bwd(q, k, v, o, do, lse, causal=False)
flop = 2.5 * 4.0 * 128 * 4 * 48 * 8192 * 8192
out = lambda: f()[0]
''',
    "gemm": r'''
a = (torch.rand((8192, 8192), device="cuda", generator=g) * 2 - 1).bfloat16()
b = (torch.rand((8192, 8192), device="cuda", generator=g) * 2 - 1).bfloat16()
c = torch.empty((8192, 8192), device="cuda", dtype=torch.bfloat16)
f = lambda: P.gemm(a, b, out=c, cta_group=int(os.environ.get("AB_CG", "2")),
                   raster_group=int(os.environ.get("AB_RASTER", "0")))
flop = 2.0 * 8192 ** 3
out = lambda: (f(), c)[1]
''',
    "ln": r'''
x = torch.randn((1152, 65536), device="cuda", generator=g)
wt = torch.randn(65536, device="cuda", generator=g)
b = torch.randn(65536, device="cuda", generator=g)
y = torch.empty_like(x)
f = lambda: P.layernorm(x, wt, b, out=y)
flop = 8.0 * 1152 * 65536 * 1e3  # GB/s reported as "TFLOPS" / 1e3
out = lambda: (f(), y)[1]
''',
}

CODE = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_10905_b200 as P
g = torch.Generator(device="cuda").manual_seed(1)
%s
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
r = out()
print(e0.elapsed_time(e1) / 10, flop, float(r.flatten()[::997].float().sum()))
'''

work = sys.argv[1]
arms = [a for a in sys.argv[2:] if "=" in a]
reps = int(sys.argv[-1]) if "=" not in sys.argv[-1] else 4
res = {a: [] for a in arms}
sums = {a: set() for a in arms}
flop = 0.0
for _ in range(reps):
    for arm in arms:
        env = dict(os.environ)
        for kv in arm.split():
            k, v = kv.split("=")
            env[k] = v
        p = subprocess.run([sys.executable, "-c", CODE % SETUP[work]], env=env, capture_output=True, text=True)
        if p.returncode != 0:
            print(arm, "FAILED", p.stderr[-800:])
            continue
        ms, flop, cs = p.stdout.split()
        res[arm].append(float(ms))
        sums[arm].add(cs)
        flop = float(flop)
for arm in arms:
    if res[arm]:
        ms = statistics.median(res[arm])
        print(f"{arm:36s} median {ms:.3f} ms {flop / ms / 1e9:7.0f} TFLOPS  {['%.3f' % v for v in res[arm]]} checksum {sums[arm]}")
