"""Per-tile timeline of the grouped MoE GEMM (configs[4]; debug aid):
    python tools/moe_trace.py [--build]
--build compiles a trace build (-DMIMW_TILE_TRACE) of the library into
/tmp/mimw_trace and re-executes itself on it.  Prints per tile class (full
256-row tiles, swapped tails of heavy groups, light groups) the count and
MMA-to-epilogue durations, and a coarse timeline of what is in flight."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--build" in sys.argv:
    dst = "/tmp/mimw_trace"
    shutil.rmtree(dst, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2605_10905_b200"), os.path.join(dst, "paper_2605_10905_b200"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(dst, "include"))
    env = {**os.environ, "MIMW_NVCC_EXTRA": "-DMIMW_TILE_TRACE"}
    subprocess.run([sys.executable, "-c", "import paper_2605_10905_b200.build as b; b.build(force=True)"],
                   cwd=dst, env=env, check=True)
    env = {**os.environ, "MIMW_B200_LIB": os.path.join(dst, "paper_2605_10905_b200", "libmimw_b200.so")}
    sys.exit(subprocess.run([sys.executable, __file__] + [a for a in sys.argv[1:] if a != "--build"],
                            env=env).returncode)

import ctypes  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402
sys.path.insert(0, ROOT)
import paper_2605_10905_b200 as P  # noqa: E402
import bench  # noqa: E402

E, K, N = bench.MOE_E, bench.MOE_K, bench.MOE_N
counts = bench.moe_counts()
if "--uniform" in sys.argv:  # every group 512 rows: full tiles only
    counts = np.full(E, 512, dtype=np.int64)
offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
g = torch.Generator(device="cuda").manual_seed(5)
x = (torch.rand((int(offs[-1]), K), device="cuda", generator=g) * 2 - 1).bfloat16()
w = torch.empty((E, K, N), device="cuda", dtype=torch.bfloat16)
for e in range(E):
    w[e] = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
y = torch.empty((int(offs[-1]), N), device="cuda", dtype=torch.bfloat16)
# host copy of the kernel's tile order (chunk 1: groups in turn, N-tiles outer, M-tiles inner);
# MIMW_MOE_WIDE (default 1): 256 x 512 tiles
WIDE = os.environ.get("MIMW_MOE_WIDE", "1") != "0"
nn = (N + 511) // 512 if WIDE else (N + 255) // 256
tiles = []
for e in range(E):
    m = int(counts[e])
    if m == 0:
        continue
    mt = (m + 255) // 256
    for t in range(mt * nn):
        r_mt, nt = t % mt, t // mt
        kind = "light" if m < 256 else ("full" if r_mt < m // 256 else "tail")
        tiles.append((e, r_mt, nt, kind, m))
tr = torch.zeros((len(tiles), 4), dtype=torch.int64, device="cuda")
L = P.lib()
L.mimw_b200_debug_tile_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    P.grouped_gemm(x, offs, w, out=y)
P._check(L.mimw_b200_debug_tile_trace(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
P.grouped_gemm(x, offs, w, out=y)
e1.record()
torch.cuda.synchronize()
P._check(L.mimw_b200_debug_tile_trace(None))
ms = e0.elapsed_time(e1)
t = tr.cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
st, iss, done = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3  # us
span = done.max()
flop = 2.0 * counts.sum() * K * N
print(f"kernel {ms:.3f} ms ({flop / ms / 1e9:.0f} TFLOPS), traced span {span / 1e3:.3f} ms, {len(tiles)} tiles")
if "--dense" in sys.argv:  # the same FLOPs as one dense GEMM [rows, K] x [K, N]
    wd = w[0].contiguous()
    for _ in range(3):
        P.gemm(x, wd, out=y)
    e0.record()
    P.gemm(x, wd, out=y)
    e1.record()
    torch.cuda.synchronize()
    msd = e0.elapsed_time(e1)
    print(f"dense {int(counts.sum())}x{N}x{K}: {msd:.3f} ms ({flop / msd / 1e9:.0f} TFLOPS)")
kinds = np.array([k for _, _, _, k, _ in tiles])
rows = np.array([m for *_, m in tiles])
dur = done - st
for k in ("full", "tail", "light"):
    s = kinds == k
    if s.any():
        print(f"{k:5s} n={s.sum():5d}  dur us: mean {dur[s].mean():6.1f} p10 {np.percentile(dur[s], 10):6.1f} "
              f"p50 {np.median(dur[s]):6.1f} p90 {np.percentile(dur[s], 90):6.1f}  sum/74 {dur[s].sum() / 74 / 1e3:.3f} ms")
nb = 40
edges = np.linspace(0, span, nb + 1)
print("timeline (bin us: avg pairs busy full/tail/light, expert ids started)")
for i in range(nb):
    a, b = edges[i], edges[i + 1]
    ov = np.clip(np.minimum(done, b) - np.maximum(st, a), 0, None) / (b - a)
    busy = {k: ov[kinds == k].sum() for k in ("full", "tail", "light")}
    ex = sorted({tiles[j][0] for j in np.nonzero((st >= a) & (st < b))[0]})
    print(f"{a:7.0f} {busy['full']:5.1f} {busy['tail']:5.1f} {busy['light']:5.1f}  e{ex[:6]}{'...' if len(ex) > 6 else ''}")
