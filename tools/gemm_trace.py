"""Per-tile timeline of the dense 8192^3 GEMM (wide 256x512 tiles; debug aid):
    python tools/gemm_trace.py --build
Per tile: MMA start (after the accumulator is free), last MMA issued, the
epilogue sees the accumulator, the epilogue has drained it.  Prints the
drain time, the MMA warp's idle gap between tiles and the first/last wave."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--build" in sys.argv:
    dst = "/tmp/mimw_gtrace"
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

n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
tiles = (n // 256) * (n // 512)
tr = torch.zeros((tiles, 4), dtype=torch.int64, device="cuda")
L = P.lib()
L.mimw_b200_debug_tile_trace.argtypes = [ctypes.c_void_p]
for _ in range(5):
    P.gemm(a, b, out=c)
P._check(L.mimw_b200_debug_tile_trace(tr.data_ptr()))
P.gemm(a, b, out=c)
torch.cuda.synchronize()
P._check(L.mimw_b200_debug_tile_trace(None))
t = tr.cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
st, iss, full, drained = ((t[:, i] - t0) / 1e3 for i in range(4))
span = drained.max()
print(f"span {span:.1f} us, {tiles} tiles")
print(f"MMA issue per tile (start -> last issue) us: median {np.median(iss - st):.2f}")
print(f"tile (start -> accumulator seen by epilogue) us: median {np.median(full - st):.2f} p90 {np.percentile(full - st, 90):.2f}")
print(f"drain (accumulator seen -> released) us: median {np.median(drained - full):.2f} p90 {np.percentile(drained - full, 90):.2f}")
# per pair (SM of the leader not recorded here): chain tiles by start order per cluster using gaps
order = np.argsort(st)
print(f"first tile start spread us: {np.sort(st)[73] - np.sort(st)[0]:.2f}; last tile end {full.max():.1f}, "
      f"last-wave idle (span - median pair busy) ...")
ends = np.sort(full)
print("tile completion times, last 80 (us):", np.round(ends[-80:][::8], 1).tolist())
