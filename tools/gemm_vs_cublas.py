"""bf16 GEMM 8192^3: ours vs cuBLAS (torch.mm) on the same operands, arms
alternated in blocks of `iters` launches, with NVML power / SM clock sampled
during each block, so the two kernels are compared at the same box state:
    python tools/gemm_vs_cublas.py [iters] [reps]
ARMS=mimw,cublas,... selects arms (mimw-r<G> = raster group G)."""
import os
import sys
import threading
import time

import torch
import pynvml

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
bt = b.t().contiguous()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
arms = {"mimw": lambda: P.gemm(a, b, out=c), "cublas": lambda: torch.mm(a, b, out=c),
        "mimw-nk": lambda: P.gemm(a, bt, out=c, b_layout=P.B_NK),
        "mimw-256": lambda: P.gemm(a, b, out=c, tile_n=256),
        "mimw-512": lambda: P.gemm(a, b, out=c, tile_n=512)}
for g in (4, 8, 16):
    arms[f"mimw-r{g}"] = (lambda g=g: P.gemm(a, b, out=c, raster_group=g))
    arms[f"mimw-512-r{g}"] = (lambda g=g: P.gemm(a, b, out=c, raster_group=g, tile_n=512))
sel = os.environ.get("ARMS", "mimw,cublas").split(",")
arms = {k: arms[k] for k in sel}
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetPowerUsage(hd) / 1e3,
                    pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.01)


for rep in range(reps):
    for name, f in arms.items():
        for _ in range(10):
            f()
        torch.cuda.synchronize()
        stop, smp = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, smp))
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / iters
        hi = [s for s in smp if s[0] > 0.6 * max(p for p, _ in smp)] or smp
        pw = sorted(p for p, _ in hi)[len(hi) // 2]
        mhz = sorted(m for _, m in hi)[len(hi) // 2]
        tf = 2 * n ** 3 / ms / 1e9
        print(f"rep {rep} {name:9s} {ms:.4f} ms {tf:7.1f} TFLOPS  power {pw:6.1f} W  sm {mhz} MHz  "
              f"TFLOP/J {tf / pw:.3f}  ({ms * iters:.0f} ms block)", flush=True)
        time.sleep(0.5)
