"""Per-rank timing of the all-gather multi-device GEMM on the paper's shapes
(GD1-GD5) with the peers emulated on one GPU (their splits
are local HBM buffers standing in for IPC-mapped NVLink memory).

For rank 0 of each shape (rows = M / world, full N, K = sum of splits):
  fused   one launch: comm pairs pull the remote splits while the GEMM runs
  plain   the GEMM alone on pre-gathered operands (the no-communication bound)
  serial  D2D copies of the remote splits, then the GEMM (gather-then-compute)

    python tools/md_sweep.py [--iters 20] [--comm 4]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402
from paper_2605_10905_b200 import multi_device as MD  # noqa: E402

SHAPES = {"GD1": (2, 8192, 2048, 16384), "GD2": (4, 8192, 2048, 16384),
          "GD3": (4, 8192, 8192, 16384), "GD4": (4, 4096, 8192, 16384),
          "GD5": (4, 16384, 4096, 8192)}


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--comm", type=int, default=0, help="comm pairs (0 = library default: comm warps in every GEMM CTA)")
    ap.add_argument("--cfgs", default="0,0,0,0",
                    help="semicolon list of box,agents,lag,comm_pairs for the fused kernel (0 = default)")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    args = ap.parse_args()
    for name in args.shapes.split(","):
        world, m, n, k = SHAPES[name]
        ks = [k // world] * world
        rows = m // world
        a = [torch.randn((m, kk), device="cuda").bfloat16() for kk in ks]
        b = [torch.randn((kk, n), device="cuda").bfloat16() for kk in ks]
        c = torch.empty((rows, n), device="cuda", dtype=torch.bfloat16)
        nb = MD.workspace_bytes(0, world, ks, rows, n)
        ws = torch.empty(nb + 1024, device="cuda", dtype=torch.uint8)
        wp = (ws.data_ptr() + 1023) & ~1023
        ap_ = [t.data_ptr() for t in a]
        bp_ = [t.data_ptr() for t in b]

        cfg = [0, 0, 0, args.comm]

        def fused():
            MD.multi_device_gemm(0, world, ap_, bp_, ks, m, n, 0, rows, c.data_ptr(), n, wp, nb,
                                 comm_pairs=cfg[3], comm_box=cfg[0], comm_agents=cfg[1],
                                 comm_lag=cfg[2])

        a_cat = torch.cat([t[:rows] for t in a], dim=1).contiguous()
        b_cat = torch.cat(b, dim=0).contiguous()

        def plain():
            P.gemm(a_cat, b_cat, out=c)

        a_land = torch.empty_like(a_cat)
        b_land = torch.empty_like(b_cat)

        def serial():
            off = ks[0]
            for s in range(1, world):
                a_land[:, off:off + ks[s]].copy_(a[s][:rows])
                b_land[off:off + ks[s]].copy_(b[s])
                off += ks[s]
            P.gemm(a_land, b_land, out=c)

        flop = 2.0 * rows * n * k
        res = {"shape": name, "world": world, "rows": rows, "n": n, "k": k}
        for label, fn in (("plain", plain), ("serial", serial)):
            ms = timeit(fn, args.iters)
            res[label + "_ms"] = round(ms, 4)
            res[label + "_tflops"] = round(flop / ms / 1e9, 1)
        for cs in args.cfgs.split(";"):
            cfg[:] = [int(x) for x in cs.split(",")]
            cfg[3] = cfg[3] or args.comm
            ms = timeit(fused, args.iters)
            res["fused_" + cs] = [round(ms, 4), round(flop / ms / 1e9, 1)]
        # correctness spot check of the fused result against plain
        fused()
        ref = torch.empty_like(c)
        P.gemm(a_cat, b_cat, out=ref)
        torch.cuda.synchronize()
        res["max_rel_vs_plain"] = float((c.float() - ref.float()).abs().max() / ref.float().abs().max())
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
