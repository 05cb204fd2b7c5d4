"""Run by tests/test_mutation_gpu.py in a subprocess, with MIMW_B200_LIB
pointing at a mutant (or the product) build: the wide-tile bf16 GEMM on a
few shapes, outputs pre-filled with NaN, checked against an fp32 torch
product.  Prints "ok" when every result is right, else the first failure."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_10905_b200 as P  # noqa: E402

SHAPES = [(4096, 4096, 1024), (1000, 2056, 520), (2304, 8192, 256), (4096, 8192, 64), (8192, 4096, 2048)]
REPS = int(os.environ.get("MUT_REPS", "3"))


def main():
    g = torch.Generator(device="cuda").manual_seed(7)
    for m, n, k in SHAPES:
        a = (torch.rand((m, k), device="cuda", generator=g) * 2 - 1).bfloat16()
        b = (torch.rand((k, n), device="cuda", generator=g) * 2 - 1).bfloat16()
        ref = a.float() @ b.float()
        scale = ref.abs().max().item()
        for r in range(REPS):
            out = torch.full((m, n), float("nan"), device="cuda", dtype=torch.bfloat16)
            P.gemm(a, b, out=out, tile_n=512)
            torch.cuda.synchronize()
            if torch.isnan(out).any():
                print(f"detected: unwritten or NaN outputs at {m}x{n}x{k} rep {r}")
                return
            err = (out.float() - ref).abs().max().item() / scale
            if err > 1e-2:
                print(f"detected: rel error {err:.3g} at {m}x{n}x{k} rep {r}")
                return
    print("ok")


if __name__ == "__main__":
    main()
