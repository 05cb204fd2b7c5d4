"""Timing of the attention backward / non-causal forward on the paper's shapes
(B=4, H=48, D=128; AFN / ABC rows) and the error of a small
case against the f64 oracle.

    python tools/fa_bwd_time.py [--seqs 1024,2048,4096,8192] [--iters 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402


def timeit(fn, iters):
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
    ap.add_argument("--seqs", default="1024,2048,4096,8192")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--h", type=int, default=48)
    ap.add_argument("--causal", type=int, default=0)
    args = ap.parse_args()
    for s in [int(x) for x in args.seqs.split(",")]:
        b, h = args.b, args.h
        g = torch.Generator(device="cuda").manual_seed(3)
        q, k, v, do = ((torch.rand((b, h, s, 128), device="cuda", generator=g) * 2 - 1).bfloat16()
                       for _ in range(4))
        causal = bool(args.causal)
        o, lse = P.attention_fwd(q, k, v, causal=causal)
        fwd_ms = timeit(lambda: P.attention_fwd(q, k, v, causal=causal, out=o, lse=lse), args.iters)
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        bwd_ms = timeit(lambda: P.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv),
                        args.iters)
        frac = 0.5 if causal else 1.0
        fwd_flop = 4.0 * b * h * s * s * 128 * frac
        res = {"seq": s, "causal": causal, "bh": b * h, "fwd_ms": round(fwd_ms, 3),
               "fwd_tflops": round(fwd_flop / fwd_ms / 1e9, 1), "bwd_ms": round(bwd_ms, 3),
               "bwd_tflops": round(2.5 * fwd_flop / bwd_ms / 1e9, 1)}
        # cuDNN / flash SDPA backward on the same box, for reference
        try:
            qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))
            with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.CUDNN_ATTENTION):
                out = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)

                def sdpa_bwd():
                    torch.autograd.grad(out, (qq, kk, vv), do, retain_graph=True)
                ms = timeit(sdpa_bwd, args.iters)
            res["cudnn_bwd_tflops"] = round(2.5 * fwd_flop / ms / 1e9, 1)
        except Exception as e:  # noqa: BLE001
            res["cudnn_bwd"] = str(e)[:80]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
