"""Per-warp cycle buckets of the attention backward kernel (build with
MIMW_NVCC_EXTRA=-DMIMW_BWD_TRACE python -m paper_2605_10905_b200.build --force):
    python tools/bwd_trace.py
Buckets: producer [1 ld_empty]; MMA [1 ld_full, 2 dp_free, 3 p_full, 4 dq_free];
softmax [1 s_full, 2 ds_free, 3 lse/D barrier]; drain [1 dq_full, 2 reduce read]; [7] total."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

b, h, s = 4, 48, 8192
q, k, v, do = ((torch.rand((b, h, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(4))
o, lse = P.attention_fwd(q, k, v, causal=False)
for _ in range(2):
    P.attention_bwd(q, k, v, o, do, lse, causal=False)
torch.cuda.synchronize()
buf = np.zeros(4 * 16 * 8, np.uint64)
r = P.lib().mimw_b200_debug_bwd_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
assert r == 0, "build with -DMIMW_BWD_TRACE"
tr = buf.reshape(4, 16, 8).astype(np.float64)
roles = ["producer", "mma", "-", "-"] + ["softmax"] * 8 + ["drain"] * 4
for w in range(16):
    tot = tr[:, w, 7].mean()
    if tot == 0:
        continue
    print(f"warp {w:2d} {roles[w]:8s} total {tot/1e6:7.2f} Mcyc  " +
          "  ".join(f"[{i}] {100 * tr[:, w, i].mean() / tot:5.1f}%" for i in range(1, 7)))
