"""Per-warp cycle buckets of the 2-simplicial kernel (build with
MIMW_NVCC_EXTRA=-DMIMW_SIMP_TRACE python -m paper_2605_10905_b200.build --force):
    python tools/simp_trace.py
Buckets: producer [0 kv_empty]; MMA [1 kv_full, 2 qp_full, 3 p_full];
prep [1 qp_empty, 2 v1_empty]; softmax [1 s_full, 2 PV wait, 3 max exchange,
4 v1_full]; [7] total cycles."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

bh, s, w1, w2 = 16, 8192, 32, 512
t = [((torch.rand((bh, s, 128), device="cuda") * 2 - 1).bfloat16()) for _ in range(5)]
for _ in range(2):
    P.simplicial_attention_fwd(*t, w1=w1, w2=w2)
torch.cuda.synchronize()
buf = np.zeros(4 * 12 * 8, np.uint64)
r = P.lib().mimw_b200_debug_simplicial_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
assert r == 0, "build with -DMIMW_SIMP_TRACE"
tr = buf.reshape(4, 12, 8).astype(np.float64)
roles = {0: "producer", 1: "mma", 2: "softmax0", 3: "softmax0", 4: "softmax0", 5: "softmax0",
         6: "softmax1", 7: "softmax1", 8: "softmax1", 9: "softmax1", 10: "prep", 11: "prep"}
for w in range(12):
    tot = tr[:, w, 7].mean()
    print(f"warp {w:2d} {roles[w]:9s} total {tot/1e6:7.2f} Mcyc  " +
          "  ".join(f"[{i}] {100 * tr[:, w, i].mean() / max(tot, 1):5.1f}%" for i in range(7)))
