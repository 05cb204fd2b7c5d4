"""Four launches of the configs[3] FA forward (for an ncu capture of one):
    ncu --set full -k regex:attention_fwd -s 2 -c 1 python tools/fa_once.py <emu> [cta_group]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

emu = int(sys.argv[1]) if len(sys.argv) > 1 else -1
cg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
q, k, v = ((torch.rand((4, 32, 8192, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
for _ in range(4):
    o, lse = P.attention_fwd(q, k, v, emu=emu, cta_group=cg)
torch.cuda.synchronize()
