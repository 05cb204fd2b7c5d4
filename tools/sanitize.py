"""Small invocations of every kernel, for compute-sanitizer (racecheck /
synccheck / memcheck) runs — the GPU analogue of the reference simulator's
vector-clock race detector (sim.cpp:282-316):
    compute-sanitizer --tool racecheck python tools/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

torch.manual_seed(0)
a = torch.randn(300, 200, device="cuda").bfloat16()
b = torch.randn(200, 264, device="cuda").bfloat16()
for cg in (1, 2, 4):
    P.gemm(a, b, cta_group=cg)
bw = torch.randn(200, 1040, device="cuda").bfloat16()
P.gemm(a, bw, tile_n=512)  # 256 x 512 wide tiles (register-drained epilogue)
P.gemm(a, bw.t().contiguous(), b_layout=P.B_NK, tile_n=512)
q, k, v = (torch.randn(1, 2, 300, 128, device="cuda").bfloat16() for _ in range(3))
P.attention_fwd(q, k, v)
P.attention_fwd(q, k, v, window=77)
P.attention_fwd(q, k, v, window=77, cta_group=2)  # 2-CTA kernel
offs = np.array([0, 5, 5, 300, 400], np.int64)
x = torch.randn(400, 128, device="cuda").bfloat16()
w = torch.randn(4, 128, 264, device="cuda").bfloat16()
P.grouped_gemm(x, offs, w)
P.grouped_gemm(x, offs, w, swap_tails=False)
ww = torch.randn(4, 128, 1040, device="cuda").bfloat16()
P.grouped_gemm(x, offs, ww, tile_n=512)  # wide, swapped tails
P.grouped_gemm(x, offs, ww, tile_n=512, swap_tails=False)  # wide, padded tails
qa = torch.randint(0, 120, (256, 256), device="cuda", dtype=torch.uint8)
sa = torch.randint(120, 130, (256, 8), device="cuda", dtype=torch.uint8)
for cg in (1, 2):
    P.gemm_mxfp8(qa.view(torch.float8_e4m3fn), sa, qa.view(torch.float8_e4m3fn), sa, cta_group=cg)
xl = torch.randn(6, 5000, device="cuda")
P.layernorm(xl, torch.ones(5000, device="cuda"), torch.zeros(5000, device="cuda"))
o_, l_ = P.attention_fwd(q, k, v, causal=False)
P.attention_bwd(q, k, v, o_, torch.randn_like(q), l_, causal=False)
o_, l_ = P.attention_fwd(q, k, v, window=77)
P.attention_bwd(q, k, v, o_, torch.randn_like(q), l_, window=77)
q1 = [torch.randn(2, 160, 128, device="cuda").bfloat16() for _ in range(5)]
P.simplicial_attention_fwd(*q1, w1=3, w2=40)
# all-gather multi-device GEMM, 3 emulated devices (sequential: no device barrier,
# which needs the ranks' kernels co-resident), both comm modes
from paper_2605_10905_b200 import multi_device as MD  # noqa: E402
sa_ = [torch.randn(300, kk, device="cuda").bfloat16() for kk in (64, 136, 0)]
sb_ = [torch.randn(kk, 264, device="cuda").bfloat16() for kk in (64, 136, 0)]
for cp in (-1, 1):
    MD.emulated_multi_device_gemm(sa_, sb_, comm_pairs=cp)
# reference-precision host entries: split-bf16 x3 attention (GEMM + softmax split kernels)
# and the f64 CUDA-core path, ragged S / D, window < S
rng = np.random.default_rng(0)
hq, hk, hv = (rng.standard_normal((75, 20)).astype(np.float32) for _ in range(3))
P.oracle_attention(hq, hk, hv, 9, 0.3, precision=P.PREC_F32_BF16X3)
P.oracle_attention(hq, hk, hv, 9, 0.3, precision=P.PREC_F32)
torch.cuda.synchronize()
print("sanitize run ok")
