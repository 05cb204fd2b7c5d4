"""Library attention on the same shape as configs[3] (B=4 H=32 S=8192 D=128
causal bf16), for context: torch SDPA backends (cuDNN, flash) and flashinfer
if importable.  Not part of the product path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

B, H, S, D = 4, 32, 8192, 128
q, k, v = ((torch.rand((B, H, S, D), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
flop = 4.0 * B * H * D * S * S / 2


def t(f, n=10):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402
res = {}
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel(be):
            f = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
            ms = t(f)
        res[name] = flop / ms / 1e9
    except Exception as e:  # noqa: BLE001
        res[name] = f"unavailable ({type(e).__name__}: {str(e)[:80]})"
ours = t(lambda: P.attention_fwd(q, k, v))
res["ours"] = flop / ours / 1e9
try:
    import flashinfer
    qf = q.transpose(1, 2).reshape(B * S, H, D).contiguous()
    kf = k.transpose(1, 2).reshape(B * S, H, D).contiguous()
    vf = v.transpose(1, 2).reshape(B * S, H, D).contiguous()
    qo = torch.arange(0, B + 1, device="cuda", dtype=torch.int32) * S
    ws = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend="auto")
    w.plan(qo, qo, H, H, D, causal=True, q_data_type=torch.bfloat16)
    ms = t(lambda: w.run(qf, kf, vf))
    res["flashinfer"] = flop / ms / 1e9
except Exception as e:  # noqa: BLE001
    res["flashinfer"] = f"unavailable ({type(e).__name__}: {str(e)[:120]})"
ours = t(lambda: P.attention_fwd(q, k, v))
res["ours_again"] = flop / ours / 1e9
for kk, vv in res.items():
    print(kk, vv if isinstance(vv, str) else f"{vv:.0f} TFLOPS")
