"""Per-item overhead of the FA forward: non-causal attention at equal total
work with shorter rows (items of 2 Q tiles x S/128 KV tiles).  If the rate
falls as S shrinks, the per-item prologue/epilogue is not hidden."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

for s, bh in ((8192, 128), (4096, 512), (2048, 2048), (1024, 8192)):
    q, k, v = ((torch.rand((1, bh, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
    for causal in (False, True):
        f = lambda: P.attention_fwd(q, k, v, causal=causal)  # noqa: E731
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        flop = 4.0 * 128 * bh * s * (s if not causal else (s + 1) / 2)
        print(f"S={s:5d} BH={bh:5d} {'causal' if causal else 'full  '} {ms:7.3f} ms {flop / ms / 1e9:6.0f} TFLOPS")
    del q, k, v
