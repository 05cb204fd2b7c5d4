"""torch.mm (cuBLAS) bf16 8192^3 on U[-1,1] operands, `n` launches: the
launch an ncu capture of cuBLAS's kernel is taken from (beside ours)."""
import sys
import torch

n = 8192
a = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
b = (torch.rand((n, n), device="cuda") * 2 - 1).bfloat16()
c = torch.empty((n, n), device="cuda", dtype=torch.bfloat16)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    torch.mm(a, b, out=c)
torch.cuda.synchronize()
