import torch, sys
sys.path.insert(0, '.')
import paper_2605_10905_b200 as P
g = torch.Generator(device="cuda").manual_seed(5)
for shape in [(2,3,1100), (1,1,512), (1,2,256)]:
    b,h,s = shape
    q, k, v = ((torch.rand((b, h, s, 128), device="cuda", generator=g) * 2 - 1).bfloat16() for _ in range(3))
    ref_o, ref_l = P.attention_fwd(q, k, v)
    torch.cuda.synchronize()
    for ctas in (13, 5, 2, 1):
        try:
            o, l = P.attention_fwd(q, k, v, max_ctas=ctas); torch.cuda.synchronize()
            print(shape, ctas, torch.equal(o, ref_o), torch.equal(l, ref_l), flush=True)
        except Exception as e:
            print(shape, ctas, 'ERR', str(e)[:100], flush=True); raise
