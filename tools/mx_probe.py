import torch, time, inspect
m=n=k=8192
a = torch.randn(m, k, device='cuda').to(torch.float8_e4m3fn)
b = torch.randn(n, k, device='cuda').to(torch.float8_e4m3fn)
def timeit(f, it=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/it
print(torch.__version__, hasattr(torch.nn.functional, 'scaled_mm'))
try:
    from torch.nn.functional import ScalingType, SwizzleType
    print([x for x in dir(ScalingType) if not x.startswith('_')], [x for x in dir(SwizzleType) if not x.startswith('_')])
except Exception as e: print('no enums', e)
# blocked (swizzled) e8m0 scales: 128x4 blocks
def to_blocked(sc):
    rows, cols = sc.shape
    n_rb, n_cb = (rows + 127)//128, (cols + 3)//4
    blocks = sc.view(n_rb, 128, n_cb, 4).permute(0, 2, 1, 3)
    rb = blocks.reshape(-1, 4, 32, 4).transpose(1, 2).reshape(-1, 32, 16)
    return rb.flatten()
sa = torch.full((m, k//32), 127, device='cuda', dtype=torch.uint8).view(torch.float8_e8m0fnu)
sb = torch.full((n, k//32), 127, device='cuda', dtype=torch.uint8).view(torch.float8_e8m0fnu)
for name, fn in [
  ('_scaled_mm blocked', lambda: torch._scaled_mm(a, b.t(), to_blocked(sa.view(torch.uint8)).view(torch.float8_e8m0fnu), to_blocked(sb.view(torch.uint8)).view(torch.float8_e8m0fnu), out_dtype=torch.bfloat16)),
  ('_scaled_mm plain', lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)),
]:
    try:
        ms = timeit(fn); print(name, ms, 2*m*n*k/ms/1e9, 'TF')
    except Exception as e: print(name, 'ERR', str(e)[:200])
try:
    from torch.nn.functional import scaled_mm, ScalingType, SwizzleType
    f = lambda: scaled_mm(a, b.t(), sa, ScalingType.BlockWise1x32, sb, ScalingType.BlockWise1x32, swizzle_a=SwizzleType.SWIZZLE_32_4_4, swizzle_b=SwizzleType.SWIZZLE_32_4_4, output_dtype=torch.bfloat16)
    ms = timeit(f); print('F.scaled_mm mx', ms, 2*m*n*k/ms/1e9)
except Exception as e: print('F.scaled_mm ERR', str(e)[:300])
one = torch.ones((), device='cuda')
ms = timeit(lambda: torch._scaled_mm(a, b.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16)); print('per-tensor', ms, 2*m*n*k/ms/1e9)
