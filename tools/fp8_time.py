import torch, os, sys, time
sys.path.insert(0, '/root/repo')
import paper_2605_10905_b200 as P
m=n=k=8192
dev='cuda'
qa = torch.randint(0, 120, (m, k), device=dev, dtype=torch.uint8)
qb = torch.randint(0, 120, (n, k), device=dev, dtype=torch.uint8)
sfa = torch.randint(120, 134, (m, k // 32), device=dev, dtype=torch.uint8)
sfb = torch.randint(120, 134, (n, k // 32), device=dev, dtype=torch.uint8)
c = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
L=P.lib(); s=torch.cuda.current_stream().cuda_stream
def step(): P._check(L.mimw_b200_gemm_mxfp8(qa.data_ptr(), sfa.data_ptr(), qb.data_ptr(), sfb.data_ptr(), c.data_ptr(), m, n, k, s))
for _ in range(5): step()
torch.cuda.synchronize()
for reps in (10, 30, 100):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter(); e0.record()
    for _ in range(reps): step()
    e1.record(); t1=time.perf_counter(); torch.cuda.synchronize()
    print(reps, 'gpu ms/step', e0.elapsed_time(e1)/reps, 'host us/call', (t1-t0)/reps*1e6)
