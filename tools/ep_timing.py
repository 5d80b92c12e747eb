import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1310_2274_b200 import ara
ctx = ara.Context(0)
for n in (100000, 800000, 8000000):
    x = torch.from_numpy(np.random.default_rng(0).lognormal(15, 1.2, n).astype(np.float32)).cuda()
    out = torch.empty(n, device='cuda')
    for _ in range(3): ara.exceedance_curve(ctx, x, 1, n, 0, out=out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ara.exceedance_curve(ctx, x, 1, n, 0, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(20): torch.sort(x, descending=True)
    t1.record(); torch.cuda.synchronize()
    print(n, "ep ms", round(ms, 4), "torch.sort ms", round(t0.elapsed_time(t1) / 20, 4))
