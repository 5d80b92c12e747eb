import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1310_2274_b200 import ara
ctx = ara.Context(0)
for n in (100000, 800000):
    x = torch.from_numpy(np.random.default_rng(0).lognormal(15, 1.2, n).astype(np.float32)).cuda()
    for _ in range(5): ara.risk_measures(ctx, x, 1, n, 0, rps=(100, 250, 500))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): ara.risk_measures(ctx, x, 1, n, 0, rps=(100, 250, 500))
    t1 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): ara.risk_measures(ctx, x, 1, n, 0, rps=(100, 250, 500))
    e1.record(); torch.cuda.synchronize()
    print(n, "host us/call", (t1 - t0) / 200 * 1e6, "event us/call", e0.elapsed_time(e1) / 200 * 1e3)
