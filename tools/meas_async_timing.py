"""Device time per ara_risk_measures_async call (queued back to back) for several
table sizes; ARA_MEAS_PER_BLOCK picks the grid (tools/gpu_*.sh sweeps it)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_2274_b200 import ara
ctx = ara.Context(0)
res = []
for n in (100000, 800000, 8000000):
    x = torch.from_numpy(np.random.default_rng(0).lognormal(15, 1.2, n).astype(np.float32)).cuda()
    out = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
    ref = ara.risk_measures_batch(ctx, x, 1, n, [0], rps=(100, 250, 500))
    for _ in range(5): ara.risk_measures_async(ctx, x, 1, n, [0], out=out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): ara.risk_measures_async(ctx, x, 1, n, [0], out=out)
    e1.record(); torch.cuda.synchronize()
    o = out.cpu().numpy()
    ok = np.array_equal(o[0, :, 0], ref[0][0]) and np.array_equal(o[0, :, 1], ref[1][0])
    res.append(f"n={n} {e0.elapsed_time(e1) / 100 * 1e3:.1f}us ok={ok}")
print(os.environ.get("ARA_MEAS_PER_BLOCK", "default"), " | ".join(res))
