"""One table's measures, for an ncu capture of select_multi_kernel."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_2274_b200 import ara
ctx = ara.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
x = torch.from_numpy(np.random.default_rng(0).lognormal(15, 1.2, n).astype(np.float32)).cuda()
out = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
for _ in range(3): ara.risk_measures_async(ctx, x, 1, n, [0], out=out)
torch.cuda.synchronize()
