"""One analysis step (ara_run with ARA_ASYNC + ara_risk_measures_async) captured
into a CUDA graph and replayed, against the same step launched eagerly:
    python tools/graph_timing.py [cfg2|cfg3|cfg1] [steps]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import aragen
from paper_1310_2274_b200 import ara

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = aragen.load_config(name)
torch.cuda.set_device(0)
s = torch.cuda.Stream()
ctx = ara.Context(0, s)
pf = aragen.build_portfolio(cfg)
P = ara.Portfolio(ctx, pf)
yet = aragen.build_yet(cfg)
Y = ara.Yet.from_dict(ctx, yet)
L, N = cfg["n_layers"], cfg["n_trials"]
layers = list(range(L)) + ([-1] if L > 1 else [])
rps = cfg["return_periods"]
ylt = torch.empty((L, N), dtype=torch.float32, device="cuda")
out = torch.empty((len(layers), len(rps), 3), dtype=torch.float64, device="cuda")
ara.prepare(ctx, P, Y, su=cfg["su"], async_=True)


def step():
    ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], ylt=ylt, async_=True)
    ara.risk_measures_async(ctx, ylt, L, N, layers, rps=rps, out=out)


with torch.cuda.stream(s):
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ref_ylt, ref_out = ylt.clone(), out.clone()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(K):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / K
ctx.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()
ylt.zero_(); out.zero_()
with torch.cuda.stream(s):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ok = torch.equal(ylt, ref_ylt) and torch.equal(out, ref_out)
    e0.record(s)
    for _ in range(K):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / K
ctx.synchronize()
print(f"{name}: eager {eager * 1e3:.1f} us/step, graph {graph * 1e3:.1f} us/step, identical={ok}")
