"""Run the fused scan on a (possibly truncated) config for ncu profiling.

    ncu --set full -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/prof \
        python tools/profile_scan.py --config cfg3 --trials 100000
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import aragen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--trials", type=int, default=100000)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--measures", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_1310_2274_b200 import ara
    cfg = aragen.load_config(a.config)
    cfg["n_trials"] = min(a.trials, cfg["n_trials"])
    pf = aragen.build_portfolio(cfg)
    yet = aragen.build_yet(cfg)
    ctx = ara.Context(0)
    P = ara.Portfolio(ctx, pf)
    Y = ara.Yet.from_dict(ctx, yet)
    for _ in range(a.runs):
        ylt = ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"])
        if a.measures:
            ara.risk_measures(ctx, ylt, cfg["n_layers"], cfg["n_trials"], 0, rps=cfg["return_periods"])
    torch.cuda.synchronize()
    _, cnt, _ = ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], debug=True)   # after the profiled launches
    print(f"trials={cfg['n_trials']} present_pairs={int(cnt.sum().item())} ylt_mean={float(ylt.mean()):.6g}")


if __name__ == "__main__":
    main()
