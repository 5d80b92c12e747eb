"""Trial sweep and phase attribution on one B200.

    python tools/sweep.py [--config cfg3] [--trials 200000,400000,600000,800000] [--runs 5]

The paper's Figures 1-2 time aggregate risk analysis with primary
uncertainty only and with secondary uncertainty for 200k..800k trials of
1,000 events, 1 layer x 16 XELTs, and expect both to scale linearly; Figure 12
 splits the 800k-trial time into (i) fetching events + lookup,
(ii) financial terms and other computation, (iii) secondary uncertainty.

Here, per trial count and per mode (SU off = mean losses, SU on), the device
times of the kernels of ara_run (CUDA events through ara_last_run_timings)
and of ara_risk_measures are reported, median of --runs after 2 warm-ups:
  compact  = YET stream + direct-access lookup (Fig 12 part i)
  sample   = draws + beta quantile + XELT/occurrence/aggregate terms -> YLT
             (parts ii + iii; SU off leaves only part ii)
  measures = PML/TVaR select + tail sort
One JSON line per (trials, mode); a last line with the linear fits.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import aragen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--trials", default="200000,400000,600000,800000")
    ap.add_argument("--runs", type=int, default=5)
    a = ap.parse_args()
    import torch
    from paper_1310_2274_b200 import ara
    cfg = aragen.load_config(a.config)
    counts = [int(x) for x in a.trials.split(",")]
    nmax = max(counts)
    K = int(cfg["events_per_trial"])
    ctx = ara.Context(0)
    P = ara.Portfolio(ctx, aragen.build_portfolio(cfg))
    ev = torch.empty(nmax * K, dtype=torch.int32).pin_memory()
    aragen.build_yet(cfg, first_trial=0, n_trials=nmax, out=ev.numpy().view(np.uint32))
    rows = []
    for n in counts:
        Y = ara.Yet(ctx, ev[: n * K], fixed_len=K, first_trial=0, n_trials=n)
        for su in (False, True):
            comp, samp, meas, tot = [], [], [], []
            ylt = torch.empty((1, n), dtype=torch.float32, device="cuda")
            for r in range(a.runs + 2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                ara.run(ctx, P, Y, seed=cfg["seed"], su=su, ylt=ylt)
                t = ara.last_run_timings(ctx)
                m0 = torch.cuda.Event(enable_timing=True)
                m0.record()
                ara.risk_measures(ctx, ylt, 1, n, 0, rps=cfg["return_periods"])
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    comp.append(t["compact_ms"]); samp.append(t["sample_ms"])
                    meas.append(m0.elapsed_time(e1)); tot.append(e0.elapsed_time(e1))
            row = {"trials": n, "su": su, "compact_ms": statistics.median(comp),
                   "sample_ms": statistics.median(samp), "measures_ms": statistics.median(meas),
                   "step_ms": statistics.median(tot)}
            row["trials_per_s"] = n / (row["step_ms"] * 1e-3)
            rows.append(row)
            print(json.dumps(row), flush=True)
        del Y
    fits = {}
    for su in (False, True):
        x = np.array([r["trials"] for r in rows if r["su"] == su], np.float64)
        for k in ("compact_ms", "sample_ms", "step_ms"):
            y = np.array([r[k] for r in rows if r["su"] == su])
            slope, icpt = np.polyfit(x, y, 1)
            resid = y - (slope * x + icpt)
            fits[f"{'su' if su else 'primary'}_{k}"] = {
                "ms_per_100k_trials": slope * 1e5, "intercept_ms": icpt,
                "max_rel_resid": float(np.max(np.abs(resid) / y))}
    at = {su: next(r for r in rows if r["trials"] == nmax and r["su"] == su) for su in (False, True)}
    fits["su_over_primary_at_max"] = at[True]["step_ms"] / at[False]["step_ms"]
    fits["config"] = a.config
    print(json.dumps({"fits": fits}))


if __name__ == "__main__":
    main()
