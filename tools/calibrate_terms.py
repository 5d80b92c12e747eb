"""Calibrate the aggregate layer terms of each config from an oracle pilot.

Writes AggR = q_0.10(S) and AggL = q_hi(S) - AggR (q_hi = the config's
``agg_limit_quantile``: 0.999, or 0.95 for cfg1 so the limit binds in 5 % of
its trials), rounded to 3 significant digits, where S is the oracle's gross
(pre-aggregate-terms) trial loss over a pilot of up to 10k trials
(SURVEY.md section 8(d)).  Calls only ``oracle/`` and ``aragen/``; the stored
values therefore never come from the CUDA path.

    python tools/calibrate_terms.py [cfg1 cfg2 ...]
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import aragen  # noqa: E402
import oracle  # noqa: E402

PILOT = 10000


def round3(x):
    if x <= 0:
        return 0.0
    e = math.floor(math.log10(x)) - 2
    return float(round(x / 10 ** e) * 10 ** e)


def calibrate(name):
    cfg = aragen.load_config(name)
    n = min(PILOT, int(cfg["n_trials"]))
    pf = aragen.build_portfolio(cfg)
    terms = pf["layer_terms"].copy()
    terms[:, 2] = 0.0
    terms[:, 3] = np.inf
    pf["layer_terms"] = terms
    yet = aragen.build_yet(cfg, 0, n)
    t = time.time()
    out = oracle.run(pf, yet, seed=int(cfg["seed"]), su=bool(cfg["su"]))
    qhi = float(cfg["agg_limit_quantile"])
    new = []
    for li in range(int(cfg["n_layers"])):
        S = out["gross"][li]
        agg_r = round3(float(np.quantile(S, 0.10)))
        agg_l = round3(float(np.quantile(S, qhi)) - agg_r)
        new.append([float(cfg["layer_terms"][li][0]), float(cfg["layer_terms"][li][1]), agg_r, agg_l])
    cfg["layer_terms"] = new
    cfg["calibration"] = {"pilot_trials": n, "script": "tools/calibrate_terms.py",
                          "rule": f"AggR=q0.10(S), AggL=q{qhi}(S)-AggR, 3 s.f., oracle gross S"}
    with open(os.path.join(aragen.CONFIG_DIR, f"{name}.json"), "w") as f:
        json.dump(cfg, f, indent=1)
    print(f"{name}: {new}  ({time.time() - t:.1f}s oracle)")


if __name__ == "__main__":
    for nm in (sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]):
        calibrate(nm)
