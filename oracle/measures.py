"""PML / VaR / TVaR from a Year Loss Table by a full sort (oracle side).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.

The paper names PML and TVaR (section 2.4) but gives no formulas
(reading G17).  We adopt SPEC.md's conventions, pinned by its worked examples
(tests/test_oracle_measures.py):

* exceedance curve: YLT sorted descending L(1) >= ... >= L(N), p_i = i/(N+1)
  (S:347);
* PML(RP): r = (N+1)/RP; r <= 1 -> L(1); r >= N -> L(N); else linear
  interpolation L(fl r) + (r - fl r)(L(fl r + 1) - L(fl r));
* VaR_q: the upper order statistic, ascending x(floor(qN)+1), clamped to N
  (S:376); TVaR_q = mean of all entries >= VaR_q, ties included;
  at a return period q = 1 - 1/RP;
* integer return periods use integer index arithmetic (reading G13b):
  fl r = (N+1)//RP, frac = ((N+1) % RP)/RP, and the VaR descending rank is
  m = ceil(N/RP);
* the portfolio roll-up is YLT_PF[i] = sum over layers of YLT[l][i] (G16).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["exceedance_curve", "pml", "var_tvar_q", "tvar_rp", "rollup", "risk_measures"]


def exceedance_curve(ylt):
    """(losses sorted descending, exceedance probabilities i/(N+1))."""
    x = np.asarray(ylt, dtype=np.float64)
    if x.size == 0:
        raise ValueError("empty YLT")
    d = np.sort(x)[::-1]
    p = np.arange(1, d.size + 1, dtype=np.float64) / (d.size + 1)
    return d, p


def pml(ylt, rp):
    """Probable Maximum Loss at return period ``rp`` (> 1)."""
    if not rp > 1:
        raise ValueError("return period must be > 1")
    d, _ = exceedance_curve(ylt)
    n = d.size
    if float(rp).is_integer():
        rp = int(rp)
        fl, frac = (n + 1) // rp, ((n + 1) % rp) / rp
    else:
        r = (n + 1) / rp
        fl = math.floor(r)
        frac = r - fl
    if fl < 1 or (fl == 1 and frac == 0):
        return float(d[0])
    if fl >= n:
        return float(d[n - 1])
    lo, hi = d[fl - 1], d[fl]          # L(fl), L(fl+1) with 1-based ranks
    return float(lo + frac * (hi - lo))


def var_tvar_q(ylt, q):
    """(VaR_q, TVaR_q) with the upper-order-statistic convention."""
    if not 0.0 < q < 1.0:
        raise ValueError("q must lie in (0,1)")
    x = np.sort(np.asarray(ylt, dtype=np.float64))
    if x.size == 0:
        raise ValueError("empty YLT")
    n = x.size
    a = min(int(math.floor(q * n)) + 1, n)     # ascending 1-based index
    var = x[a - 1]
    tail = x[x >= var][::-1]              # ties below index a included; descending sum
    return float(var), float(tail.sum() / tail.size)


def tvar_rp(ylt, rp):
    """(VaR, TVaR) at return period ``rp``: q = 1 - 1/rp, integer ranks (G13b)."""
    if not rp > 1:
        raise ValueError("return period must be > 1")
    x = np.asarray(ylt, dtype=np.float64)
    if x.size == 0:
        raise ValueError("empty YLT")
    if not float(rp).is_integer():
        return var_tvar_q(x, 1.0 - 1.0 / rp)
    n = x.size
    m = max(1, min(n, -(-n // int(rp))))        # descending rank ceil(N/RP)
    d = np.sort(x)[::-1]
    var = d[m - 1]
    tail = d[d >= var]                    # descending order: permutation-invariant sum
    return float(var), float(tail.sum() / tail.size)


def rollup(ylt_layers):
    """Portfolio YLT: sum over layers, per trial (reading G16)."""
    return np.asarray(ylt_layers, dtype=np.float64).sum(axis=0)


def risk_measures(ylt, rps=(100, 250, 500)):
    """dict rp -> (PML, TVaR) for one YLT vector."""
    out = {}
    for rp in rps:
        out[rp] = (pml(ylt, rp), tvar_rp(ylt, rp)[1])
    return out
