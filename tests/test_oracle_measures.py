"""Pins for the oracle's PML / TVaR (SPEC conventions S:345-387,
readings G13b, G16, G17): SPEC worked examples, constants, the analytic
truncated-normal tail expectation, permutation invariance, scale equivariance,
monotonicity, integer index arithmetic."""
import math

import numpy as np
import pytest
import scipy.stats as st

from oracle import measures as M


def test_exceedance_curve_example(golden):
    c = golden["exceedance_curve"][0]
    d, p = M.exceedance_curve(c["ylt"])
    assert d.tolist() == c["sorted"] and p.tolist() == c["p"], c["src"]


def test_pml_endpoint_example(golden):
    c = golden["pml"][0]
    ylt = np.random.default_rng(0).uniform(size=c["ylt_n"])
    assert M.pml(ylt, c["rp"]) == ylt.max(), c["src"]


def test_pml_interpolation_by_hand():
    # 5-point curve [50, 40, 30, 20, 10]; rp with r = (N+1)/rp = 2.5 -> midway L(2), L(3)
    ylt = [10, 30, 50, 20, 40]
    assert M.pml(ylt, 6 / 2.5) == pytest.approx(35.0)
    assert M.pml(ylt, 3) == 40.0          # r = 2 exactly -> L(2)
    assert M.pml(ylt, 1.1) == 10.0        # r >= N -> L(N)


def test_tvar_examples(golden):
    c = golden["tvar"][0]
    var, tv = M.var_tvar_q(c["ylt"], c["q"])
    assert (var, tv) == (c["var"], c["tvar"]), c["src"]
    assert M.tvar_rp(c["ylt"], 4) == (c["var"], c["tvar"])
    c = golden["tvar"][1]
    x = np.maximum(np.random.default_rng(42).standard_normal(100000), 0.0)
    _, tv = M.var_tvar_q(x, c["q"])
    assert tv == pytest.approx(c["tvar"], rel=c["rtol"]), c["src"]
    z = st.norm.ppf(c["q"])
    assert c["tvar"] == pytest.approx(st.norm.pdf(z) / (1 - c["q"]), rel=1e-12)


def test_constant_ylt():
    ylt = np.full(1000, 7.25)
    for rp in (2, 100, 250, 500, 1001):
        assert M.pml(ylt, rp) == 7.25
        assert M.tvar_rp(ylt, rp) == (7.25, 7.25)


def test_properties():
    rng = np.random.default_rng(1)
    ylt = rng.lognormal(10, 1, 20011)
    ylt[:50] = 0.0
    perm = rng.permutation(ylt)
    prev_p, prev_t = -1, -1
    for rp in (2, 10, 100, 250, 500, 1000):
        p, (v, t) = M.pml(ylt, rp), M.tvar_rp(ylt, rp)
        assert p == M.pml(perm, rp) and (v, t) == M.tvar_rp(perm, rp)
        assert M.pml(3.5 * ylt, rp) == pytest.approx(3.5 * p, rel=1e-15)
        assert M.tvar_rp(3.5 * ylt, rp)[1] == pytest.approx(3.5 * t, rel=1e-14)
        assert t >= v
        assert p >= prev_p and t >= prev_t
        prev_p, prev_t = p, t


def test_integer_rank_arithmetic():
    # G13b: N = 800k, RP = 100 -> VaR descending rank 8000, PML r = 8000.01
    n = 800000
    ylt = np.arange(n, 0, -1, dtype=np.float64)        # descending rank i has value n-i+1
    v, _ = M.tvar_rp(ylt, 100)
    assert v == n - 8000 + 1
    p = M.pml(ylt, 100)
    assert p == pytest.approx((n - 8000 + 1) - 0.01, abs=1e-9)
    # the floating formula floor((1-1/RP) N) agrees for divisible N (G13b)
    for N in (1000, 100000, 800000, 1000000):
        for RP in (100, 250, 500):
            assert N - math.floor((1 - 1 / RP) * N) == -(-N // RP)


def test_domain_errors():
    with pytest.raises(ValueError):
        M.pml([], 100)
    with pytest.raises(ValueError):
        M.pml([1.0], 1.0)
    with pytest.raises(ValueError):
        M.tvar_rp([1.0], 0.5)


def test_rollup():
    y = np.array([[1.0, 2.0, 3.0], [10.0, 0.0, 5.0]])
    assert M.rollup(y).tolist() == [11.0, 2.0, 8.0]
