"""Pins for the oracle's RNG and special functions (readings G1, G4,
G11, G12) against things other than itself: Random123 known-answer vectors,
SPEC.md worked examples, closed forms, scipy and mpmath."""
import math

import mpmath
import numpy as np
import pytest
import scipy.special as sp

import oracle as O


def test_philox_kat(golden):
    for case in golden["philox4x32_10"]:
        ctr = [int(x, 16) for x in case["ctr"]]
        key = [int(x, 16) for x in case["key"]]
        out = [int(x, 16) for x in case["out"]]
        assert list(O.philox4x32_10(ctr, key)) == out, case["src"]


def test_uniform_map_exact():
    # U(x) = (2(x>>9)+1) 2^-24 (G4): extremes, symmetry, fp32 exactness.
    assert O.u01(0) == 2.0 ** -24
    assert O.u01(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    rng = np.random.default_rng(1)
    for x in rng.integers(0, 2 ** 32, 2000, dtype=np.uint64):
        u = O.u01(int(x))
        assert float(np.float32(u)) == u
        m = int(x) >> 9
        mirror = (2 ** 23 - 1 - m) << 9
        assert O.u01(mirror) + u == 1.0
        assert 0.0 < u < 1.0


def test_z_keys_differ_by_tag_and_index():
    s = 12345
    a = O.z_prog(s, 0, 7, 3)
    b = O.z_event(s, 7, 3, 0)
    assert a != b           # tags 1 and 2 are different streams
    assert O.z_event(s, 7, 3, 1) != b
    assert O.z_event(s, 8, 3, 0) != b
    # reproducible
    assert O.z_event(s, 7, 3, 0) == b


def test_normal_examples(golden):
    for c in golden["normal_cdf"]:
        assert O.norm_cdf(c["x"]) == pytest.approx(c["y"], abs=c.get("tol", 0) or 1e-15), c["src"]
    for c in golden["normal_quantile"]:
        assert O.norm_quantile(c["p"]) == pytest.approx(c["y"], abs=c.get("tol", 0) or 1e-15), c["src"]


def test_normal_vs_scipy_and_mpmath():
    ps = np.concatenate([10.0 ** -np.arange(1, 16), [0.01, 0.1, 0.2, 0.3, 0.4, 0.45, 0.49999]])
    ps = np.concatenate([ps, 1 - ps[ps > 1e-14]])
    for p in ps:
        x = O.norm_quantile(p)
        assert x == pytest.approx(sp.ndtri(p), rel=2e-14, abs=1e-15)
    # deep tails against mpmath at 40 digits
    mpmath.mp.dps = 40
    for p in [2.0 ** -24, 3.5e-14, 1e-10]:
        ref = float(-mpmath.sqrt(2) * mpmath.erfinv(1 - 2 * mpmath.mpf(p)))
        assert O.norm_quantile(p) == pytest.approx(ref, rel=1e-14)
    for v in np.linspace(-8, 8, 161):
        # conditioning of Phi at v: relative error ~ v^2 * eps in the argument
        ref = float(mpmath.ncdf(mpmath.mpf(float(v))))
        assert O.norm_cdf(v) == pytest.approx(ref, rel=4e-16 * (1 + v * v), abs=1e-300)
        assert O.norm_cdf(v) == pytest.approx(1 - O.norm_cdf(-v), abs=1e-15)


def test_normal_round_trip():
    # S:57 round trip |q(Phi(x)) - x| <= 1e-9 for |x| <= 6, taken on the lower
    # tail (Phi(x) for x > 0 is within 1e-16 of 1 in fp64, so x > 0 goes
    # through the antisymmetry q(1-p) = -q(p) instead).
    for x in np.linspace(-6, 6, 241):
        if x <= 0:
            assert O.norm_quantile(O.norm_cdf(x)) == pytest.approx(x, abs=1e-9)
        else:
            assert -O.norm_quantile(O.norm_cdf(-x)) == pytest.approx(x, abs=1e-9)


def test_lnbeta_examples(golden):
    for c in golden["ln_beta"]:
        assert O.lnbeta(c["a"], c["b"]) == pytest.approx(c["y"], abs=1e-14), c["src"]
    for a, b in [(0.3, 346.0), (39.0, 0.31), (4.4375, 13.3125)]:
        assert O.lnbeta(a, b) == pytest.approx(float(sp.betaln(a, b)), rel=1e-13)


def test_beta_cdf_examples_and_closed_forms(golden):
    for c in golden["beta_cdf"]:
        assert O.beta_cdf(c["x"], c["a"], c["b"]) == pytest.approx(c["y"], abs=1e-15), c["src"]
    for x in np.linspace(0.01, 0.99, 25):
        assert O.beta_cdf(x, 2, 2) == pytest.approx(3 * x * x - 2 * x ** 3, rel=1e-13)
        assert O.beta_cdf(x, 3.5, 1) == pytest.approx(x ** 3.5, rel=1e-13)
        assert O.beta_cdf(x, 1, 2.5) == pytest.approx(1 - (1 - x) ** 2.5, rel=1e-13)
        assert O.beta_cdf(x, 0.5, 0.5) == pytest.approx(2 / math.pi * math.asin(math.sqrt(x)), rel=1e-13)
        # reflection identity
        assert O.beta_cdf(x, 2.7, 11.0) == pytest.approx(1 - O.beta_cdf(1 - x, 11.0, 2.7), abs=1e-14)
    assert O.beta_cdf(0.0, 2, 3) == 0.0 and O.beta_cdf(1.0, 2, 3) == 1.0


def test_beta_cdf_vs_scipy_and_quadrature():
    rng = np.random.default_rng(2)
    for _ in range(400):
        a, b = 10 ** rng.uniform(-1, 2, 2)
        x = rng.uniform(0.001, 0.999)
        assert O.beta_cdf(x, a, b) == pytest.approx(float(sp.betainc(a, b, x)), rel=1e-11, abs=1e-300)
    mpmath.mp.dps = 30
    for a, b, x in [(0.3, 346.0, 2e-4), (39.0, 0.31, 0.995), (2.5, 7.5, 0.3)]:
        ref = float(mpmath.betainc(a, b, 0, x, regularized=True))
        assert O.beta_cdf(x, a, b) == pytest.approx(ref, rel=1e-12)


def test_beta_quantile_examples(golden):
    for c in golden["beta_quantile"]:
        assert O.beta_quantile(c["p"], c["a"], c["b"]) == pytest.approx(c["y"], rel=1e-12), c["src"]


def test_beta_quantile_closed_forms():
    for p in [1e-12, 1e-6, 0.01, 0.2, 0.5, 0.8, 0.99]:
        assert O.beta_quantile(p, 3.2, 1.0) == pytest.approx(p ** (1 / 3.2), rel=1e-12)
        assert O.beta_quantile(p, 1.0, 4.5) == pytest.approx(1 - (1 - p) ** (1 / 4.5), rel=1e-12)
        assert O.beta_quantile(p, 0.5, 0.5) == pytest.approx(math.sin(math.pi * p / 2) ** 2, rel=1e-12)
        x = O.beta_quantile(p, 2.0, 2.0)
        assert 3 * x * x - 2 * x ** 3 == pytest.approx(p, rel=1e-12)
    for a in [0.4, 1.0, 7.0, 150.0]:
        assert O.beta_quantile(0.5, a, a) == pytest.approx(0.5, rel=1e-12)


def test_beta_quantile_vs_scipy_generator_range():
    # the generator's (alpha, beta) range (DESIGN.md input recipe): a in [0.3, 39], b in [0.31, 346]
    rng = np.random.default_rng(3)
    worst, iters = 0.0, []
    for _ in range(3000):
        a = 10 ** rng.uniform(np.log10(0.3), np.log10(39))
        b = 10 ** rng.uniform(np.log10(0.31), np.log10(346))
        p = 10 ** rng.uniform(-14, np.log10(0.5))
        x, it = O.beta_quantile(p, a, b, return_iters=True)
        iters.append(it)
        worst = max(worst, abs(x / sp.betaincinv(a, b, p) - 1))
    assert worst < 1e-10
    assert max(iters) < 200


def test_beta_quantile_round_trip_grid():
    for a in [0.3, 1.0, 3.0, 30.0, 300.0]:
        for b in [0.3, 1.0, 5.0, 50.0, 350.0]:
            for p in [1e-10, 1e-4, 0.1, 0.5, 0.9]:
                x = O.beta_quantile(p, a, b)
                assert O.beta_cdf(x, a, b) == pytest.approx(p, rel=1e-9, abs=1e-10)


def test_beta_quantile_tail_mpmath():
    # the oracle's x brackets the 40-digit root: I(x(1-1e-10)) < p < I(x(1+1e-10))
    mpmath.mp.dps = 40
    for a, b, p in [(0.35, 120.0, 1e-5), (0.3, 346.0, 1e-12), (2.0, 300.0, 3.5e-14)]:
        x = mpmath.mpf(O.beta_quantile(p, a, b))
        I = lambda t: mpmath.betainc(a, b, 0, t, regularized=True)
        assert I(x * (1 - mpmath.mpf(1e-10))) < p < I(x * (1 + mpmath.mpf(1e-10)))


def test_beta_quantile_monotone_in_p():
    ps = np.linspace(1e-6, 1 - 1e-6, 400)
    xs = [O.beta_quantile(p, 0.7, 9.0) for p in ps]
    assert all(x2 >= x1 for x1, x2 in zip(xs, xs[1:]))
