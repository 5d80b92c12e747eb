"""Pins for the oracle's secondary-uncertainty sampler (section 3):
SPEC worked examples, the paper's two extreme cases, an independent
scipy transcription of steps 1-5 + the beta quantile, and the closed-form mean
and standard deviation of the loss draw (mean mu_l, sd sigma_I+sigma_C: the
Beta(alpha,beta) of P:229-236 has mean mu_beta and variance sigma_beta^2)."""
import numpy as np
import pytest
import scipy.special as sp
import scipy.stats as st

import oracle as O


def test_beta_params_examples(golden):
    for c in golden["beta_params"]:
        a, b = O.beta_params(c["mu"], c["sigma"], c["max"])
        assert a == pytest.approx(c["alpha"], rel=1e-14), c["src"]
        assert b == pytest.approx(c["beta"], rel=1e-14), c["src"]


def test_beta_params_mean_variance_identity():
    rng = np.random.default_rng(4)
    for _ in range(200):
        mx = rng.uniform(1e4, 1e7)
        mu = mx * rng.uniform(0.05, 0.95)
        mub = mu / mx
        sig = mx * rng.uniform(0.01, 0.99) * np.sqrt(mub * (1 - mub))
        a, b = O.beta_params(mu, sig, mx)
        assert a / (a + b) == pytest.approx(mub, rel=1e-12)
        assert a * b / ((a + b) ** 2 * (a + b + 1)) == pytest.approx((sig / mx) ** 2, rel=1e-10)


def test_beta_params_cap():
    # sigma_beta >= sigma_max is replaced by a value very close (G9: 1-1e-6)
    a, b = O.beta_params(50.0, 60.0, 100.0)
    eps = 1e-6
    k = (1 / (1 - eps)) ** 2 - 1
    assert a == pytest.approx(0.5 * k, rel=1e-6) and b == pytest.approx(0.5 * k, rel=1e-6)
    assert 0 < a < 1e-5
    # exactly at the cap (inclusive reading)
    a2, _ = O.beta_params(25.0, 100 * np.sqrt(0.25 * 0.75), 100.0)
    assert 0 < a2 < 1e-5


def test_combine_examples_and_extremes(golden):
    for c in golden["combine"]:
        v, z, q = O.combine(c["zp"], c["ze"], c["si"], c["sc"])
        assert v == c["v"] and z == c["z"], c["src"]
    rng = np.random.default_rng(5)
    for _ in range(2000):
        zp, ze = rng.uniform(1e-7, 1 - 1e-7, 2)
        s = rng.uniform(0.1, 10)
        v, z, q = O.combine(zp, ze, 0.0, s)           # sigma_I = 0 => v = v_E
        assert v == pytest.approx(sp.ndtri(ze), abs=1e-12)
        v, z, q = O.combine(zp, ze, s, 0.0)           # sigma_C = 0 => v = v_Prog,E
        assert v == pytest.approx(sp.ndtri(zp), abs=1e-12)
        assert z == pytest.approx(sp.ndtr(v), rel=1e-13)
        assert q == pytest.approx(sp.ndtr(-v), rel=1e-13)


def test_combine_unit_variance():
    # v has unit variance when v_P, v_E are independent N(0,1)
    rng = np.random.default_rng(6)
    n = 200000
    zp, ze = rng.uniform(size=(2, n))
    si, sc = 3.0, 1.7
    vs = np.array([O.combine(a, b, si, sc)[0] for a, b in zip(zp[:20000], ze[:20000])])
    # the same linear map in numpy on all n (the transcription of P:196-217)
    sig = si + sc
    wi, wc = si / sig, sc / sig
    v_np = (sp.ndtri(zp) * wi + sp.ndtri(ze) * wc) / np.sqrt(wi * wi + wc * wc)
    np.testing.assert_allclose(vs, v_np[:20000], rtol=1e-12, atol=1e-12)
    assert 0.99 <= v_np.var() <= 1.01
    assert 0.97 <= vs.var() <= 1.03


def _scipy_sample(mu, si, sc, mx, zp, ze):
    """Independent transcription of P:196-248 with scipy special functions."""
    sig = si + sc
    if sig == 0:
        return mu
    if mu == 0:
        return 0.0
    if mu == mx:
        return mx
    sb, mb = sig / mx, mu / mx
    smax = np.sqrt(mb * (1 - mb))
    if sb >= smax:
        sb = smax * (1 - 1e-6)
    k = (smax / sb) ** 2 - 1
    a, b = mb * k, (1 - mb) * k
    wi, wc = si / sig, sc / sig
    v = (sp.ndtri(zp) * wi + sp.ndtri(ze) * wc) / np.sqrt(wi * wi + wc * wc)
    z, q = sp.ndtr(v), sp.ndtr(-v)
    if z <= 0.5:
        return mx * sp.betaincinv(a, b, z)
    return mx * (1 - sp.betaincinv(b, a, q))


def test_sample_loss_examples(golden):
    for c in golden["apply_su"]:
        got = O.sample_loss(c["mu"], c["si"], c["sc"], c["max"], c["zp"], c["ze"])
        assert got == pytest.approx(c["loss"], rel=1e-12), c["src"]
    assert O.sample_loss(0.0, 1.0, 1.0, 10.0, 0.3, 0.6) == 0.0       # G10
    assert O.sample_loss(10.0, 1.0, 1.0, 10.0, 0.3, 0.6) == 10.0     # G10


def test_sample_loss_vs_scipy_transcription():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        mu = 10 ** rng.uniform(4, 7)
        mx = (2 + 8 * rng.uniform()) * mu
        si = (0.1 + 0.4 * rng.uniform()) * mu
        sc = (0.05 + 0.25 * rng.uniform()) * mu
        zp, ze = (rng.integers(0, 2 ** 23, 2) * 2 + 1) * 2.0 ** -24
        got = O.sample_loss(mu, si, sc, mx, zp, ze)
        ref = _scipy_sample(mu, si, sc, mx, zp, ze)
        assert got == pytest.approx(ref, rel=1e-9, abs=1e-300)
        assert 0.0 <= got <= mx


def test_sample_monotone_in_zprog_when_sigma_c_zero():
    zs = np.linspace(0.001, 0.999, 300)
    xs = [O.sample_loss(3e5, 1e5, 0.0, 1.5e6, z, 0.123) for z in zs]
    assert all(b >= a for a, b in zip(xs, xs[1:]))


@pytest.mark.parametrize("rec", [
    (1.0e4, 0.3e4, 0.1e4, 2.5e4),
    (3.3e5, 0.5e5, 0.9e5, 3.0e6),
    (2.0e6, 0.45e6, 0.3e6, 4.5e6),
    (7.0e6, 2.1e6, 1.2e6, 1.4e7),
    (5.0e4, 0.2e4, 1.5e4, 9.0e5),
])
def test_sample_distribution_mean_sd_ks(rec):
    # closed form [derived]: loss = max_l * Beta(alpha,beta) has mean mu_l and sd
    # max_l*sigma_beta = sigma_I + sigma_C when z ~ U(0,1)
    mu, si, sc, mx = rec
    n = 100000
    rng = np.random.default_rng(int(mu) % 1000)
    zp, ze = rng.uniform(size=(2, n))
    x = O.sample_batch(mu, si, sc, mx, zp, ze)
    sd = si + sc
    assert abs(x.mean() - mu) < 4 * sd / np.sqrt(n)
    assert x.std() == pytest.approx(sd, rel=0.02)
    a, b = O.beta_params(mu, sd, mx)
    assert st.kstest(x / mx, st.beta(a, b).cdf).pvalue > 1e-4
    assert (x >= 0).all() and (x <= mx).all()


# ---- the sigma_beta cap regime (reading G9): alpha, beta in [1e-6, 1e-3] --
from mp_pins import mp_lower_quantile as _mp_lower_quantile  # noqa: E402


@pytest.mark.parametrize("a,b", [(1e-3, 1e-3), (5e-4, 1e-3), (1e-4, 3e-4), (2e-6, 1e-6), (1e-6, 1e-6),
                                 (1e-3, 3e-6)])
def test_quantile_cap_regime_vs_mpmath(a, b):
    # lower tail: the oracle's Newton/bisection against mpmath's I_x; values
    # far below 1e-300 round to 0 on both sides (the near-Bernoulli step)
    for p in (1e-3, 0.05, 0.3, 0.45, 0.49, 0.55, 0.7, 0.99):
        lower_mass = b / (a + b)                 # P(X -> 0) of the limiting Bernoulli
        if p < lower_mass:                       # solve directly (G13: z <= 1/2 side)
            x = O.beta_quantile(p, a, b)
            ref = _mp_lower_quantile(p, a, b)
            assert x == pytest.approx(ref, rel=1e-10, abs=1e-305), (a, b, p, x, ref)
        else:                                    # complementary equation I_y(b, a) = 1 - p
            y = O.beta_quantile(1.0 - p, b, a)
            ref = _mp_lower_quantile(1.0 - p, b, a)
            assert y == pytest.approx(ref, rel=1e-10, abs=1e-305), (a, b, p, y, ref)


def test_sample_loss_capped_records_vs_mpmath():
    # capped records (sigma >= sigma_max): the loss is max_l * x with
    # (alpha, beta) ~ 2e-6 (mu_beta, 1 - mu_beta); a near-Bernoulli draw whose
    # value is 0 / max_l except within ~1e-5 of the step -- each against mpmath
    for mu, si, sc, mx in [(30.0, 80.0, 0.0, 100.0), (50.0, 40.0, 30.0, 100.0), (80.0, 10.0, 90.0, 100.0),
                           (2.0e5, 3.0e5, 1.0e5, 1.0e6)]:
        a, b = O.beta_params(mu, si + sc, mx)
        assert 0 < a < 1e-5 and 0 < b < 1e-5
        for zp, ze in [(0.1, 0.2), (0.5, 0.5), (0.9, 0.3), (0.99, 0.95), (0.02, 0.97)]:
            got = O.sample_loss(mu, si, sc, mx, zp, ze)
            _, z, q = O.combine(zp, ze, si, sc)
            if z <= 0.5:
                ref = mx * _mp_lower_quantile(z, a, b)
            else:
                ref = mx * (1.0 - _mp_lower_quantile(q, b, a))
            assert got == pytest.approx(ref, rel=1e-10, abs=1e-300 * mx), (mu, si, sc, zp, ze, got, ref)
