"""The shared input generator (aragen): determinism, slicing consistency (any
trial range or rank gives the same events), distinct events per XELT, the
value recipe's ranges, and that no generated record hits the sigma cap."""
import numpy as np
import pytest
import scipy.stats as st

import aragen


def small_cfg(**kw):
    cfg = aragen.load_config("cfg1")
    cfg.update(kw)
    return cfg


def test_yet_deterministic_and_sliceable():
    cfg = small_cfg()
    a = aragen.build_yet(cfg)
    b = aragen.build_yet(cfg, n_threads=3)
    assert np.array_equal(a["events"], b["events"])
    part = aragen.build_yet(cfg, first_trial=250, n_trials=300)
    K = cfg["events_per_trial"]
    assert np.array_equal(part["events"], a["events"][250 * K:550 * K])
    picked = aragen.yet_for_trials(cfg, [7, 999, 3])
    assert np.array_equal(picked["events"][:K], a["events"][7 * K:8 * K])
    assert np.array_equal(picked["events"][K:2 * K], a["events"][999 * K:1000 * K])
    assert a["events"].max() < cfg["catalog"]


def test_yet_uniform_chi2():
    cfg = small_cfg(n_trials=1000, events_per_trial=1000, catalog=100)
    ev = aragen.build_yet(cfg)["events"]
    counts = np.bincount(ev, minlength=100)
    assert st.chisquare(counts).pvalue > 0.01


def test_variable_length_trials():
    cfg = small_cfg(k_min=80, k_max=150)
    y = aragen.build_yet(cfg, first_trial=10, n_trials=50)
    lens = np.diff(y["trial_off"].astype(np.int64))
    assert lens.min() >= 80 and lens.max() <= 150 and len(set(lens.tolist())) > 5
    y2 = aragen.build_yet(cfg, first_trial=20, n_trials=10)
    s = int(y["trial_off"][10])
    assert np.array_equal(y2["events"], y["events"][s:s + y2["events"].size])


def test_portfolio_recipe():
    cfg = small_cfg(n_layers=2, elts_per_layer=3, records_per_elt=500, catalog=2000,
                    layer_terms=[[1e5, 5e6, 1e7, 2e7], [2e5, 5e6, 1e7, 2e7]])
    pf = aragen.build_portfolio(cfg)
    pf2 = aragen.build_portfolio(cfg)
    assert all(np.array_equal(pf[k], pf2[k]) for k in ("rec_event", "rec_mean", "rec_max"))
    R = 500
    for j in range(6):
        ev = pf["rec_event"][j * R:(j + 1) * R]
        assert len(set(ev.tolist())) == R and ev.max() < 2000
    mu = pf["rec_mean"].astype(np.float64)
    assert mu.min() >= 1e4 and mu.max() < 1e7
    r = pf["rec_max"] / pf["rec_mean"]
    assert r.min() >= 2 * (1 - 1e-6) and r.max() <= 10 * (1 + 1e-6)
    assert (pf["rec_sigma_i"] / mu).min() >= 0.1 * (1 - 1e-6)
    assert (pf["rec_sigma_c"] / mu).max() <= 0.3 * (1 + 1e-6)
    # no record reaches the sigma_beta cap: (fI + fC)^2 <= 0.64 < max/mu - 1
    sig = pf["rec_sigma_i"].astype(np.float64) + pf["rec_sigma_c"]
    mub = mu / pf["rec_max"]
    assert (sig / pf["rec_max"] < np.sqrt(mub * (1 - mub))).all()
    assert pf["layer_elts"].tolist() == list(range(6))
    assert pf["layer_terms"].shape == (2, 4)


def test_sigma_scale_zero_and_integer_mu():
    cfg = small_cfg(sigma_scale=0.0, integer_mu=True)
    pf = aragen.build_portfolio(cfg)
    assert (pf["rec_sigma_i"] == 0).all() and (pf["rec_sigma_c"] == 0).all()
    assert np.array_equal(pf["rec_mean"], np.round(pf["rec_mean"]))


def test_pack_yet_roundtrip():
    # the packed YET storage encoding: id x at bits [x*b, (x+1)*b), LSB first
    rng = np.random.default_rng(3)
    for bits in (1, 5, 14, 20, 21, 31, 32):
        n = 777 + bits
        ev = rng.integers(0, 2 ** bits, n, dtype=np.uint64).astype(np.uint32)
        w = aragen.pack_yet(ev, bits)
        assert w.size == (n * bits + 31) // 32
        big = int.from_bytes(w.tobytes(), "little")
        got = [(big >> (i * bits)) & ((1 << bits) - 1) for i in range(n)]
        assert np.array_equal(np.array(got, np.uint64), ev.astype(np.uint64))
    with pytest.raises(ValueError):
        aragen.pack_yet(np.array([1 << 20], np.uint32), 20)
    assert aragen.yet_bits(1_000_000) == 20 and aragen.yet_bits(2_000_000) == 21
    assert aragen.yet_bits(1 << 20) == 20 and aragen.yet_bits((1 << 20) + 1) == 21
