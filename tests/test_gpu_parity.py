"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
the same seeded inputs.

Bars: lookup counts and hashes bit-exact; uniforms
bit-exact; YLT entry-wise |g - o| <= 1e-4 |o| + 1e-6 S_o (S_o = the
oracle's gross trial sum, the floor near the aggregate-retention clip);
PML / TVaR within 1e-4 relative (+ the same floor); sigma = 0 with
integer means bit-exact."""
import numpy as np
import pytest

import aragen
import oracle
from oracle import measures as OM

pytestmark = pytest.mark.gpu

REL, FLOOR = 1e-4, 1e-6


@pytest.fixture(scope="module")
def A():
    import torch
    assert torch.cuda.is_available()
    from paper_1310_2274_b200 import ara
    return ara


@pytest.fixture(scope="module")
def ctx(A):
    return A.Context(0)


def ylt_check(g, ref, li=None):
    o, S = ref["ylt"], ref["gross"]
    if li is not None:
        o, S = o[li], S[li]
    g = np.asarray(g, np.float64)
    err = np.abs(g - o)
    tol = REL * np.abs(o) + FLOOR * S
    bad = err > tol
    assert not bad.any(), (f"{bad.sum()} of {bad.size} YLT entries out of tolerance; worst "
                           f"{(err / np.maximum(tol, 1e-300)).max():.3g}x tol")
    nz = o > 0
    return float((err[nz] / o[nz]).max()) if nz.any() else 0.0


def run_both(A, ctx, pf, yet, seed, su=True, trial_index=None):
    P = A.Portfolio(ctx, pf)
    Y = A.Yet.from_dict(ctx, yet)
    ylt, cnt, hsh = A.run(ctx, P, Y, seed=seed, su=su, debug=True)
    ref = oracle.run(pf, yet, seed=seed, su=su, trial_index=trial_index)
    return (ylt.cpu().numpy(), cnt.cpu().numpy().astype(np.uint32),
            hsh.cpu().numpy().view(np.uint64)), ref


# ---- row a3: draws ----------------------------------------------------------
def test_uniforms_bit_exact(A, ctx):
    rng = np.random.default_rng(0)
    n = 20000
    ctr = np.stack([rng.integers(0, 2 ** 32, n), rng.integers(0, 2 ** 32, n),
                    rng.integers(0, 256, n), rng.integers(1, 3, n)], 1).astype(np.uint32)
    seed = 0x123456789ABCDEF
    u = A.draw_uniforms(ctx, seed, ctr)
    for t in range(0, n, 37):
        i, k, j, tag = (int(x) for x in ctr[t])
        ref = oracle.z_prog(seed, j, i, k) if tag == 1 else oracle.z_event(seed, i, k, j)
        assert float(u[t]) == ref


# ---- row a4, step 2: v = Phi^-1(U(x)) as the kernels take it -------------------
def test_normal_quantiles_vs_oracle(A, ctx):
    # every tail value down to 2^-24 for the first 2^13 grid points of each
    # tail, then a stride through the body; both halves of the 32-bit word
    m = np.concatenate([np.arange(0, 1 << 13), np.arange(1 << 13, 1 << 22, 61)]).astype(np.uint64)
    m = np.concatenate([m, (1 << 23) - 1 - m])
    bits = (m << 9 | (m * 2654435761 & 0x1FF)).astype(np.uint32)      # low 9 bits are ignored
    v = A.normal_quantiles(ctx, bits).astype(np.float64)
    ref = np.array([oracle.norm_quantile((2.0 * float(x) + 1.0) * 2.0 ** -24) for x in m])
    err = np.abs(v - ref)
    # fp32 result: relative 4e-7 (erfcinvf's 4 ulp), absolute 1e-7 near v = 0
    assert np.all(err <= 4e-7 * np.abs(ref) + 1e-7), f"worst {err.max()} at v={ref[err.argmax()]}"
    assert np.all(np.sign(v) == np.sign(ref))


# ---- rows a4-a6: the sampler ---------------------------------------------------
def gen_records(n, seed=0):
    cfg = aragen.load_config("cfg3")
    cfg.update(records_per_elt=n, catalog=max(n, 1000))
    pf = aragen.build_portfolio(cfg)
    from paper_1310_2274_b200 import ara
    recs = np.empty(n, ara.RECORD_DTYPE)
    recs["event_id"] = 0
    recs["mean_loss"] = pf["rec_mean"][:n]
    recs["sigma_i"] = pf["rec_sigma_i"][:n]
    recs["sigma_c"] = pf["rec_sigma_c"][:n]
    recs["max_loss"] = pf["rec_max"][:n]
    return recs


def grid_uniforms(rng, n):
    return ((rng.integers(0, 2 ** 23, n) * 2 + 1) * 2.0 ** -24).astype(np.float32)


def test_sampler_vs_oracle(A, ctx):
    n = 200000
    recs = gen_records(n)
    rng = np.random.default_rng(1)
    zp, ze = grid_uniforms(rng, n), grid_uniforms(rng, n)
    g = A.sample_losses(ctx, recs, zp, ze).astype(np.float64)
    o = oracle.sample_batch(recs["mean_loss"], recs["sigma_i"], recs["sigma_c"], recs["max_loss"],
                            zp.astype(np.float64), ze.astype(np.float64))
    mx = recs["max_loss"].astype(np.float64)
    rel = np.abs(g - o) / np.maximum(o, 1e-300)
    assert (np.abs(g - o) <= 1e-4 * o + 1e-7 * mx).all()
    big = o > 1e-3 * mx
    assert np.quantile(rel[big], 0.99) < 5e-6
    assert np.median(rel[big]) < 5e-7
    assert abs(np.mean((g[big] - o[big]) / o[big])) < 2e-7      # no systematic bias
    assert ((g >= 0) & (g <= mx)).all()


def test_sampler_exact_mode_vs_oracle(A, ctx):
    # ARA_EXACT: the per-sample fp64 solve, no tables
    n = 20000
    recs = gen_records(n)
    rng = np.random.default_rng(3)
    zp, ze = grid_uniforms(rng, n), grid_uniforms(rng, n)
    g = A.sample_losses(ctx, recs, zp, ze, exact=True).astype(np.float64)
    t = A.sample_losses(ctx, recs, zp, ze).astype(np.float64)
    o = oracle.sample_batch(recs["mean_loss"], recs["sigma_i"], recs["sigma_c"], recs["max_loss"],
                            zp.astype(np.float64), ze.astype(np.float64))
    mx = recs["max_loss"].astype(np.float64)
    assert (np.abs(g - o) <= 1e-5 * o + 1e-8 * mx).all()
    assert (np.abs(t - g) <= 1e-5 * g + 1e-8 * mx).all()          # table vs exact solve


def _gen_alpha_beta(n):
    # the generator's records -> (alpha, beta) by P:229-236 in numpy (uncapped range)
    recs = gen_records(n)
    mu, mx = recs["mean_loss"].astype(np.float64), recs["max_loss"].astype(np.float64)
    sig = recs["sigma_i"].astype(np.float64) + recs["sigma_c"].astype(np.float64)
    mb, sb = mu / mx, sig / mx
    k = mb * (1 - mb) / sb ** 2 - 1
    return mb * k, (1 - mb) * k


def test_fp64_solver_vs_scipy(A, ctx):
    # row a6's device fp64 solve (it builds every quantile table and serves
    # ARA_EXACT) pinned directly to scipy's betaincinv -- not to the oracle --
    # over the generator's (alpha, beta) range and v in [-7.5, 7.5]; both x
    # and 1 - x to full relative precision
    import scipy.special as sp
    a, b = _gen_alpha_beta(6000)
    rng = np.random.default_rng(11)
    v = np.concatenate([rng.uniform(-7.5, 7.5, a.size - 8), [-7.5, -5, -1e-3, 0.0, 1e-3, 3, 5, 7.5]])
    x, y = A.beta_quantiles(ctx, a, b, v)
    lo = v <= 0
    xr = sp.betaincinv(a[lo], b[lo], sp.ndtr(v[lo]))
    yr = sp.betaincinv(b[~lo], a[~lo], sp.ndtr(-v[~lo]))
    np.testing.assert_allclose(x[lo], xr, rtol=1e-10, atol=0)
    np.testing.assert_allclose(y[~lo], yr, rtol=1e-10, atol=0)
    np.testing.assert_allclose(x + y, 1.0, rtol=0, atol=4e-16)
    # closed forms: Beta(a,1) -> p^(1/a); Beta(1,b) -> 1-(1-p)^(1/b); Beta(1/2,1/2) -> sin^2(pi p/2)
    vv = np.linspace(-6, 6, 41)
    p, q = sp.ndtr(vv), sp.ndtr(-vv)
    for aa in (0.3, 2.5, 40.0):
        x1, y1 = A.beta_quantiles(ctx, np.full(vv.size, aa), 1.0, vv)
        np.testing.assert_allclose(x1[vv <= 0], p[vv <= 0] ** (1 / aa), rtol=1e-11)
        np.testing.assert_allclose(y1[vv > 0], -np.expm1(np.log1p(-q[vv > 0]) / aa), rtol=1e-10)
    x2, _ = A.beta_quantiles(ctx, np.full(vv.size, 0.5), 0.5, vv)
    np.testing.assert_allclose(x2[vv <= 0], np.sin(np.pi * p[vv <= 0] / 2) ** 2, rtol=1e-11)


def test_fp64_solver_cap_regime_vs_mpmath(A, ctx):
    # the sigma_beta-capped regime (G9): alpha, beta in [1e-6, 1e-3],
    # a near-Bernoulli law; x and 1 - x against an mpmath bisection on I_x
    import scipy.special as sp
    from mp_pins import mp_lower_quantile
    cases = [(a_, b_, v_) for a_, b_ in [(1e-3, 1e-3), (5e-4, 1e-3), (2e-6, 1e-6), (1e-3, 3e-6)]
             for v_ in (-3.0, -0.5, -0.01, 0.02, 0.4, 2.5)]
    a, b, v = (np.array(c, np.float64) for c in zip(*cases))
    x, y = A.beta_quantiles(ctx, a, b, v)
    for t in range(len(cases)):
        if v[t] <= 0:
            ref = mp_lower_quantile(float(sp.ndtr(v[t])), a[t], b[t])
            assert x[t] == pytest.approx(ref, rel=1e-9, abs=1e-305), (cases[t], x[t], ref)
        else:
            ref = mp_lower_quantile(float(sp.ndtr(-v[t])), b[t], a[t])
            assert y[t] == pytest.approx(ref, rel=1e-9, abs=1e-305), (cases[t], y[t], ref)


def test_capped_records_fall_back_to_exact(A, ctx):
    # records at the sigma_beta cap (G9: alpha, beta ~ 1e-6) are near-Bernoulli;
    # their table fails the midpoint check and the scan uses the fp64 solve
    cfg = aragen.load_config("cfg1")
    cfg.update(n_trials=300, catalog=500, records_per_elt=200)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    pf["rec_sigma_i"] = pf["rec_sigma_i"].copy()
    pf["rec_sigma_i"][::7] = pf["rec_max"][::7]                   # sigma >= sigma_max -> capped
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 21)
    assert np.array_equal(cnt, ref["count"])
    ylt_check(g, ref)
    r = np.zeros(3, A.RECORD_DTYPE)
    r["max_loss"] = 100.0; r["mean_loss"] = [30, 50, 80]; r["sigma_i"] = [80, 60, 50]
    zz = np.linspace(0.01, 0.99, 99).astype(np.float32)
    for j in range(3):
        rr = np.repeat(r[j:j + 1], len(zz))
        g = A.sample_losses(ctx, rr, zz, zz).astype(np.float64)
        o = oracle.sample_batch(rr["mean_loss"], rr["sigma_i"], rr["sigma_c"], rr["max_loss"],
                                zz.astype(np.float64), zz.astype(np.float64))
        assert np.isfinite(g).all()
        # away from the Bernoulli step at z = 1 - mu_beta, where fp32 vs fp64 v decides
        far = np.abs(zz - (1 - r["mean_loss"][j] / 100.0)) > 1e-3
        assert (np.abs(g - o) <= 1e-4 * o + 1e-6 * 100)[far].all(), (j, g, o)


def test_scan_exact_mode(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 200
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    g = A.run(ctx, P, Y, seed=cfg["seed"], exact=True).cpu().numpy()
    ref = oracle.run(pf, yet, seed=cfg["seed"])
    ylt_check(g, ref)


def test_sampler_extreme_v_and_edges(A, ctx):
    recs = gen_records(4000)
    rng = np.random.default_rng(2)
    n = len(recs)
    # deepest tails of the uniform grid: v up to |7.5|
    zp = np.where(rng.uniform(size=n) < 0.5, 2.0 ** -24, 1 - 2.0 ** -24).astype(np.float32)
    ze = zp.copy()
    g = A.sample_losses(ctx, recs, zp, ze).astype(np.float64)
    o = oracle.sample_batch(recs["mean_loss"], recs["sigma_i"], recs["sigma_c"], recs["max_loss"],
                            zp.astype(np.float64), ze.astype(np.float64))
    mx = recs["max_loss"].astype(np.float64)
    assert np.isfinite(g).all()
    assert (np.abs(g - o) <= 1e-4 * o + 1e-7 * mx).all()
    # degenerate records (G10) and sigma_I = 0 / sigma_C = 0 extremes
    from paper_1310_2274_b200 import ara
    r = np.zeros(6, ara.RECORD_DTYPE)
    r["max_loss"] = 100.0
    r["mean_loss"] = [30, 0, 100, 25, 25, 50]
    r["sigma_i"] = [0, 5, 5, 10, 0, 60]
    r["sigma_c"] = [0, 5, 5, 0, 10, 0]
    zp = np.array([0.3, 0.3, 0.3, 0.9, 0.9, 0.7], np.float32)
    ze = np.array([0.6, 0.6, 0.6, 0.2, 0.2, 0.1], np.float32)
    g = A.sample_losses(ctx, r, zp, ze).astype(np.float64)
    assert g[0] == 30 and g[1] == 0 and g[2] == 100
    for t in (3, 4, 5):     # sigma_C = 0 uses z_P only, sigma_I = 0 z_E only, capped
        o = oracle.sample_loss(r["mean_loss"][t], r["sigma_i"][t], r["sigma_c"][t], 100.0,
                               float(zp[t]), float(ze[t]))
        assert abs(g[t] - o) <= 1e-4 * o + 1e-5, (t, g[t], o)


# ---- the whole path on cfg1 (rows a1-a11) ------------------------------------
def test_cfg1_full(A, ctx):
    cfg = aragen.load_config("cfg1")
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, cfg["seed"])
    assert np.array_equal(cnt, ref["count"])
    assert np.array_equal(hsh, ref["hash"])
    ylt_check(g, ref)
    lim = pf["layer_terms"][0][3]
    assert (g >= 0).all() and (g <= lim).all()
    assert (g == np.float32(lim)).sum() == (ref["ylt"] == lim).sum()     # limit binds identically


def test_primary_integer_bit_exact(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg.update(sigma_scale=0.0, integer_mu=True, n_trials=600, catalog=3000, records_per_elt=900,
               layer_terms=[[2e5, 5e6, 2.0e7, 3.0e7]])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    for su in (False, True):
        (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 5, su=su)
        assert np.array_equal(cnt, ref["count"])
        assert np.array_equal(g, ref["ylt"].astype(np.float32))


def test_primary_fast_path_integer_bit_exact(A, ctx):
    # no draw is taken (SU off, or every sigma = 0 with SU on): the streaming
    # pass over the per-(event, layer) occurrence losses of ara_create_portfolio
    # (no debug lookup -> the fast path); integer means and terms: bit-exact
    cfg = aragen.load_config("cfg1")
    cfg.update(sigma_scale=0.0, integer_mu=True, n_trials=600, catalog=3000, records_per_elt=900,
               layer_terms=[[2e5, 5e6, 2.0e7, 3.0e7]])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ref = oracle.run(pf, yet, seed=5, su=False)
    for su in (False, True):
        g = A.run(ctx, P, Y, seed=5, su=su).cpu().numpy()
        assert np.array_equal(g, ref["ylt"].astype(np.float32))
        ylt, occ = A.run_ep(ctx, P, Y, seed=5, su=su)
        assert np.array_equal(ylt.cpu().numpy(), g)
        assert np.array_equal(occ.cpu().numpy(), ref["occ_max"].astype(np.float32))


@pytest.mark.parametrize("n_layers,J,ragged,terms", [(1, 16, False, False), (3, 4, True, True), (8, 3, False, True),
                                                     (2, 5, True, False)])
def test_primary_fast_path_vs_oracle(A, ctx, n_layers, J, ragged, terms, monkeypatch):
    # the fast path (1, 2 -> 2, 3 -> 4 and 8 layers per event sector; CSR
    # trials; XELT terms) against the oracle with SU off, and against the
    # two-kernel path of the same run (ARA_NO_PRIMARY_PATH, a test aid)
    cfg = aragen.load_config("cfg1")
    cfg.update(n_layers=n_layers, elts_per_layer=J, catalog=4000, records_per_elt=700, n_trials=500,
               layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(n_layers)])
    if ragged:
        cfg.update(k_min=0, k_max=170)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    if terms:
        rng = np.random.default_rng(n_layers)
        n_elts = n_layers * J
        pf["elt_terms"] = np.stack([rng.uniform(0, 2e4, n_elts), rng.uniform(1e5, 1e7, n_elts),
                                    rng.uniform(0.2, 1.0, n_elts)], 1)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ref = oracle.run(pf, yet, seed=3, su=False)
    ylt, occ = A.run_ep(ctx, P, Y, seed=3, su=False)
    g, m = ylt.cpu().numpy(), occ.cpu().numpy()
    for li in range(n_layers):
        ylt_check(g[li], ref, li)
        o = ref["occ_max"][li]
        assert (np.abs(m[li] - o) <= 1e-6 * o).all()
    monkeypatch.setenv("ARA_NO_PRIMARY_PATH", "1")
    g2 = A.run(ctx, P, Y, seed=3, su=False).cpu().numpy()
    assert (np.abs(g2.astype(np.float64) - g) <= 1e-5 * np.abs(g) + 1e-6 * ref["gross"]).all()


def test_ragged_empty_trials_and_repeats(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg.update(k_min=0, k_max=150, n_trials=700, catalog=300, records_per_elt=120)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg, first_trial=1000, n_trials=700)
    lens = np.diff(yet["trial_off"].astype(np.int64))
    assert (lens == 0).any() and lens.max() > 64
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 9)
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    ylt_check(g, ref)


@pytest.mark.parametrize("n_layers,J", [(8, 16), (3, 14), (1, 1), (2, 33)])
def test_multi_layer_and_wide_masks(A, ctx, n_layers, J):
    cfg = aragen.load_config("cfg1")
    terms = [[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(n_layers)]
    cfg.update(n_layers=n_layers, elts_per_layer=J, catalog=4000, records_per_elt=600,
               n_trials=300, layer_terms=terms)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    pf["layer_prog"] = (np.arange(n_layers) % 3).astype(np.uint32)    # several programs (G26)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 77)
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    for li in range(n_layers):
        ylt_check(g[li], ref, li)


@pytest.mark.parametrize("n_layers,J", [(8, 16), (1, 224)])
def test_heavy_overlap_many_pairs_per_lane(A, ctx, n_layers, J):
    # every XELT holds half the catalogue: a lane's 4 events carry up to
    # 4 x 224 = 896 pairs (> 127: every bit slice of the compaction's ballot
    # prefix sum is exercised); counts, hashes and YLT against the oracle
    cfg = aragen.load_config("cfg1")
    terms = [[2e5 * (l + 1), 5e6, 1.0e6, 5.0e9] for l in range(n_layers)]
    cfg.update(n_layers=n_layers, elts_per_layer=J, catalog=1000, records_per_elt=500,
               n_trials=60, events_per_trial=64, layer_terms=terms)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 17)
    assert cnt.sum(0).max() > 64 * 0.5 * n_layers * J * 0.8        # ~half of all slots present
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    for li in range(n_layers):
        ylt_check(g[li], ref, li)


@pytest.mark.parametrize("n_layers,J,K", [(1, 2, 3000), (3, 4, 1500)])
def test_long_trials_span_several_segments(A, ctx, n_layers, J, K):
    # more present pairs per trial than one sampler segment holds (768 for one
    # layer, fewer with more layers): occurrence runs and trial sums carry
    # across segments; every trial still matches the oracle
    cfg = aragen.load_config("cfg1")
    terms = [[2e5 * (l + 1), 5e6, 1.0e6, 5.0e9] for l in range(n_layers)]
    cfg.update(n_layers=n_layers, elts_per_layer=J, catalog=5000, records_per_elt=2000,
               n_trials=40, events_per_trial=K, layer_terms=terms)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 91)
    assert cnt.sum(0).min() > 800                      # several segments per trial
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    for li in range(n_layers):
        ylt_check(g[li], ref, li)


def test_shared_elts_and_xelt_terms(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg.update(n_layers=1, elts_per_layer=4, catalog=2000, records_per_elt=500, n_trials=400,
               layer_terms=[[1e5, 5e6, 0.0, np.inf]])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    # two layers over overlapping XELTs, same program -> identical draws
    pf["layer_prog"] = np.zeros(2, np.uint32)
    pf["layer_elt_off"] = np.array([0, 3, 6], np.uint64)
    pf["layer_elts"] = np.array([0, 1, 2, 1, 2, 3], np.uint32)
    pf["layer_terms"] = np.array([[1e5, 5e6, 0.0, np.inf], [0.0, np.inf, 1e6, 4e7]])
    pf["elt_terms"] = np.array([[1e4, 2e6, 0.5], [0.0, np.inf, 1.0], [5e3, 1e7, 0.8], [0, 3e6, 0.25]])
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, 3)
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    for li in range(2):
        ylt_check(g[li], ref, li)


def _heavy_trial_yet(cfg, pf):
    # trials 0-9 as generated, trial 10 = 400 events present in 2 XELTs each
    # (800 pairs, > 2x the expected pairs of its region), trials 11-50 as generated
    yet = aragen.build_yet(cfg)
    R = cfg["records_per_elt"]
    both = np.intersect1d(pf["rec_event"][:R], pf["rec_event"][R:2 * R])
    assert both.size > 50
    heavy = np.random.default_rng(4).choice(both, 400).astype(np.uint32)
    K = cfg["events_per_trial"]
    ev = np.concatenate([yet["events"][:10 * K], heavy, yet["events"][10 * K:]])
    off = np.concatenate([np.arange(11, dtype=np.uint64) * K, 10 * K + 400 + np.arange(0, 41, dtype=np.uint64) * K])
    return {"trial_off": off, "events": ev, "first_trial": 0}


def test_pair_region_overflow_pass(A, ctx):
    # a trial whose present pairs exceed its region (2x expected + 128) is
    # compacted again into an exactly sized region of the overflow pool and
    # sampled by the same kernel; counts/hashes/YLT exact
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 50
    pf = aragen.build_portfolio(cfg)
    y2 = _heavy_trial_yet(cfg, pf)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, y2, cfg["seed"])
    assert cnt[0, 10] == 800
    assert A.last_run_timings(ctx)["redo_ms"] > 0          # the overflow pass ran
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    ylt_check(g, ref)


@pytest.mark.parametrize("cap", ["0", "1", "64"])
def test_overflow_pass_bit_identical(A, ctx, cap, monkeypatch):
    # whether a trial overflows its region depends on the region size (and so
    # on the loaded YET's mean length); the YLT must not: every trial forced
    # through the overflow pass (ARA_PAIR_CAP, a test aid), a CSR YET with one
    # heavy trial run whole and as two shards -- all bit-identical
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 50
    pf = aragen.build_portfolio(cfg)
    y2 = _heavy_trial_yet(cfg, pf)
    P = A.Portfolio(ctx, pf)
    full = A.run(ctx, P, A.Yet.from_dict(ctx, y2), seed=7, debug=True)
    off = y2["trial_off"].astype(np.int64)
    parts = []
    for lo, hi in ((0, 12), (12, 51)):
        ys = {"trial_off": (off[lo:hi + 1] - off[lo]).astype(np.uint64),
              "events": y2["events"][off[lo]:off[hi]], "first_trial": lo}
        parts.append(A.run(ctx, P, A.Yet.from_dict(ctx, ys), seed=7).cpu().numpy())
    assert np.array_equal(np.concatenate(parts, axis=1), full[0].cpu().numpy())
    monkeypatch.setenv("ARA_PAIR_CAP", cap)
    forced = A.run(ctx, P, A.Yet.from_dict(ctx, y2), seed=7, debug=True)
    for x, y in zip(full, forced):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_determinism_and_sharding(A, ctx):
    cfg = aragen.load_config("cfg1")
    pf = aragen.build_portfolio(cfg)
    full = aragen.build_yet(cfg)
    P = A.Portfolio(ctx, pf)
    Y = A.Yet.from_dict(ctx, full)
    a = A.run(ctx, P, Y, seed=11).cpu().numpy()
    b = A.run(ctx, P, Y, seed=11).cpu().numpy()
    assert np.array_equal(a, b)
    parts = []
    for r in range(4):        # trial-sharded "ranks": global keying -> identical YLT
        n = cfg["n_trials"] // 4
        y = aragen.build_yet(cfg, first_trial=r * n, n_trials=n)
        parts.append(A.run(ctx, P, A.Yet.from_dict(ctx, y), seed=11).cpu().numpy())
    assert np.array_equal(np.concatenate(parts, axis=1), a)


@pytest.mark.parametrize("K", [1000, 1002, 64])
def test_fixed_length_equals_csr_form(A, ctx, K):
    # the same trials as a fixed-length YET (compaction: the VEC specialisation
    # with 4-byte index entries; primary path: round-robin trials) and as CSR
    # offsets (per-id loads, 8-byte entries, dynamic scheduler): the YLT is a
    # function of the YET's contents alone -- bit-identical YLT, counts, hashes,
    # with and without draws (K = 1002: not a multiple of 4, no VEC either side)
    cfg = aragen.load_config("cfg3")
    cfg.update(n_trials=6000, events_per_trial=K, layer_terms=[[2e5, 5e6, 1.0e6, 5.0e9]])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P = A.Portfolio(ctx, pf)
    fixed = A.Yet.from_dict(ctx, yet)
    off = np.arange(cfg["n_trials"] + 1, dtype=np.uint64) * np.uint64(K)
    csr = A.Yet(ctx, yet["events"], trial_off=off)
    for su in (True, False):
        for dbg in (True, False):
            a = A.run(ctx, P, fixed, seed=13, su=su, debug=dbg)
            b = A.run(ctx, P, csr, seed=13, su=su, debug=dbg)
            for x, y in zip(a if dbg else [a], b if dbg else [b]):
                assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


_IX_SCRIPT = r"""
import sys, hashlib, numpy as np
sys.path.insert(0, {root!r})
import aragen
from paper_1310_2274_b200 import ara
ctx = ara.Context(0)
cfg = aragen.load_config("cfg3")
cfg.update(n_trials=20000, layer_terms=[[2e5, 5e6, 1.0e6, 5.0e9]])
pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
P, Y = ara.Portfolio(ctx, pf), ara.Yet.from_dict(ctx, yet)
h = hashlib.sha256()
for x in ara.run(ctx, P, Y, seed=3, debug=True):
    h.update(x.cpu().numpy().tobytes())
print(h.hexdigest())
"""


def test_compaction_index_entry_widths_identical():
    # the compaction's packed 4-byte index entries (first | count << 24) and the
    # 8-byte (first, count) pairs it falls back to (>= 2^24 device records; forced
    # here by ARA_COMPACT_IX4=0, read once per process): bit-identical YLT, counts, hashes
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", _IX_SCRIPT.format(root=root)], env=dict(os.environ, ARA_COMPACT_IX4=v),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip())
    assert outs[0] == outs[1]


@pytest.mark.parametrize("n_layers,J,K", [(1, 16, 1000), (3, 4, 1500)])
def test_packed_wide_pairs_and_batching_identical(A, ctx, n_layers, J, K, monkeypatch):
    # 4-byte packed and 8-byte pair records, any trial batching
    # (ARA_BATCH_TRIALS) and the two-stream schedule (ARA_OVERLAP): each
    # trial in the same order, bit-identical YLT, counts and hashes
    cfg = aragen.load_config("cfg3")
    terms = [[2e5 * (l + 1), 5e6, 1.0e6, 5.0e9] for l in range(n_layers)]
    cfg.update(n_layers=n_layers, elts_per_layer=J, n_trials=20000, events_per_trial=K, layer_terms=terms)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P = A.Portfolio(ctx, pf)
    Y = A.Yet.from_dict(ctx, yet)
    for su in (True, False):
        ref = A.run(ctx, P, Y, seed=5, su=su, debug=True)                 # 4-byte packed pairs
        outs = [A.run(ctx, P, Y, seed=5, su=su, debug=True, wide_pairs=True)]  # 8-byte pairs
        for env in ({"ARA_BATCH_TRIALS": "777"}, {"ARA_BATCH_TRIALS": "20000"}, {"ARA_OVERLAP": "1"},
                    {"ARA_OVERLAP": "1", "ARA_BATCH_TRIALS": "3000"}):
            with monkeypatch.context() as m:
                for k_, v_ in env.items():
                    m.setenv(k_, v_)
                outs.append(A.run(ctx, P, Y, seed=5, su=su, debug=True))
        for o in outs:
            for x, y in zip(ref, o):
                assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_event_out_of_range(A, ctx):
    cfg = aragen.load_config("cfg1")
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg, n_trials=10)
    yet["events"][17] = cfg["catalog"]
    P = A.Portfolio(ctx, pf)
    Y = A.Yet.from_dict(ctx, yet)
    with pytest.raises(A.AraError) as ei:
        A.run(ctx, P, Y, seed=1)
    assert ei.value.code == A.ERANGE


# ---- row a12: PML / TVaR -------------------------------------------------------
@pytest.mark.parametrize("n", [1, 7, 1000, 100003, 800000, 3000001])
def test_measures_vs_oracle_sort(A, ctx, n):
    import torch
    rng = np.random.default_rng(n)
    x = rng.lognormal(15, 1.2, n).astype(np.float32)
    x[rng.uniform(size=n) < 0.1] = 0.0                       # retention clip mass
    x[rng.uniform(size=n) < 0.002] = np.float32(3.0e8)       # limit clip ties
    rps = [2, 10, 100, 250, 500] if n >= 1000 else [1.5, 2, 4]
    d = torch.from_numpy(x).cuda()
    pml, tvar = A.risk_measures(ctx, d, 1, n, 0, rps=rps)
    pml2, tvar2, var = A.risk_measures_var(ctx, d, 1, n, 0, rps=rps)
    assert np.array_equal(pml, pml2) and np.array_equal(tvar, tvar2)
    for q, rp in enumerate(rps):
        if OM.tvar_rp(x, rp) is None:
            continue
        assert pml[q] == pytest.approx(OM.pml(x.astype(np.float64), rp), rel=1e-12, abs=1e-9)
        vo, to = OM.tvar_rp(x.astype(np.float64), rp)
        assert tvar[q] == pytest.approx(to, rel=1e-10)
        assert var[q] == vo                     # an order statistic: exact


def _adversarial_table(kind, n, rng):
    """Tables whose keys stress the joint select's digit boundaries (12-, 10-, 10-bit
    digits of the order-preserving key): ties, keys that differ only in the low
    digit or only across a digit boundary, negative values, subnormals."""
    if kind == "all_equal":
        return np.full(n, 123456.75, dtype=np.float32)
    if kind == "low_bits":            # one high prefix, the last 10 bits random
        base = np.float32(7.5e6).view(np.uint32) & ~np.uint32(0x3ff)
        return (base | rng.integers(0, 1024, n, dtype=np.uint32)).view(np.float32)
    if kind == "digit_edges":         # keys at +-1 ulp around 2^10 / 2^20 key boundaries
        base = np.float32(3.0e7).view(np.uint32) & ~np.uint32(0xfffff)
        off = rng.choice(np.array([0, 1, 0x3ff, 0x400, 0x401, 0xfffff, 0x100000, 0x100001], np.uint32), n)
        return (base - np.uint32(0x100000) + off).view(np.float32)
    if kind == "signed":              # negative and positive values, zeros of both signs
        x = (rng.standard_normal(n) * 1e5).astype(np.float32)
        x[rng.uniform(size=n) < 0.05] = np.float32(-0.0)
        x[rng.uniform(size=n) < 0.05] = np.float32(0.0)
        return x
    if kind == "subnormal":           # mostly zero, a tail of subnormal and tiny normal values
        x = np.zeros(n, dtype=np.float32)
        m = rng.uniform(size=n) < 0.3
        x[m] = rng.integers(1, 1 << 23, int(m.sum()), dtype=np.uint32).view(np.float32)
        x[rng.uniform(size=n) < 0.01] = np.float32(2.0e-30)
        return x
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["all_equal", "low_bits", "digit_edges", "signed", "subnormal"])
@pytest.mark.parametrize("n", [1000, 100003, 800000])
def test_measures_adversarial_keys(A, ctx, kind, n):
    # the joint select (<= 4 return periods) and the tail-sort path (> 4) against
    # the oracle's sort: VaR exact, PML to rounding, TVaR to the fixed-point sum
    import torch
    rng = np.random.default_rng([n, len(kind), ord(kind[0])])
    x = _adversarial_table(kind, n, rng)
    d = torch.from_numpy(x).cuda()
    for rps in ([100, 250, 500], [2, 10, 100, 250, 500]):
        pml, tvar, var = A.risk_measures_var(ctx, d, 1, n, 0, rps=rps)
        x64 = x.astype(np.float64)
        for q, rp in enumerate(rps):
            vo, to = OM.tvar_rp(x64, rp)
            assert var[q] == vo, (kind, n, rp)
            assert pml[q] == pytest.approx(OM.pml(x64, rp), rel=1e-12, abs=0.0)
            assert tvar[q] == pytest.approx(to, rel=1e-9, abs=0.0)


@pytest.mark.parametrize("rp_min", [533, 266, 133, 66, 33])
def test_measures_every_sort_size(A, ctx, rp_min):
    # the deepest rank decides the sort size (1024 E values, E = 2 .. 32 in
    # registers per thread): each size once, against the oracle's sort
    import torch
    n = 800000
    rng = np.random.default_rng(rp_min)
    x = rng.lognormal(15, 1.2, n).astype(np.float32)
    x[rng.uniform(size=n) < 0.1] = 0.0
    x[rng.uniform(size=n) < 0.002] = np.float32(3.0e8)
    rps = [rp_min, 2 * rp_min + 1, 1000]
    d = torch.from_numpy(x).cuda()
    pml, tvar = A.risk_measures(ctx, d, 1, n, 0, rps=rps)
    for q, rp in enumerate(rps):
        assert pml[q] == pytest.approx(OM.pml(x.astype(np.float64), rp), rel=1e-12, abs=1e-9)
        assert tvar[q] == pytest.approx(OM.tvar_rp(x.astype(np.float64), rp)[1], rel=1e-10)


@pytest.mark.parametrize("rps", [[2, 3, 10, 100, 250, 500], [33, 66, 133, 266, 533]])
def test_measures_many_return_periods(A, ctx, rps):
    # more than 4 return periods: the tail-sort path (k <= 32768) or the deep
    # per-rank selects (RP 2 at 800k trials); 1-4: the joint select -- all equal
    import torch
    n = 800000
    rng = np.random.default_rng(len(rps))
    x = rng.lognormal(15, 1.2, n).astype(np.float32)
    x[rng.uniform(size=n) < 0.1] = 0.0
    x[rng.uniform(size=n) < 0.002] = np.float32(3.0e8)
    d = torch.from_numpy(x).cuda()
    pml, tvar, var = A.risk_measures_var(ctx, d, 1, n, 0, rps=rps)
    for q, rp in enumerate(rps):
        assert pml[q] == pytest.approx(OM.pml(x.astype(np.float64), rp), rel=1e-12, abs=1e-9)
        vo, to = OM.tvar_rp(x.astype(np.float64), rp)
        assert tvar[q] == pytest.approx(to, rel=1e-10) and var[q] == vo
        p1, t1, v1 = A.risk_measures_var(ctx, d, 1, n, 0, rps=[rp])       # joint select
        assert p1[0] == pml[q] and v1[0] == var[q] and t1[0] == pytest.approx(tvar[q], rel=1e-12)


def test_measures_rollup_and_shards(A, ctx):
    import torch
    rng = np.random.default_rng(5)
    L, n, P = 3, 40000, 4
    y = rng.lognormal(12, 1, (P, L, n // P)).astype(np.float32)
    d = torch.from_numpy(y).cuda()
    flat = y.transpose(1, 0, 2).reshape(L, n)            # [L][n] in shard order
    for layer in (-1, 0, 2):
        v = flat.sum(axis=0, dtype=np.float32) if layer < 0 else flat[layer]
        if layer < 0:
            v = (flat[0] + flat[1]) + flat[2]            # fp32, ascending layer order
        pml, tvar = A.risk_measures(ctx, d, L, n, layer, rps=(100, 250), n_shards=P)
        for q, rp in enumerate((100, 250)):
            assert pml[q] == pytest.approx(OM.pml(v.astype(np.float64), rp), rel=1e-12)
            assert tvar[q] == pytest.approx(OM.tvar_rp(v.astype(np.float64), rp)[1], rel=1e-10)


def test_measures_errors(A, ctx):
    import torch
    d = torch.zeros(10, device="cuda")
    with pytest.raises(A.AraError):
        A.risk_measures(ctx, d, 1, 10, 0, rps=(1.0,))
    with pytest.raises(A.AraError):
        A.risk_measures(ctx, d, 1, 0, 0, rps=(10,))
    pml, tvar = A.risk_measures(ctx, d, 1, 10, 0, rps=(10,))
    assert pml[0] == 0 and tvar[0] == 0


# ---- full-size configurations: every trial against the oracle ----------------
def _measures_pure_rel(A, ctx, ylt_dev, ref_ylt, L, N, layers, rps, shards=1):
    """PML / TVaR of each side from its own YLT: pure 1e-4 relative."""
    for layer in layers:
        pml, tvar = A.risk_measures(ctx, ylt_dev, L, N, layer, rps=rps, n_shards=shards)
        o = OM.rollup(ref_ylt) if layer < 0 else ref_ylt[layer]
        for q, rp in enumerate(rps):
            po, to = OM.pml(o, rp), OM.tvar_rp(o, rp)[1]
            assert abs(pml[q] - po) <= REL * abs(po), (layer, rp, pml[q], po)
            assert abs(tvar[q] - to) <= REL * abs(to), (layer, rp, tvar[q], to)


def _pure_fraction(g, o):
    nz = o > 0
    return float((np.abs(g[nz] - o[nz]) <= REL * o[nz]).mean()) if nz.any() else 1.0


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_size_every_trial(A, ctx, name):
    # BASELINE's own sizes: cfg3 = the paper's headline run (800k trials x
    # 1,000 events x 16 XELTs, SU on) and cfg2 (100k x 1,000, 2M catalogue,
    # sigma = 0): the GPU YLT of EVERY trial against the fp64 oracle run over
    # all trials (the north star's acceptance), lookup counts bit-exact, and
    # PML / TVaR at 1-in-100/250/500 at pure 1e-4 relative
    import torch
    cfg = aragen.load_config(name)
    pf = aragen.build_portfolio(cfg)
    N, K = cfg["n_trials"], cfg["events_per_trial"]
    ev = torch.empty(N * K, dtype=torch.int32).pin_memory()
    yet = aragen.build_yet(cfg, out=ev.numpy().view(np.uint32))
    P = A.Portfolio(ctx, pf)
    Y = A.Yet(ctx, ev, fixed_len=K, n_trials=N)
    ylt_d, cnt, _ = A.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], debug=True)
    ylt = ylt_d.cpu().numpy()
    ref = oracle.run(pf, yet, seed=cfg["seed"], su=cfg["su"])
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), ref["count"])
    ylt_check(ylt, ref)
    assert _pure_fraction(ylt[0].astype(np.float64), ref["ylt"][0]) > 0.999
    lim = pf["layer_terms"][0][3]
    assert (ylt >= 0).all() and (ylt <= lim).all()
    _measures_pure_rel(A, ctx, ylt_d, ref["ylt"], 1, N, [0], cfg["return_periods"])


def test_cfg5_rank_shard_every_trial(A, ctx):
    # cfg5 as rank 7 of 8 holds it: global trials [875000, 1000000) of the
    # 1M-trial, 8-layer x 16-XELT, 2M-event analysis at full portfolio size;
    # every layer of every trial of the shard against the oracle (global
    # trial indices), then the shard's per-layer and roll-up measures at pure
    # 1e-4 relative
    import torch
    cfg = aragen.load_config("cfg5")
    pf = aragen.build_portfolio(cfg)
    N, K, L = cfg["n_trials"], cfg["events_per_trial"], cfg["n_layers"]
    lo, n = 7 * N // 8, N // 8
    ev = torch.empty(n * K, dtype=torch.int32).pin_memory()
    yet = aragen.build_yet(cfg, first_trial=lo, n_trials=n, out=ev.numpy().view(np.uint32))
    P = A.Portfolio(ctx, pf)
    Y = A.Yet(ctx, ev, fixed_len=K, first_trial=lo, n_trials=n)
    ylt_d = A.run(ctx, P, Y, seed=cfg["seed"], su=True)
    ylt = ylt_d.cpu().numpy()
    assert ylt.shape == (L, n)
    ref = oracle.run(pf, yet, seed=cfg["seed"], su=True,
                     trial_index=np.arange(lo, lo + n, dtype=np.uint64))
    for li in range(L):
        ylt_check(ylt[li], ref, li)
    _measures_pure_rel(A, ctx, ylt_d, ref["ylt"], L, n, [0, L - 1, -1], cfg["return_periods"])


@pytest.mark.parametrize("name,n", [("cfg1", None), ("cfg3", 20000), ("cfg5", 4000)])
def test_measures_end_to_end(A, ctx, name, n):
    cfg = aragen.load_config(name)
    if n is not None:
        cfg["n_trials"] = n
    if name == "cfg5":
        cfg.update(catalog=200000, records_per_elt=2000)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ylt = A.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"])
    ref = oracle.run(pf, yet, seed=cfg["seed"], su=cfg["su"])
    ylt_check(ylt.cpu().numpy(), ref)
    rps = [10, 50, 100] if cfg["n_trials"] < 20000 else cfg["return_periods"]
    L = cfg["n_layers"]
    for layer in ([0] if L == 1 else [0, L - 1, -1]):
        pml, tvar = A.risk_measures(ctx, ylt, L, cfg["n_trials"], layer, rps=rps)
        o = OM.rollup(ref["ylt"]) if layer < 0 else ref["ylt"][layer]
        S = ref["gross"].sum(axis=0) if layer < 0 else ref["gross"][layer]
        floor = FLOOR * S.max()
        for q, rp in enumerate(rps):
            po, to = OM.pml(o, rp), OM.tvar_rp(o, rp)[1]
            assert abs(pml[q] - po) <= REL * abs(po) + floor, (layer, rp, pml[q], po)
            assert abs(tvar[q] - to) <= REL * abs(to) + floor, (layer, rp, tvar[q], to)


# ---- OEP basis (NEXT-3, reading G29): largest occurrence loss per (layer, trial)
def occ_check(m, ref, pf, li):
    # per-sample relative error <= 1e-5 (G12) on l = g + OccR gives the floor
    o = ref["occ_max"][li]
    occr = float(pf["layer_terms"][li][0])
    m = np.asarray(m, np.float64)
    tol = REL * o + 1e-5 * occr + 1e-3
    bad = np.abs(m - o) > tol
    assert not bad.any(), f"{bad.sum()} occ_max entries out of tolerance (layer {li})"
    assert (m >= 0).all() and (m <= float(pf["layer_terms"][li][1])).all()


def _oep_case(name):
    cfg = aragen.load_config("cfg1")
    if name == "cfg1":
        pass
    elif name == "layers8":
        cfg.update(n_layers=8, elts_per_layer=16, catalog=4000, records_per_elt=600, n_trials=300,
                   layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(8)])
    elif name == "layers3_long":
        cfg.update(n_layers=3, elts_per_layer=4, catalog=5000, records_per_elt=2000, n_trials=40,
                   events_per_trial=1500, layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e9] for l in range(3)])
    elif name == "long1":
        cfg.update(n_layers=1, elts_per_layer=2, catalog=5000, records_per_elt=2000, n_trials=40,
                   events_per_trial=3000, layer_terms=[[2e5, 5e6, 1.0e6, 5.0e9]])
    elif name == "ragged":
        cfg.update(k_min=0, k_max=150, n_trials=700, catalog=300, records_per_elt=120)
    return cfg


@pytest.mark.parametrize("name", ["cfg1", "layers8", "layers3_long", "long1", "ragged"])
@pytest.mark.parametrize("exact", [False, True])
def test_occ_max_vs_oracle(A, ctx, name, exact):
    cfg = _oep_case(name)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ylt, occ = A.run_ep(ctx, P, Y, seed=cfg["seed"], exact=exact)
    ref = oracle.run(pf, yet, seed=cfg["seed"])
    g, m = ylt.cpu().numpy(), occ.cpu().numpy()
    for li in range(pf["layer_terms"].shape[0]):
        ylt_check(g[li], ref, li)
        occ_check(m[li], ref, pf, li)
    # the YLT does not depend on whether occ_max is requested
    assert np.array_equal(g, A.run(ctx, P, Y, seed=cfg["seed"], exact=exact).cpu().numpy())


def test_occ_max_redo_trials(A, ctx):
    # a trial redone by the fp64-capable kernel (its pairs overflow the region)
    # gets occ_max from that kernel
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 50
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    R, K = cfg["records_per_elt"], cfg["events_per_trial"]
    both = np.intersect1d(pf["rec_event"][:R], pf["rec_event"][R:2 * R])
    heavy = np.random.default_rng(4).choice(both, 400).astype(np.uint32)
    ev = np.concatenate([yet["events"][:10 * K], heavy, yet["events"][10 * K:]])
    off = np.concatenate([np.arange(11, dtype=np.uint64) * K,
                          10 * K + 400 + np.arange(0, 41, dtype=np.uint64) * K])
    y2 = {"trial_off": off, "events": ev, "first_trial": 0}
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, y2)
    ylt, occ = A.run_ep(ctx, P, Y, seed=cfg["seed"])
    assert A.last_run_timings(ctx)["redo_ms"] > 0
    ref = oracle.run(pf, y2, seed=cfg["seed"])
    ylt_check(ylt.cpu().numpy(), ref)
    occ_check(occ.cpu().numpy()[0], ref, pf, 0)


def test_occ_max_measures_oep(A, ctx):
    # OEP PML / TVaR = the measures of the occ_max table (per layer)
    cfg = aragen.load_config("cfg3")
    cfg["n_trials"] = 20000
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ylt, occ = A.run_ep(ctx, P, Y, seed=cfg["seed"])
    ref = oracle.run(pf, yet, seed=cfg["seed"])
    occ_check(occ.cpu().numpy()[0], ref, pf, 0)
    rps = cfg["return_periods"]
    pml, tvar = A.risk_measures(ctx, occ, 1, cfg["n_trials"], 0, rps=rps)
    o = ref["occ_max"][0]
    floor = 1e-5 * pf["layer_terms"][0][0] + 1e-3
    for q, rp in enumerate(rps):
        po, to = OM.pml(o, rp), OM.tvar_rp(o, rp)[1]
        assert abs(pml[q] - po) <= REL * abs(po) + floor, (rp, pml[q], po)
        assert abs(tvar[q] - to) <= REL * abs(to) + floor, (rp, tvar[q], to)


def test_run_ep_errors(A, ctx):
    import torch
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 10
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    ylt = torch.empty((1, 10), dtype=torch.float32, device="cuda")
    with pytest.raises(A.AraError):
        A._check(A.lib.ara_run_ep(ctx.h, P.h, Y.h, 1, A.SU, A._p(ylt), None, None, None))
    with pytest.raises(A.AraError):                  # host memory for occ_max
        A._check(A.lib.ara_run_ep(ctx.h, P.h, Y.h, 1, A.SU, A._p(ylt), A._p(np.zeros((1, 10), np.float32)),
                                  None, None))


# ---- packed YET upload (storage encoding; ara_yet_refill_packed) -------------
@pytest.mark.parametrize("ragged", [False, True])
def test_packed_refill_matches_plain(A, ctx, ragged):
    cfg = aragen.load_config("cfg1")
    if ragged:
        cfg.update(k_min=0, k_max=150, n_trials=700)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P = A.Portfolio(ctx, pf)
    Y0 = A.Yet.from_dict(ctx, yet)
    ref = A.run(ctx, P, Y0, seed=cfg["seed"], debug=True)
    for bits in (aragen.yet_bits(cfg["catalog"]), 17, 32):
        words = aragen.pack_yet(yet["events"], bits)
        if yet.get("fixed_len"):
            Y = A.Yet(ctx, None, fixed_len=yet["fixed_len"], n_trials=len(yet["trial_off"]) - 1)
        else:
            Y = A.Yet(ctx, None, trial_off=yet["trial_off"])
        Y.refill_packed(words, bits)
        got = A.run(ctx, P, Y, seed=cfg["seed"], debug=True)
        for a, b in zip(got, ref):
            assert np.array_equal(a.cpu().numpy(), b.cpu().numpy()), bits
        # the same words from device memory (unpacked where they are, no staging):
        # an exact-size buffer, so the unpack must not read past its last word
        import torch
        dw = torch.from_numpy(np.ascontiguousarray(words).view(np.int32)).cuda()
        Y.refill(np.zeros(yet["events"].size, np.uint32))
        Y.refill_packed(dw, bits)
        got = A.run(ctx, P, Y, seed=cfg["seed"], debug=True)
        for a, b in zip(got, ref):
            assert np.array_equal(a.cpu().numpy(), b.cpu().numpy()), ("device words", bits)


def test_packed_refill_errors(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 20
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P = A.Portfolio(ctx, pf)
    Y = A.Yet(ctx, None, fixed_len=yet["fixed_len"], n_trials=20)
    w = aragen.pack_yet(yet["events"], 20)
    for bad in (0, 33):
        with pytest.raises(A.AraError):
            Y.refill_packed(w, bad)
    ev = yet["events"].copy()
    ev[17] = cfg["catalog"] + 5                     # out of the catalogue, fits in 20 bits
    Y.refill_packed(aragen.pack_yet(ev, 20), 20)
    with pytest.raises(A.AraError) as ei:
        A.run(ctx, P, Y, seed=1)
    assert ei.value.code == 2                       # ARA_ERANGE


# ---- paper-literal RNG alternatives of reading G2 (NEXT-4) -------------------
@pytest.mark.parametrize("rng,mode", [("record", 1), ("occurrence", 2)])
@pytest.mark.parametrize("case", ["cfg1", "layers3", "exact", "batched"])
def test_rng_modes_vs_oracle(A, ctx, rng, mode, case, monkeypatch):
    cfg = aragen.load_config("cfg1")
    if case == "batched":
        monkeypatch.setenv("ARA_BATCH_TRIALS", "97")
    if case == "layers3":
        cfg.update(n_layers=3, elts_per_layer=4, catalog=4000, records_per_elt=600, n_trials=300,
                   layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(3)])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    g, cnt, hsh = A.run(ctx, P, Y, seed=cfg["seed"], debug=True, rng=rng, exact=(case == "exact"))
    ref = oracle.run(pf, yet, seed=cfg["seed"], rng_mode=mode)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), ref["count"])
    g = g.cpu().numpy()
    for li in range(g.shape[0]):
        ylt_check(g[li], ref, li)
    # a different reading gives different losses (the modes are wired through)
    g0 = A.run(ctx, P, Y, seed=cfg["seed"]).cpu().numpy()
    assert not np.array_equal(g0, g)


def test_rng_modes_exclusive(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 10
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    import torch
    ylt = torch.empty((1, 10), dtype=torch.float32, device="cuda")
    with pytest.raises(A.AraError):
        A._check(A.lib.ara_run(ctx.h, P.h, Y.h, 1, A.SU | 32 | 64, A._p(ylt), None, None))


# ---- exceedance curve (NEXT-3): the YLT sorted descending --------------------
@pytest.mark.parametrize("n", [1, 1000, 4097, 100003, 800000])
def test_exceedance_curve_is_the_sorted_ylt(A, ctx, n):
    import torch
    rng = np.random.default_rng(n)
    x = rng.lognormal(15, 1.2, n).astype(np.float32)
    x[rng.uniform(size=n) < 0.1] = 0.0                      # ties at 0 and at the limit
    x[rng.uniform(size=n) < 0.01] = np.float32(3.0e8)
    curve = A.exceedance_curve(ctx, torch.from_numpy(x).cuda(), 1, n, 0).cpu().numpy()
    assert np.array_equal(curve, np.sort(x)[::-1])           # a permutation: bit-exact


def test_exceedance_curve_rollup_shards_and_cfg1(A, ctx):
    import torch
    rng = np.random.default_rng(9)
    L, n, P = 3, 40000, 4
    y = rng.lognormal(12, 1, (P, L, n // P)).astype(np.float32)
    flat = y.transpose(1, 0, 2).reshape(L, n)
    d = torch.from_numpy(y).cuda()
    for layer in (-1, 1):
        v = (flat[0] + flat[1]) + flat[2] if layer < 0 else flat[layer]
        got = A.exceedance_curve(ctx, d, L, n, layer, n_shards=P).cpu().numpy()
        assert np.array_equal(got, np.sort(v)[::-1])
    # on a run's YLT: the curve's order statistics are the measures' inputs
    cfg = aragen.load_config("cfg1")
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    ylt = A.run(ctx, A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet), seed=cfg["seed"])
    curve = A.exceedance_curve(ctx, ylt, 1, cfg["n_trials"], 0).cpu().numpy()
    assert np.array_equal(curve, np.sort(ylt.cpu().numpy()[0])[::-1])
    _, _, var = A.risk_measures_var(ctx, ylt, 1, cfg["n_trials"], 0, rps=(10, 50))
    N = cfg["n_trials"]
    for q, rp in enumerate((10, 50)):
        assert var[q] == curve[-(-N // rp) - 1]               # VaR = L(ceil(N/RP))


# ---- portfolios larger than one kernel group (thousands of XELTs) ------
@pytest.mark.parametrize("n_layers,J", [(20, 16), (65, 3)])
def test_large_portfolio_in_groups(A, ctx, n_layers, J):
    # > 8 layers or > 224 (layer, XELT) slots: groups of consecutive layers,
    # one run each over the same YET; lookup exact, YLT / occ_max / roll-up
    # measures against the oracle
    cfg = aragen.load_config("cfg1")
    terms = [[1e5 * (l % 5 + 1), 5e6, 1.0e6, 5.0e7] for l in range(n_layers)]
    cfg.update(n_layers=n_layers, elts_per_layer=J, catalog=20000, records_per_elt=400,
               n_trials=200, layer_terms=terms)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    pf["layer_prog"] = (np.arange(n_layers) % 4).astype(np.uint32)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    g, cnt, hsh = A.run(ctx, P, Y, seed=31, debug=True)
    ref = oracle.run(pf, yet, seed=31)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), ref["count"])
    assert np.array_equal(hsh.cpu().numpy().view(np.uint64), ref["hash"])
    gn = g.cpu().numpy()
    for li in range(n_layers):
        ylt_check(gn[li], ref, li)
    ylt, occ = A.run_ep(ctx, P, Y, seed=31)
    assert np.array_equal(ylt.cpu().numpy(), gn)
    for li in (0, n_layers // 2, n_layers - 1):
        occ_check(occ.cpu().numpy()[li], ref, pf, li)
    pml, tvar = A.risk_measures(ctx, g, n_layers, cfg["n_trials"], -1, rps=(10, 50))
    o = OM.rollup(ref["ylt"])
    floor = FLOOR * ref["gross"].sum(axis=0).max()
    for q, rp in enumerate((10, 50)):
        assert abs(pml[q] - OM.pml(o, rp)) <= REL * abs(OM.pml(o, rp)) + floor
        assert abs(tvar[q] - OM.tvar_rp(o, rp)[1]) <= REL * abs(OM.tvar_rp(o, rp)[1]) + floor


def test_measures_batch_equals_single_calls(A, ctx):
    # the batched call (one read-back for every table) == one call per table
    import torch
    rng = np.random.default_rng(21)
    L, n, P = 5, 60000, 3
    y = torch.from_numpy(rng.lognormal(13, 1, (P, L, n // P)).astype(np.float32)).cuda()
    layers = [0, 3, -1, 4]
    pml, tvar, var = A.risk_measures_batch(ctx, y, L, n, layers, rps=(100, 250, 500), n_shards=P)
    for i, layer in enumerate(layers):
        p1, t1, v1 = A.risk_measures_var(ctx, y, L, n, layer, rps=(100, 250, 500), n_shards=P)
        assert np.array_equal(pml[i], p1) and np.array_equal(tvar[i], t1) and np.array_equal(var[i], v1)


def test_measures_async_equals_batch(A, ctx):
    # ara_risk_measures_async (device output, no sync) == the batched call, bit
    # for bit, also when queued behind other work and reused across calls
    import torch
    rng = np.random.default_rng(22)
    L, n, P = 3, 90000, 2
    layers = [0, -1, 2]
    out = torch.empty((len(layers), 3, 3), dtype=torch.float64, device="cuda")
    for rep in range(3):
        y = torch.from_numpy(rng.lognormal(13 + rep, 1, (P, L, n // P)).astype(np.float32)).cuda()
        A.risk_measures_async(ctx, y, L, n, layers, rps=(100, 250, 500), n_shards=P, out=out)
        torch.cuda.synchronize()
        pml, tvar, var = A.risk_measures_batch(ctx, y, L, n, layers, rps=(100, 250, 500), n_shards=P)
        o = out.cpu().numpy()
        assert np.array_equal(o[:, :, 0], pml) and np.array_equal(o[:, :, 1], tvar) and np.array_equal(o[:, :, 2], var)
    with pytest.raises(A.AraError):                   # host output buffer (binding check)
        A.risk_measures_async(ctx, y, L, n, layers, out=np.zeros((3, 3, 3)))
    with pytest.raises(A.AraError):                   # host output buffer (the library's check)
        A.risk_measures_async(ctx, y, L, n, layers, out=torch.zeros((3, 3, 3), dtype=torch.float64))
    with pytest.raises(A.AraError):                   # too small
        A.risk_measures_async(ctx, y, L, n, layers, out=torch.zeros((2, 3, 3), dtype=torch.float64, device="cuda"))


def test_batch_and_curve_errors(A, ctx):
    import torch
    y = torch.ones((2, 100), dtype=torch.float32, device="cuda")
    with pytest.raises(A.AraError):                   # > 4 return periods
        A.risk_measures_batch(ctx, y, 2, 100, [0, 1], rps=(2, 3, 4, 5, 6))
    with pytest.raises(A.AraError):                   # layer out of range
        A.risk_measures_batch(ctx, y, 2, 100, [0, 2])
    with pytest.raises(A.AraError):                   # return period <= 1
        A.risk_measures_batch(ctx, y, 2, 100, [0], rps=(1.0,))
    with pytest.raises(A.AraError):                   # layer out of range
        A.exceedance_curve(ctx, y, 2, 100, 3)
    with pytest.raises(A.AraError):                   # shards must divide n_total
        A.exceedance_curve(ctx, y, 2, 100, 0, n_shards=3)
    c = A.exceedance_curve(ctx, y, 2, 100, -1).cpu().numpy()
    assert (c == 2.0).all()                           # constant roll-up


# ---- the paper's data model: draws supplied with the inputs (NEXT-4) ---------
@pytest.mark.parametrize("case", ["cfg1", "layers3", "exact", "ragged", "ep"])
def test_supplied_z_vs_oracle(A, ctx, case):
    # z_(Prog,E) per YET occurrence and z_(E) per XELT record
    # given as inputs (ARA_RNG_SUPPLIED): the split path, ARA_EXACT, CSR
    # trials, several programs, and run_ep (fp64-capable kernel) against the
    # oracle fed the same numbers
    cfg = aragen.load_config("cfg1")
    if case == "layers3":
        cfg.update(n_layers=3, elts_per_layer=4, catalog=4000, records_per_elt=600, n_trials=300,
                   layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(3)])
    if case == "ragged":
        cfg.update(k_min=0, k_max=150, n_trials=700)
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    if case == "layers3":
        pf["layer_prog"] = np.array([0, 1, 1], np.uint32)
    rng = np.random.default_rng(123)
    n_prog = int(pf["layer_prog"].max()) + 1
    zp = ((rng.integers(0, 2 ** 23, (n_prog, yet["events"].size)) * 2 + 1) * 2.0 ** -24).astype(np.float32)
    ze = ((rng.integers(0, 2 ** 23, pf["rec_event"].size) * 2 + 1) * 2.0 ** -24).astype(np.float32)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    P.set_z(ze)
    Y.set_z(zp)
    ref = oracle.run(pf, yet, seed=cfg["seed"], z_prog=zp.astype(np.float64), z_event=ze.astype(np.float64))
    if case == "ep":
        g, _ = A.run_ep(ctx, P, Y, seed=cfg["seed"], rng="supplied")
        g = g.cpu().numpy()
    else:
        g, cnt, _ = A.run(ctx, P, Y, seed=cfg["seed"], debug=True, rng="supplied", exact=(case == "exact"))
        assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), ref["count"])
        g = g.cpu().numpy()
    for li in range(g.shape[0]):
        ylt_check(g[li], ref, li)
    # the seed plays no part: the numbers come with the inputs
    g2 = A.run(ctx, P, Y, seed=cfg["seed"] + 99, rng="supplied").cpu().numpy()
    assert np.array_equal(g2, A.run(ctx, P, Y, seed=cfg["seed"], rng="supplied").cpu().numpy())


def test_supplied_z_survives_packed_refill(A, ctx):
    # the YET's supplied z_(Prog,E) stay attached when its ids are re-uploaded
    # from a packed copy (the staging buffer grows on the first packed upload:
    # it once freed the z array with it -- a dangling pointer and a double free)
    cfg = aragen.load_config("cfg1")
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    rng = np.random.default_rng(7)
    zp = ((rng.integers(0, 2 ** 23, (1, yet["events"].size)) * 2 + 1) * 2.0 ** -24).astype(np.float32)
    ze = ((rng.integers(0, 2 ** 23, pf["rec_event"].size) * 2 + 1) * 2.0 ** -24).astype(np.float32)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    P.set_z(ze)
    Y.set_z(zp)
    before = A.run(ctx, P, Y, seed=1, rng="supplied").cpu().numpy()
    bits = aragen.yet_bits(cfg["catalog"])
    Y.refill_packed(aragen.pack_yet(np.ascontiguousarray(yet["events"], np.uint32), bits), bits)
    filler = A.Portfolio(ctx, pf)                 # allocations that could reuse a freed z array
    after = A.run(ctx, P, Y, seed=1, rng="supplied").cpu().numpy()
    assert np.array_equal(before, after)
    del filler, Y                                 # destroy: no double free, no error left behind
    P2 = A.Portfolio(ctx, pf)
    assert P2.info()["n_device_records"] > 0


def test_supplied_z_errors(A, ctx):
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 20
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    with pytest.raises(A.AraError):                       # nothing supplied yet
        A.run(ctx, P, Y, seed=1, rng="supplied")
    with pytest.raises(A.AraError):                       # z outside (0, 1)
        P.set_z(np.zeros(pf["rec_event"].size, np.float32))
    with pytest.raises(A.AraError):
        Y.set_z(np.ones(yet["events"].size, np.float32))
    P.set_z(np.full(pf["rec_event"].size, 0.5, np.float32))
    Y.set_z(np.full(yet["events"].size, 0.5, np.float32))
    pf2 = dict(pf, layer_prog=np.array([1], np.uint32))   # program 1 not supplied
    P2 = A.Portfolio(ctx, pf2)
    P2.set_z(np.full(pf["rec_event"].size, 0.5, np.float32))
    with pytest.raises(A.AraError):
        A.run(ctx, P2, Y, seed=1, rng="supplied")
    A.run(ctx, P, Y, seed=1, rng="supplied")


def test_group_byte_budget_splits_passes(A, ctx, monkeypatch):
    # ARA_GROUP_BYTES bounds each kernel group's gathered tables (one pass over
    # the YET per group): 1 group or one per layer -> the same
    # lookups bit for bit and the same YLT / occ_max up to the summation order
    # (a layer's runs are summed in stretches of the group's pair list, G28)
    cfg = aragen.load_config("cfg1")
    cfg.update(n_layers=4, elts_per_layer=3, catalog=5000, records_per_elt=800, n_trials=300,
               layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(4)])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    one = A.Portfolio(ctx, pf)
    monkeypatch.setenv("ARA_GROUP_BYTES", "1")
    per_layer = A.Portfolio(ctx, pf)
    monkeypatch.delenv("ARA_GROUP_BYTES")
    Y = A.Yet.from_dict(ctx, yet)
    a = A.run(ctx, one, Y, seed=4, debug=True)
    b = A.run(ctx, per_layer, Y, seed=4, debug=True)
    assert A.last_run_timings(ctx)["launches"] >= 8          # 4 groups x (compaction + sampler)
    assert np.array_equal(a[1].cpu().numpy(), b[1].cpu().numpy())
    assert np.array_equal(a[2].cpu().numpy(), b[2].cpu().numpy())
    ga, gb = a[0].cpu().numpy().astype(np.float64), b[0].cpu().numpy().astype(np.float64)
    assert (np.abs(ga - gb) <= 1e-6 * np.abs(ga) + 1e-3).all()
    ref = oracle.run(pf, yet, seed=4)
    for li in range(4):
        ylt_check(gb[li], ref, li)
    ea, eb = A.run_ep(ctx, one, Y, seed=4), A.run_ep(ctx, per_layer, Y, seed=4)
    ma, mb = ea[1].cpu().numpy().astype(np.float64), eb[1].cpu().numpy().astype(np.float64)
    assert (np.abs(ma - mb) <= 1e-6 * ma + 1e-3).all()


def test_shared_xelts_many_layers(A, ctx):
    # NEXT-2: 1,000 XELTs shared across 12 layers (each layer covers 200 of
    # them, so an XELT sits in ~2.4 layers; 12 kernel groups), several
    # programs; every (layer, XELT) slot reads the one quantile table of its
    # record (the record store), lookups bit-exact, YLT and roll-up measures
    # against the oracle
    rng = np.random.default_rng(2024)
    n_elts, R, C, L = 1000, 30, 10000, 12
    ev, mu, si, sc, mx = [], [], [], [], []
    for j in range(n_elts):
        e = np.sort(rng.choice(C, R, replace=False)).astype(np.uint32)
        m = (10 ** rng.uniform(4, 7, R)).astype(np.float32)
        ev.append(e); mu.append(m); mx.append((m * rng.uniform(2, 10, R)).astype(np.float32))
        si.append((m * rng.uniform(0.1, 0.5, R)).astype(np.float32)); sc.append((m * rng.uniform(0.05, 0.3, R)).astype(np.float32))
    lel = [np.sort(rng.choice(n_elts, 200, replace=False)).astype(np.uint32) for _ in range(L)]
    pf = {"catalog_size": C, "elt_off": np.arange(n_elts + 1, dtype=np.uint64) * np.uint64(R),
          "rec_event": np.concatenate(ev), "rec_mean": np.concatenate(mu), "rec_sigma_i": np.concatenate(si),
          "rec_sigma_c": np.concatenate(sc), "rec_max": np.concatenate(mx), "elt_terms": None,
          "layer_prog": (np.arange(L) % 3).astype(np.uint32),
          "layer_elt_off": np.arange(L + 1, dtype=np.uint64) * np.uint64(200),
          "layer_elts": np.concatenate(lel),
          "layer_terms": np.array([[2e5 * (l % 4 + 1), 5e6, 5e7, 5e8] for l in range(L)])}
    cfg = aragen.load_config("cfg1")
    cfg.update(catalog=C, n_trials=300, events_per_trial=200)
    yet = aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    info = P.info()
    n_dev = info["n_device_records"]
    assert n_dev == L * 200 * R
    g, cnt, hsh = A.run(ctx, P, Y, seed=8, debug=True)
    ref = oracle.run(pf, yet, seed=8)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), ref["count"])
    assert np.array_equal(hsh.cpu().numpy().view(np.uint64), ref["hash"])
    gn = g.cpu().numpy()
    for li in range(L):
        ylt_check(gn[li], ref, li)
    pml, tvar = A.risk_measures(ctx, g, L, cfg["n_trials"], -1, rps=(10, 50))
    o = OM.rollup(ref["ylt"])
    for q, rp in enumerate((10, 50)):
        assert pml[q] == pytest.approx(OM.pml(o, rp), rel=1e-4)
        assert tvar[q] == pytest.approx(OM.tvar_rp(o, rp)[1], rel=1e-4)
    # one table per input record (the record store: n_elts * R = 30k tables, not one
    # per device record: 72k): <= 200 B per device record (484 B in round 1)
    per_dev = info["device_bytes"] / n_dev
    assert per_dev <= 200, (info, per_dev)


# ---- ARA_ASYNC: no host synchronisation inside ara_run ----------------------
@pytest.mark.parametrize("case", ["split", "primary", "overflow", "capped", "exact", "groups"])
def test_async_runs_equal_sync(A, ctx, case, monkeypatch):
    # the same YLT, counts and hashes bit for bit, whether ara_run waits for
    # its status (sync: host-sized overflow / redo passes) or not (device-sized
    # passes); errors none
    cfg = aragen.load_config("cfg1")
    if case == "groups":
        cfg.update(n_layers=4, elts_per_layer=3, catalog=5000, records_per_elt=800, n_trials=300,
                   layer_terms=[[2e5 * (l + 1), 5e6, 1.0e6, 5.0e7] for l in range(4)])
        monkeypatch.setenv("ARA_GROUP_BYTES", "1")
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    if case == "capped":
        pf["rec_sigma_i"] = pf["rec_sigma_i"].copy()
        pf["rec_sigma_i"][::7] = pf["rec_max"][::7]          # table-less records: the fp64 redo pass
    if case == "overflow":
        monkeypatch.setenv("ARA_PAIR_CAP", "1")              # every trial through the overflow pass
    P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
    kw = dict(seed=13, su=case != "primary", exact=case == "exact")
    ref = A.run(ctx, P, Y, **kw)
    got = A.run(ctx, P, Y, async_=True, **kw)
    ctx.synchronize()
    assert np.array_equal(ref.cpu().numpy(), got.cpu().numpy())
    if case != "primary":
        r2 = A.run(ctx, P, Y, debug=True, **kw)
        g2 = A.run(ctx, P, Y, debug=True, async_=True, **kw)
        ctx.synchronize()
        for x, y in zip(r2, g2):
            assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())
    assert A.last_run_timings(ctx)["sample_ms"] > 0


def test_async_errors_reported_at_synchronize(A, monkeypatch):
    ctx2 = A.Context(0)                                      # a fresh context: a small pre-sized pool
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 200
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    P, Y = A.Portfolio(ctx2, pf), A.Yet.from_dict(ctx2, yet)
    monkeypatch.setenv("ARA_PAIR_CAP", "1")
    monkeypatch.setenv("ARA_ASYNC_POOL_PAIRS", "100")
    A.run(ctx2, P, Y, seed=1, async_=True)                   # returns at once
    with pytest.raises(A.AraError) as ei:
        ctx2.synchronize()
    assert ei.value.code == A.ENOMEM
    ctx2.synchronize()                                       # the latch is cleared
    monkeypatch.delenv("ARA_PAIR_CAP")
    yet["events"][17] = cfg["catalog"]                       # an event id out of range
    Y2 = A.Yet.from_dict(ctx2, yet)
    A.run(ctx2, P, Y2, seed=1, async_=True)
    with pytest.raises(A.AraError) as ei:
        ctx2.synchronize()
    assert ei.value.code == A.ERANGE


# ---- multi-rank bench path through libara (ranks sharing the GPU over gloo) ----
@pytest.mark.parametrize("cfg_name,ranks", [("cfg1", 2), ("cfg1", 3), ("layers5", 2), ("layers5", 3)])
def test_bench_multirank_measures_equal(cfg_name, ranks, tmp_path):
    # bench.py's multi-rank path (trial shards with global Philox keys, the YLT
    # all-gather, measures on the gathered layout, max-over-ranks timing) with
    # libara on every rank: 2 and 3 ranks (unequal shards for 3) sharing one GPU
    # over gloo print the same PML / TVaR as the 1-rank run
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if cfg_name == "layers5":                 # cfg5's shape, small: 5 layers + the roll-up = 6 tables, each
        cfg = aragen.load_config("cfg5")      # rank computing its round-robin share (bench.table_shard)
        cfg.update(name="layers5", n_layers=5, n_trials=3000, catalog=200000, records_per_elt=4000,
                   layer_terms=cfg["layer_terms"][:5])
        cfg_name = str(tmp_path / "layers5.json")
        with open(cfg_name, "w") as f:
            json.dump(cfg, f)
    args = ["--config", cfg_name, "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    one = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    env = dict(os.environ, ARA_BENCH_BACKEND="gloo")
    port = str(29600 + ranks)
    multi = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                            f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port", port,
                            os.path.join(root, "bench.py"), "--gpus", str(ranks)] + args,
                           cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert multi.returncode == 0, multi.stderr[-2000:]
    a = json.loads(one.stdout.strip().splitlines()[-1])
    b = json.loads(multi.stdout.strip().splitlines()[-1])
    assert b["n_gpus"] == ranks and a["measures"] == b["measures"]


@pytest.mark.parametrize("su", [True, False])
def test_large_catalog_coarse_bitmap(A, ctx, su):
    # a 5M-event catalogue: the shared-memory bitmap holds one bit per 8 events
    # (shift 3), so most bitmap hits are false and the index entry (or, without
    # draws, the occurrence loss) decides; lookups bit-exact, YLT within the bar
    cfg = aragen.load_config("cfg3")
    cfg.update(catalog=5_000_000, n_layers=1, elts_per_layer=4, records_per_elt=50_000, n_trials=1500,
               layer_terms=[[2e5, 5e6, 1.0e5, 5.0e9]])
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    (g, cnt, hsh), ref = run_both(A, ctx, pf, yet, seed=17, su=su)
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(hsh, ref["hash"])
    ylt_check(g[0], ref, 0)
    if not su:                                  # the primary kernel (no debug lookup) on the same trials
        P, Y = A.Portfolio(ctx, pf), A.Yet.from_dict(ctx, yet)
        gp = A.run(ctx, P, Y, seed=17, su=False).cpu().numpy()
        ylt_check(gp[0], ref, 0)
