"""Pins for the oracle's Algorithm 1 and financial terms
(P:176-179): SPEC worked examples, a brute-force straight-line reference in
pure Python (its own Philox, scipy special functions, linear search over the
XELT records instead of the direct-access table), exact integer sums with
sigma = 0, additivity over XELTs, order invariance (G6), thread-count
determinism."""
import numpy as np
import pytest
import scipy.special as sp

import oracle as O

M32 = 0xFFFFFFFF


def philox_py(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c3 ^ k1) & M32, p0 & M32
    return c0, c1, c2, c3


def u_py(x):
    return (2 * (x >> 9) + 1) * 2.0 ** -24


def loss_py(mu, si, sc, mx, zp, ze):
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
    return mx * sp.betaincinv(a, b, z) if z <= 0.5 else mx * (1 - sp.betaincinv(b, a, q))


def brute_force(pf, yet, seed, su, trial_index, rng_mode=0, z_prog=None, z_event=None):
    """Straight-line Algorithm 1: linear search over each XELT's record list.
    z_prog [program][occurrence] / z_event [record] given: the paper's data
    model, draws supplied with the YET and the XELT records."""
    key = (seed & M32, (seed >> 32) & M32)
    nl = len(pf["layer_prog"])
    n = len(yet["trial_off"]) - 1
    ylt = np.zeros((nl, n)); gross = np.zeros((nl, n)); occ_max = np.zeros((nl, n))
    for li in range(nl):
        p = int(pf["layer_prog"][li])
        occr, occl, aggr, aggl = pf["layer_terms"][li]
        elts = pf["layer_elts"][int(pf["layer_elt_off"][li]):int(pf["layer_elt_off"][li + 1])]
        for t in range(n):
            i = int(trial_index[t])
            S = 0.0
            evs = yet["events"][int(yet["trial_off"][t]):int(yet["trial_off"][t + 1])]
            for k, e in enumerate(evs):
                l = 0.0
                for j in elts:
                    j = int(j)
                    lo, hi = int(pf["elt_off"][j]), int(pf["elt_off"][j + 1])
                    hit = [r for r in range(lo, hi) if int(pf["rec_event"][r]) == int(e)]
                    if not hit:
                        continue
                    r = hit[0]
                    mu, si, sc, mx = (float(pf[f][r]) for f in
                                      ("rec_mean", "rec_sigma_i", "rec_sigma_c", "rec_max"))
                    if su:
                        o = int(yet["trial_off"][t]) + k
                        zp = u_py(philox_py((i & M32, k, p, 1), key)[0]) if z_prog is None else float(z_prog[p][o])
                        if z_event is not None:  # supplied with the record
                            ze = float(z_event[r])
                        elif rng_mode == 1:      # (A) z_E stored per XELT record
                            ze = u_py(philox_py((r - lo, j, 0, 6), key)[0])
                        elif rng_mode == 2:      # (B) z_E per occurrence, shared by XELTs
                            ze = u_py(philox_py((i & M32, k, 0, 7), key)[0])
                        else:
                            ze = u_py(philox_py((i & M32, k, j, 2), key)[0])
                        x = loss_py(mu, si, sc, mx, zp, ze)
                    else:
                        x = mu
                    if pf.get("elt_terms") is not None:
                        R, Lm, sh = pf["elt_terms"][j]
                        x = sh * min(max(x - R, 0.0), Lm)
                    l += x
                g = min(max(l - occr, 0.0), occl)
                S += g
                occ_max[li, t] = max(occ_max[li, t], g)
            gross[li, t] = S
            ylt[li, t] = min(max(S - aggr, 0.0), aggl)
    brute_force.occ_max = occ_max
    return ylt, gross


def tiny_case(rng, n_layers=None, n_elts=None, n_trials=None, sigma=True, integer=False,
              xelt_terms=False):
    C = int(rng.integers(5, 40))
    n_elts = n_elts or int(rng.integers(1, 5))
    recs = {k: [] for k in ("rec_event", "rec_mean", "rec_sigma_i", "rec_sigma_c", "rec_max")}
    off = [0]
    for j in range(n_elts):
        R = int(rng.integers(0, C + 1))
        evs = rng.choice(C, size=R, replace=False)
        for e in evs:
            mu = float(rng.integers(1, 1000)) if integer else float(10 ** rng.uniform(2, 6))
            recs["rec_event"].append(int(e))
            recs["rec_mean"].append(mu)
            recs["rec_max"].append(mu * float(rng.uniform(1.5, 8)) if not integer else mu * 3)
            recs["rec_sigma_i"].append(mu * float(rng.uniform(0, 0.4)) if sigma else 0.0)
            recs["rec_sigma_c"].append(mu * float(rng.uniform(0, 0.3)) if sigma else 0.0)
        off.append(off[-1] + R)
    nl = n_layers or int(rng.integers(1, 4))
    lel, loff = [], [0]
    for _ in range(nl):
        m = int(rng.integers(1, n_elts + 1))
        lel += sorted(rng.choice(n_elts, size=m, replace=False).tolist())
        loff.append(len(lel))
    if integer:
        terms = [[float(rng.integers(0, 500)), float(rng.integers(1, 3000)),
                  float(rng.integers(0, 2000)), float(rng.integers(1, 20000))] for _ in range(nl)]
    else:
        terms = [[float(rng.uniform(0, 1e4)), float(rng.uniform(1e4, 1e6)),
                  float(rng.uniform(0, 1e5)), float(rng.uniform(1e5, 1e7))] for _ in range(nl)]
    pf = {"catalog_size": C, "elt_off": np.array(off, np.uint64),
          **{k: np.array(v, np.uint32 if k == "rec_event" else np.float64) for k, v in recs.items()},
          "elt_terms": (np.array([[float(rng.uniform(0, 100)), float(rng.uniform(1e3, 1e5)),
                                   float(rng.uniform(0.1, 1))] for _ in range(n_elts)])
                        if xelt_terms else None),
          "layer_prog": rng.integers(0, 3, nl).astype(np.uint32),
          "layer_elt_off": np.array(loff, np.uint64), "layer_elts": np.array(lel, np.uint32),
          "layer_terms": np.array(terms)}
    n = n_trials or int(rng.integers(1, 20))
    lens = rng.integers(0, 11, n)
    toff = np.zeros(n + 1, np.uint64); toff[1:] = np.cumsum(lens)
    yet = {"trial_off": toff, "events": rng.integers(0, C, int(toff[-1])).astype(np.uint32)}
    return pf, yet


def test_occ_agg_terms_examples(golden):
    for c in golden["occ_terms"]:
        assert O.occ_terms(c["l"], c["R"], c["L"]) == c["y"], c["src"]
    for c in golden["agg_terms"]:
        assert O.agg_terms(c["s"], c["R"], c["L"]) == c["y"], c["src"]
    assert O.xelt_terms(150.0, 100.0, 30.0, 0.5) == 15.0


@pytest.mark.parametrize("seed", range(100))
def test_engine_vs_brute_force(seed):
    # <= 3 layers x 4 XELTs x 20 trials x 10 events, 100 seeds
    rng = np.random.default_rng(1000 + seed)
    pf, yet = tiny_case(rng, xelt_terms=(seed % 4 == 0))
    su = seed % 5 != 0
    tidx = rng.integers(0, 2 ** 32, len(yet["trial_off"]) - 1, dtype=np.uint64)
    rseed = int(rng.integers(0, 2 ** 63))
    got = O.run(pf, yet, seed=rseed, su=su, n_threads=2, trial_index=tidx)
    ylt, gross = brute_force(pf, yet, rseed, su, tidx)
    np.testing.assert_allclose(got["gross"], gross, rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(got["occ_max"], brute_force.occ_max, rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(got["ylt"], ylt, rtol=1e-9, atol=1e-6 * max(1.0, gross.max()))


def test_engine_integer_sigma0_exact():
    rng = np.random.default_rng(77)
    for _ in range(20):
        pf, yet = tiny_case(rng, sigma=False, integer=True)
        got = O.run(pf, yet, seed=1, su=True)
        ylt, gross = brute_force(pf, yet, 1, False, np.arange(len(yet["trial_off"]) - 1))
        assert np.array_equal(got["gross"], gross)
        assert np.array_equal(got["ylt"], ylt)
        assert np.array_equal(got["ylt"], np.round(got["ylt"]))


def test_engine_sigma0_su_on_equals_su_off():
    rng = np.random.default_rng(78)
    pf, yet = tiny_case(rng, sigma=False, n_trials=15)
    a = O.run(pf, yet, seed=9, su=True)
    b = O.run(pf, yet, seed=9, su=False)
    assert np.array_equal(a["ylt"], b["ylt"])


def test_engine_lookup_count_and_hash():
    rng = np.random.default_rng(79)
    pf, yet = tiny_case(rng, n_layers=2, n_elts=3, n_trials=12)
    got = O.run(pf, yet, seed=3, su=False)
    for li in range(2):
        elts = pf["layer_elts"][int(pf["layer_elt_off"][li]):int(pf["layer_elt_off"][li + 1])]
        for t in range(12):
            evs = yet["events"][int(yet["trial_off"][t]):int(yet["trial_off"][t + 1])]
            cnt, h = 0, 0
            for k, e in enumerate(evs):
                for j in elts:
                    lo, hi = int(pf["elt_off"][j]), int(pf["elt_off"][j + 1])
                    for r in range(lo, hi):
                        if pf["rec_event"][r] == e:
                            cnt += 1
                            h = (h + O.lookup_hash(k, int(j), r - lo)) % 2 ** 64
            assert got["count"][li, t] == cnt
            assert int(got["hash"][li, t]) == h


def test_engine_additivity_over_xelts():
    # identity terms (OccR=0, OccL=inf, AggR=0, AggL=inf): YLT(A u B) = YLT(A) + YLT(B)
    rng = np.random.default_rng(80)
    pf, yet = tiny_case(rng, n_layers=1, n_elts=4, n_trials=15)
    pf["layer_terms"] = np.array([[0.0, np.inf, 0.0, np.inf]])
    pf["layer_prog"] = np.zeros(1, np.uint32)

    def with_elts(elts):
        q = dict(pf)
        q["layer_elts"] = np.array(elts, np.uint32)
        q["layer_elt_off"] = np.array([0, len(elts)], np.uint64)
        return O.run(q, yet, seed=5, su=True)["ylt"][0]

    np.testing.assert_allclose(with_elts([0, 1, 2, 3]), with_elts([0, 1]) + with_elts([2, 3]),
                               rtol=1e-12)


def test_engine_yearloss_order_invariant_sigma0():
    # reading G6: with sigma = 0 the year loss g_agg(sum_k g_occ(l_k)) does not
    # depend on the order of occurrences, even when the aggregate limit binds.
    rng = np.random.default_rng(81)
    pf, yet = tiny_case(rng, sigma=False, integer=True, n_trials=10)
    base = O.run(pf, yet, seed=1, su=False)["ylt"]
    ev = yet["events"].copy()
    for t in range(10):
        s, e = int(yet["trial_off"][t]), int(yet["trial_off"][t + 1])
        ev[s:e] = rng.permutation(ev[s:e])
    perm = O.run(pf, {"trial_off": yet["trial_off"], "events": ev}, seed=1, su=False)["ylt"]
    assert np.array_equal(base, perm)


def test_engine_thread_count_determinism():
    rng = np.random.default_rng(82)
    pf, yet = tiny_case(rng, n_trials=19)
    outs = [O.run(pf, yet, seed=11, su=True, n_threads=t) for t in (1, 2, 8)]
    for o in outs[1:]:
        for k in ("ylt", "gross", "count", "hash"):
            assert np.array_equal(o[k], outs[0][k])


def test_engine_empty_and_bounds():
    rng = np.random.default_rng(83)
    pf, _ = tiny_case(rng, n_trials=3)
    yet = {"trial_off": np.zeros(4, np.uint64), "events": np.zeros(0, np.uint32)}
    out = O.run(pf, yet, seed=1, su=True)
    assert (out["ylt"] == 0).all() and (out["count"] == 0).all()
    pf2, yet2 = tiny_case(rng, n_trials=15)
    out2 = O.run(pf2, yet2, seed=2, su=True)
    for li in range(len(pf2["layer_prog"])):
        assert (out2["ylt"][li] >= 0).all() and (out2["ylt"][li] <= pf2["layer_terms"][li][3]).all()
    bad = dict(yet2); bad["events"] = yet2["events"].copy()
    if bad["events"].size:
        bad["events"][0] = pf2["catalog_size"]
        with pytest.raises(O.OracleError):
            O.run(pf2, bad, seed=2)


# ---- OEP basis: the largest occurrence loss per (layer, trial) (reading G29)
def test_occ_max_properties():
    # 0 <= occ_max <= OccL; occ_max <= S <= K * occ_max (S is a sum of K terms,
    # each in [0, occ_max])
    rng = np.random.default_rng(91)
    for _ in range(30):
        pf, yet = tiny_case(rng)
        got = O.run(pf, yet, seed=int(rng.integers(0, 2 ** 40)), su=True)
        K = np.diff(yet["trial_off"]).astype(np.float64)
        occl = np.asarray(pf["layer_terms"])[:, 1][:, None]
        m, S = got["occ_max"], got["gross"]
        assert (m >= 0).all() and (m <= occl).all()
        assert (m <= S * (1 + 1e-12) + 1e-9).all()
        assert (S <= K[None, :] * m * (1 + 1e-12) + 1e-9).all()


def test_occ_max_single_occurrence_equals_gross():
    # one occurrence per trial: the trial sum has one term, so occ_max == S
    rng = np.random.default_rng(92)
    pf, yet = tiny_case(rng, n_trials=19)
    n = 19
    yet = {"trial_off": np.arange(n + 1, dtype=np.uint64),
           "events": rng.integers(0, pf["catalog_size"], n).astype(np.uint32)}
    got = O.run(pf, yet, seed=5, su=True)
    assert np.array_equal(got["occ_max"], got["gross"])


def test_occ_max_sigma0_is_max_of_means():
    # sigma = 0, one XELT, OccR = 0, OccL = inf: each occurrence loss is the
    # record's mean (or 0 if absent), so occ_max = max over the trial's events
    # of the mean -- computed here straight from the record arrays
    rng = np.random.default_rng(93)
    pf, yet = tiny_case(rng, n_layers=1, n_elts=1, sigma=False, n_trials=25)
    pf["layer_elt_off"] = np.array([0, 1], np.uint64)
    pf["layer_elts"] = np.array([0], np.uint32)
    pf["layer_terms"] = np.array([[0.0, np.inf, 0.0, np.inf]])
    mean_of = dict(zip(pf["rec_event"][:int(pf["elt_off"][1])].tolist(),
                       pf["rec_mean"][:int(pf["elt_off"][1])].tolist()))
    got = O.run(pf, yet, seed=3, su=True)
    for t in range(25):
        evs = yet["events"][int(yet["trial_off"][t]):int(yet["trial_off"][t + 1])]
        want = max([mean_of.get(int(e), 0.0) for e in evs], default=0.0)
        assert got["occ_max"][0, t] == want


# ---- paper-literal RNG alternatives of reading G2 (NEXT-4) ------------------
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("seed", range(20))
def test_engine_rng_modes_vs_brute_force(mode, seed):
    rng = np.random.default_rng(5000 + 100 * mode + seed)
    pf, yet = tiny_case(rng, xelt_terms=(seed % 3 == 0))
    tidx = rng.integers(0, 2 ** 32, len(yet["trial_off"]) - 1, dtype=np.uint64)
    rseed = int(rng.integers(0, 2 ** 63))
    got = O.run(pf, yet, seed=rseed, su=True, n_threads=2, trial_index=tidx, rng_mode=mode)
    ylt, gross = brute_force(pf, yet, rseed, True, tidx, rng_mode=mode)
    np.testing.assert_allclose(got["gross"], gross, rtol=1e-9, atol=1e-6)


def _one_record_case(n_elts, n_trials=40):
    # every XELT holds the same single record on event 3 (sigma_I = 0, so
    # v = v_E); identity terms; each trial is one occurrence of event 3
    pf = {"catalog_size": 10, "elt_off": np.arange(n_elts + 1, dtype=np.uint64),
          "rec_event": np.full(n_elts, 3, np.uint32), "rec_mean": np.full(n_elts, 1000.0),
          "rec_sigma_i": np.zeros(n_elts), "rec_sigma_c": np.full(n_elts, 300.0),
          "rec_max": np.full(n_elts, 5000.0), "elt_terms": None,
          "layer_prog": np.zeros(1, np.uint32), "layer_elt_off": np.array([0, n_elts], np.uint64),
          "layer_elts": np.arange(n_elts, dtype=np.uint32),
          "layer_terms": np.array([[0.0, np.inf, 0.0, np.inf]])}
    yet = {"trial_off": np.arange(n_trials + 1, dtype=np.uint64), "events": np.full(n_trials, 3, np.uint32)}
    return pf, yet


def test_rng_mode_record_constant_across_trials():
    # (A): the record's z_E is a property of the record -> with sigma_I = 0 its
    # loss is the same in every trial; under G2 it varies
    pf, yet = _one_record_case(1)
    a = O.run(pf, yet, seed=11, rng_mode=1)["ylt"][0]
    g = O.run(pf, yet, seed=11, rng_mode=0)["ylt"][0]
    assert np.all(a == a[0]) and np.unique(g).size == g.size
    assert a[0] == O.sample_loss(1000.0, 0.0, 300.0, 5000.0, 0.5, O.z_event_record(11, 0, 0))


def test_rng_mode_occurrence_shared_by_xelts():
    # (B): one z_E per occurrence for every XELT -> identical records in two
    # XELTs give equal losses, so the two-XELT trial loss is exactly twice the
    # one-XELT loss; under G2 the two draws differ
    pf2, yet = _one_record_case(2)
    pf1, _ = _one_record_case(1)
    two = O.run(pf2, yet, seed=12, rng_mode=2)["ylt"][0]
    one = O.run(pf1, yet, seed=12, rng_mode=2)["ylt"][0]
    assert np.array_equal(two, 2.0 * one)
    two0 = O.run(pf2, yet, seed=12, rng_mode=0)["ylt"][0]
    one0 = O.run(pf1, yet, seed=12, rng_mode=0)["ylt"][0]
    assert not np.array_equal(two0, 2.0 * one0)


# ---- the paper's data model: z_(Prog,E) in the YET, z_(E) in the XELT (NEXT-4)
def _supplied(rng, pf, yet):
    n_prog = int(pf["layer_prog"].max()) + 1
    zp = (rng.integers(0, 2 ** 23, (n_prog, yet["events"].size)) * 2 + 1) * 2.0 ** -24
    ze = (rng.integers(0, 2 ** 23, pf["rec_event"].size) * 2 + 1) * 2.0 ** -24
    return zp, ze


@pytest.mark.parametrize("seed", range(20))
def test_engine_supplied_z_vs_brute_force(seed):
    rng = np.random.default_rng(7000 + seed)
    pf, yet = tiny_case(rng, xelt_terms=(seed % 3 == 0))
    zp, ze = _supplied(rng, pf, yet)
    tidx = rng.integers(0, 2 ** 32, len(yet["trial_off"]) - 1, dtype=np.uint64)
    got = O.run(pf, yet, seed=1, su=True, n_threads=2, trial_index=tidx, z_prog=zp, z_event=ze)
    ylt, gross = brute_force(pf, yet, 1, True, tidx, z_prog=zp, z_event=ze)
    np.testing.assert_allclose(got["gross"], gross, rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(got["ylt"], ylt, rtol=1e-9, atol=1e-6)


def test_engine_supplied_z_reproduces_record_mode():
    # supplying the very numbers reading (A) draws -- z_(Prog,E) = Philox
    # (i, k, p, 1) per occurrence, z_(E) = Philox (r, j, 0, 6) per record --
    # gives the (A) run bit for bit: the supplied path changes only where the
    # numbers come from
    rng = np.random.default_rng(71)
    pf, yet = tiny_case(rng, n_layers=3, n_elts=4, n_trials=15)
    seed = 987654321
    n = len(yet["trial_off"]) - 1
    n_prog = int(pf["layer_prog"].max()) + 1
    zp = np.empty((n_prog, yet["events"].size))
    for p_ in range(n_prog):
        for t in range(n):
            for o in range(int(yet["trial_off"][t]), int(yet["trial_off"][t + 1])):
                zp[p_, o] = O.z_prog(seed, p_, t, o - int(yet["trial_off"][t]))
    ze = np.empty(pf["rec_event"].size)
    for j in range(len(pf["elt_off"]) - 1):
        for r in range(int(pf["elt_off"][j]), int(pf["elt_off"][j + 1])):
            ze[r] = O.z_event_record(seed, j, r - int(pf["elt_off"][j]))
    a = O.run(pf, yet, seed=seed, rng_mode=1)
    b = O.run(pf, yet, seed=seed, z_prog=zp, z_event=ze)
    assert np.array_equal(a["ylt"], b["ylt"]) and np.array_equal(a["gross"], b["gross"])


def test_engine_supplied_median_draws():
    # z_(Prog,E) = z_(E) = 1/2 -> v = 0 -> every loss is max_l times the
    # Beta(alpha, beta) median (scipy), a closed-form run
    rng = np.random.default_rng(72)
    pf, yet = tiny_case(rng, n_layers=1, n_elts=3, n_trials=10)
    zp = np.full((int(pf["layer_prog"].max()) + 1, yet["events"].size), 0.5)
    ze = np.full(pf["rec_event"].size, 0.5)
    got = O.run(pf, yet, seed=3, z_prog=zp, z_event=ze)
    med = np.empty(pf["rec_event"].size)
    for r in range(med.size):
        mu, si, sc, mx = (float(pf[f][r]) for f in ("rec_mean", "rec_sigma_i", "rec_sigma_c", "rec_max"))
        if si + sc == 0:
            med[r] = mu
            continue
        a, b = O.beta_params(mu, si + sc, mx)
        med[r] = mx * sp.betaincinv(a, b, 0.5)
    occr, occl, aggr, aggl = pf["layer_terms"][0]
    elts = pf["layer_elts"][:int(pf["layer_elt_off"][1])]
    for t in range(len(yet["trial_off"]) - 1):
        S = 0.0
        for e in yet["events"][int(yet["trial_off"][t]):int(yet["trial_off"][t + 1])]:
            l = sum(med[r] for j in elts for r in range(int(pf["elt_off"][j]), int(pf["elt_off"][j + 1]))
                    if int(pf["rec_event"][r]) == int(e))
            S += min(max(l - occr, 0.0), occl)
        assert got["gross"][0, t] == pytest.approx(S, rel=1e-10, abs=1e-6)
