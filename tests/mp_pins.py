"""Independent pins computed with mpmath (test helper; no method arithmetic of
the oracle or the CUDA path)."""


def mp_lower_quantile(p, a, b):
    """x with I_x(a, b) = p by bisection on ln x at 40 digits (mpmath's own
    regularised incomplete beta): an independent pin for the tiny-parameter,
    near-Bernoulli regime that scipy's double-precision inverse cannot resolve
    below ~1e-308."""
    import mpmath as mp
    with mp.workdps(40):
        p, a, b = mp.mpf(p), mp.mpf(a), mp.mpf(b)
        f = lambda u: mp.betainc(a, b, 0, mp.e ** u, regularized=True) - p  # noqa: E731
        lo, hi = mp.mpf(-800000), mp.mpf(0)
        if f(lo) >= 0:
            return 0.0
        for _ in range(110):
            m = (lo + hi) / 2
            if f(m) < 0:
                lo = m
            else:
                hi = m
        return float(mp.e ** ((lo + hi) / 2))
