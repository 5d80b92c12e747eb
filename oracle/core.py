"""ctypes wrapper over ``liboracle.so`` (the fp64 C oracle).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Compiles the C file
with plain ``gcc -O2`` (no fast-math) on first use if the library is missing
or older than its source.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ara_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

__all__ = [
    "build_oracle", "lib", "philox4x32_10", "u01", "z_prog", "z_event", "z_event_record", "z_event_occ",
    "norm_cdf", "norm_quantile", "lnbeta", "beta_cdf", "beta_quantile",
    "beta_params", "combine", "sample_loss", "sample_batch", "occ_terms", "agg_terms",
    "xelt_terms", "lookup_hash", "run", "OracleError",
]


class OracleError(RuntimeError):
    pass


def build_oracle(force: bool = False) -> str:
    """Compile ``liboracle.so`` (fp64, IEEE, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build_oracle())
        d, u32, u64, i32 = C.c_double, C.c_uint32, C.c_uint64, C.c_int
        P = C.POINTER
        L.orc_philox4x32_10.argtypes = [P(u32), P(u32), P(u32)]
        L.orc_u01.argtypes = [u32]; L.orc_u01.restype = d
        L.orc_z_prog.argtypes = [u64, u32, u64, u32]; L.orc_z_prog.restype = d
        L.orc_z_event.argtypes = [u64, u64, u32, u32]; L.orc_z_event.restype = d
        L.orc_norm_cdf.argtypes = [d]; L.orc_norm_cdf.restype = d
        L.orc_norm_quantile.argtypes = [d]; L.orc_norm_quantile.restype = d
        L.orc_lnbeta.argtypes = [d, d]; L.orc_lnbeta.restype = d
        L.orc_beta_cdf.argtypes = [d, d, d]; L.orc_beta_cdf.restype = d
        L.orc_beta_quantile.argtypes = [d, d, d, P(d)]; L.orc_beta_quantile.restype = i32
        L.orc_beta_params.argtypes = [d, d, d, P(d), P(d)]
        L.orc_combine.argtypes = [d, d, d, d, P(d), P(d)]; L.orc_combine.restype = d
        L.orc_sample_loss.argtypes = [d, d, d, d, d, d, P(d)]; L.orc_sample_loss.restype = i32
        L.orc_occ_terms.argtypes = [d, d, d]; L.orc_occ_terms.restype = d
        L.orc_agg_terms.argtypes = [d, d, d]; L.orc_agg_terms.restype = d
        L.orc_xelt_terms.argtypes = [d, d, d, d]; L.orc_xelt_terms.restype = d
        L.orc_sample_batch.argtypes = [u64] + [C.c_void_p] * 7
        L.orc_sample_batch.restype = i32
        L.orc_lookup_hash.argtypes = [u32, u32, u32]; L.orc_lookup_hash.restype = u64
        vp = C.c_void_p
        L.orc_run.argtypes = [u32, u32, vp, vp, vp, vp, vp, vp, vp,
                              u32, vp, vp, vp, vp, u64, vp, vp, vp,
                              u64, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp]
        L.orc_run.restype = i32
        L.orc_z_event_record.argtypes = [u64, u32, u32]; L.orc_z_event_record.restype = d
        L.orc_z_event_occ.argtypes = [u64, u64, u32]; L.orc_z_event_occ.restype = d
        _lib = L
    return _lib


# ---- scalar helpers (thin) -------------------------------------------------
def philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def u01(x):
    return lib().orc_u01(int(x))


def z_prog(seed, p, i, k):
    return lib().orc_z_prog(seed, p, i, k)


def z_event(seed, i, k, j):
    return lib().orc_z_event(seed, i, k, j)


def z_event_record(seed, j, r):
    return lib().orc_z_event_record(seed, j, r)


def z_event_occ(seed, i, k):
    return lib().orc_z_event_occ(seed, i, k)


def norm_cdf(v):
    return lib().orc_norm_cdf(float(v))


def norm_quantile(p):
    return lib().orc_norm_quantile(float(p))


def lnbeta(a, b):
    return lib().orc_lnbeta(float(a), float(b))


def beta_cdf(x, a, b):
    return lib().orc_beta_cdf(float(x), float(a), float(b))


def beta_quantile(p, a, b, return_iters=False):
    out = C.c_double()
    it = lib().orc_beta_quantile(float(p), float(a), float(b), C.byref(out))
    if it < 0:
        raise OracleError(f"beta quantile did not converge: p={p} a={a} b={b}")
    return (out.value, it) if return_iters else out.value


def beta_params(mu_l, sigma, max_l):
    a, b = C.c_double(), C.c_double()
    lib().orc_beta_params(float(mu_l), float(sigma), float(max_l), C.byref(a), C.byref(b))
    return a.value, b.value


def combine(z_prog_, z_e, sigma_i, sigma_c):
    """Steps 1-5 of section 3.2; returns (v, z, q)."""
    z, q = C.c_double(), C.c_double()
    v = lib().orc_combine(float(z_prog_), float(z_e), float(sigma_i), float(sigma_c),
                          C.byref(z), C.byref(q))
    return v, z.value, q.value


def sample_loss(mu_l, sigma_i, sigma_c, max_l, z_prog_, z_e):
    out = C.c_double()
    st = lib().orc_sample_loss(float(mu_l), float(sigma_i), float(sigma_c), float(max_l),
                               float(z_prog_), float(z_e), C.byref(out))
    if st != 0:
        raise OracleError("beta quantile did not converge")
    return out.value


def sample_batch(mu, sigma_i, sigma_c, max_l, z_prog_, z_e):
    """Vectorised ``sample_loss`` (plain loop in C)."""
    arrs = [np.ascontiguousarray(np.broadcast_to(np.asarray(a, np.float64), np.shape(z_e)))
            for a in (mu, sigma_i, sigma_c, max_l, z_prog_, z_e)]
    out = np.empty(np.shape(z_e), np.float64)
    st = lib().orc_sample_batch(out.size, *[_ptr(a) for a in arrs], _ptr(out))
    if st != 0:
        raise OracleError("beta quantile did not converge")
    return out


def occ_terms(l, occ_r, occ_l):
    return lib().orc_occ_terms(float(l), float(occ_r), float(occ_l))


def agg_terms(s, agg_r, agg_l):
    return lib().orc_agg_terms(float(s), float(agg_r), float(agg_l))


def xelt_terms(x, ret, lim, share):
    return lib().orc_xelt_terms(float(x), float(ret), float(lim), float(share))


def lookup_hash(k, j, r):
    return lib().orc_lookup_hash(int(k), int(j), int(r))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def run(portfolio, yet, seed, su=True, n_threads=None, trial_index=None, rng_mode=0, z_prog=None, z_event=None):
    """Algorithm 1 over every layer; returns dict(ylt, gross, count, hash,
    occ_max) -- occ_max = per (layer, trial) largest occurrence loss net of
    the occurrence terms (line 11), the basis of the OEP (reading G29).
    ``rng_mode``: 0 = reading G2 (z_E per trial, occurrence, XELT); 1 = (A)
    z_E stored per XELT record; 2 = (B) z_E per occurrence shared by XELTs.
    ``z_prog`` [n_programs][n_occurrences] and ``z_event`` [n_records] given
    (rng_mode 3, the paper's data model, P:55 / P:76): the draws are these
    supplied numbers -- z_(Prog,E) of occurrence o of the YET for program p,
    z_(E) of each XELT record -- instead of Philox draws.

    ``portfolio``: dict with catalog_size, elt_off[n_elts+1], rec_event,
    rec_mean, rec_sigma_i, rec_sigma_c, rec_max (any float dtype; converted
    exactly to fp64), optional elt_terms[n_elts,3], layer_prog[n_layers],
    layer_elt_off[n_layers+1], layer_elts, layer_terms[n_layers,4].
    ``yet``: dict with trial_off[n+1] (uint64) and events (uint32), and
    first_trial (global index of trial 0) unless ``trial_index`` is given.
    """
    pf = portfolio
    n_elts = len(pf["elt_off"]) - 1
    n_layers = len(pf["layer_prog"])
    elt_off = np.ascontiguousarray(pf["elt_off"], dtype=np.uint64)
    rec_event = np.ascontiguousarray(pf["rec_event"], dtype=np.uint32)
    f64 = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    rm, rsi, rsc, rmax = (f64(pf["rec_mean"]), f64(pf["rec_sigma_i"]),
                          f64(pf["rec_sigma_c"]), f64(pf["rec_max"]))
    et = pf.get("elt_terms")
    et = None if et is None else f64(et).reshape(-1)
    lprog = np.ascontiguousarray(pf["layer_prog"], dtype=np.uint32)
    loff = np.ascontiguousarray(pf["layer_elt_off"], dtype=np.uint64)
    lelts = np.ascontiguousarray(pf["layer_elts"], dtype=np.uint32)
    lterms = f64(pf["layer_terms"]).reshape(-1)
    toff = np.ascontiguousarray(yet["trial_off"], dtype=np.uint64)
    ev = np.ascontiguousarray(yet["events"], dtype=np.uint32)
    n = len(toff) - 1
    if trial_index is None:
        trial_index = np.arange(n, dtype=np.uint64) + np.uint64(yet.get("first_trial", 0))
    tidx = np.ascontiguousarray(trial_index, dtype=np.uint64)
    ylt = np.zeros((n_layers, n), dtype=np.float64)
    gross = np.zeros((n_layers, n), dtype=np.float64)
    count = np.zeros((n_layers, n), dtype=np.uint32)
    hsh = np.zeros((n_layers, n), dtype=np.uint64)
    occ_max = np.zeros((n_layers, n), dtype=np.float64)
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    zp = ze = None
    if z_prog is not None or z_event is not None:
        assert z_prog is not None and z_event is not None, "supply both z_prog and z_event"
        rng_mode = 3
        zp = f64(z_prog).reshape(-1)
        ze = f64(z_event).reshape(-1)
        assert zp.size % max(ev.size, 1) == 0 and zp.size >= ev.size * (int(lprog.max()) + 1 if lprog.size else 1)
        assert ze.size == rec_event.size
        assert ((zp > 0) & (zp < 1)).all() and ((ze > 0) & (ze < 1)).all(), "z values must lie in (0, 1)"
    st = lib().orc_run(int(pf["catalog_size"]), n_elts, _ptr(elt_off), _ptr(rec_event),
                       _ptr(rm), _ptr(rsi), _ptr(rsc), _ptr(rmax), _ptr(et),
                       n_layers, _ptr(lprog), _ptr(loff), _ptr(lelts), _ptr(lterms),
                       n, _ptr(tidx), _ptr(toff), _ptr(ev),
                       int(seed) & 0xFFFFFFFFFFFFFFFF, 1 if su else 0, int(n_threads),
                       _ptr(ylt), _ptr(gross), _ptr(count), _ptr(hsh), _ptr(occ_max), int(rng_mode),
                       _ptr(zp), _ptr(ze))
    if st == -1:
        raise OracleError("a beta quantile did not converge")
    if st == -2:
        raise OracleError("event id out of range")
    if st == -3:
        raise OracleError("out of memory building the direct-access table")
    return {"ylt": ylt, "gross": gross, "count": count, "hash": hsh, "occ_max": occ_max}
