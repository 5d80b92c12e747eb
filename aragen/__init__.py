"""Seeded synthetic inputs for ARA (YET, XELTs, portfolio) -- shared by the
tests, ``bench.py`` and ``smoke()``.

This module holds none of the method's arithmetic (no lookup, sampler or
terms); it only produces the three input tables of Algorithm 1
with the shapes of the paper's workloads and the value recipe in DESIGN.md.
Random numbers come from its own Philox4x32-10 copy in ``aragen.c``, keyed by
global trial / record index so any slice can be generated on any rank.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aragen.c")
_LIB = os.path.join(_HERE, "libaragen.so")
CONFIG_DIR = os.path.join(os.path.dirname(_HERE), "configs")

__all__ = ["build_aragen", "load_config", "build_portfolio", "build_yet",
           "yet_for_trials", "trial_lengths", "CONFIG_NAMES"]

CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


def build_aragen(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", tmp,
                               _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        L = C.CDLL(build_aragen())
        vp, u32, u64, i32, d = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
        L.aragen_yet.argtypes = [u64, u32, u64, u64, vp, u32, vp, i32]
        L.aragen_yet.restype = i32
        L.aragen_trial_lengths.argtypes = [u64, u64, u64, u32, u32, vp]
        L.aragen_elt.argtypes = [u64, u32, u32, u32, d, i32, vp, vp, vp, vp, vp]
        L.aragen_elt.restype = i32
        L.aragen_pack_bits.argtypes = [vp, u64, u32, vp, i32]
        L.aragen_pack_bits.restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def load_config(name_or_dict):
    """A config dict (shape, seed, terms).  Names resolve to configs/<name>.json."""
    if isinstance(name_or_dict, dict):
        return dict(name_or_dict)
    with open(os.path.join(CONFIG_DIR, f"{name_or_dict}.json")) as f:
        return json.load(f)


def build_portfolio(cfg):
    """XELT records + one program of ``n_layers`` layers, each covering
    ``elts_per_layer`` distinct XELTs (reading G15), as flat numpy arrays."""
    cfg = load_config(cfg)
    L = _L()
    C_ = int(cfg["catalog"])
    nl, J, R = int(cfg["n_layers"]), int(cfg["elts_per_layer"]), int(cfg["records_per_elt"])
    n_elts = nl * J
    seed = int(cfg["seed"])
    ev = np.empty(n_elts * R, np.uint32)
    mu = np.empty(n_elts * R, np.float32)
    si = np.empty_like(mu); sc = np.empty_like(mu); mx = np.empty_like(mu)
    scale = float(cfg.get("sigma_scale", 1.0))
    integer_mu = int(bool(cfg.get("integer_mu", False)))
    for j in range(n_elts):
        s = slice(j * R, (j + 1) * R)
        st = L.aragen_elt(seed, j, C_, R, scale, integer_mu, _p(ev[s]), _p(mu[s]),
                          _p(si[s]), _p(sc[s]), _p(mx[s]))
        if st != 0:
            raise ValueError("records_per_elt > catalog")
    terms = np.array(cfg["layer_terms"], dtype=np.float64).reshape(nl, 4)
    return {
        "catalog_size": C_,
        "elt_off": np.arange(n_elts + 1, dtype=np.uint64) * np.uint64(R),
        "rec_event": ev, "rec_mean": mu, "rec_sigma_i": si, "rec_sigma_c": sc, "rec_max": mx,
        "elt_terms": None,
        "layer_prog": np.zeros(nl, np.uint32),
        "layer_elt_off": np.arange(nl + 1, dtype=np.uint64) * np.uint64(J),
        "layer_elts": np.arange(n_elts, dtype=np.uint32),
        "layer_terms": terms,
    }


def trial_lengths(cfg, first_trial, n_trials):
    cfg = load_config(cfg)
    out = np.empty(n_trials, np.uint32)
    _L().aragen_trial_lengths(int(cfg["seed"]), int(first_trial), int(n_trials),
                              int(cfg["k_min"]), int(cfg["k_max"]), _p(out))
    return out


def build_yet(cfg, first_trial=0, n_trials=None, n_threads=None, out=None):
    """YET event ids for global trials [first_trial, first_trial+n_trials).

    Fixed ``events_per_trial`` unless the config gives ``k_min``/``k_max``
    (then CSR offsets).  ``out`` may be a preallocated (e.g. pinned) uint32
    array of the right length."""
    cfg = load_config(cfg)
    if n_trials is None:
        n_trials = int(cfg["n_trials"]) - first_trial
    if "k_min" in cfg:
        lens = trial_lengths(cfg, first_trial, n_trials)
        off = np.zeros(n_trials + 1, np.uint64)
        np.cumsum(lens, out=off[1:])
        fixed = 0
    else:
        fixed = int(cfg["events_per_trial"])
        off = None
    total = int(off[-1]) if off is not None else n_trials * fixed
    ev = np.empty(total, np.uint32) if out is None else out
    assert ev.dtype == np.uint32 and ev.size == total and ev.flags.c_contiguous
    st = _L().aragen_yet(int(cfg["seed"]), int(cfg["catalog"]), int(first_trial),
                         int(n_trials), _p(off), fixed, _p(ev), int(n_threads or os.cpu_count() or 1))
    if st != 0:
        raise ValueError("bad YET spec")
    if off is None:
        off = np.arange(n_trials + 1, dtype=np.uint64) * np.uint64(fixed)
    return {"trial_off": off, "events": ev, "first_trial": int(first_trial),
            "fixed_len": fixed}


def yet_for_trials(cfg, trial_indices):
    """Event ids of an arbitrary list of global trials (CSR), for sampled
    parity checks at full size."""
    cfg = load_config(cfg)
    parts = [build_yet(cfg, int(i), 1, n_threads=1) for i in trial_indices]
    off = np.zeros(len(parts) + 1, np.uint64)
    off[1:] = np.cumsum([p["events"].size for p in parts])
    ev = np.concatenate([p["events"] for p in parts]) if parts else np.zeros(0, np.uint32)
    return {"trial_off": off, "events": ev,
            "trial_index": np.asarray(trial_indices, dtype=np.uint64)}


def yet_bits(catalog):
    """Bits per event id of the packed YET storage: ceil(log2(catalog))."""
    return max(1, int(catalog - 1).bit_length())


def pack_yet(events, bits, out=None, n_threads=None):
    """Bit-pack uint32 event ids (storage encoding for the packed upload,
    ara_yet_refill_packed): LSB-first, ceil(n*bits/32) uint32 words."""
    ev = np.ascontiguousarray(events, np.uint32)
    words = (ev.size * bits + 31) // 32
    if out is None:
        out = np.empty(words, np.uint32)
    assert out.dtype == np.uint32 and out.size >= words
    st = _L().aragen_pack_bits(_p(ev), ev.size, int(bits), _p(out), int(n_threads or os.cpu_count() or 1))
    if st != 0:
        raise ValueError("an event id does not fit in %d bits" % bits)
    return out[:words]
