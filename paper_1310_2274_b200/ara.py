"""Thin Python binding of libara's C ABI (include/ara.h).

Argument marshalling only: every step of the method runs in libara's CUDA
kernels.  PyTorch supplies device memory and the current CUDA stream.  There
is no CPU fallback: importing this module without the built library, or
creating a context without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ARA_LIB_PATH") or os.path.join(_HERE, "lib", "libara.so")

OK, EINVAL, ERANGE, EDUP, ENOMEM, ECUDA, ECONVERGE, ENCCL = range(8)
SU = 1
DEBUG_LOOKUP = 2
EXACT = 4
WIDE_PAIRS = 16
MAX_SLOTS = 224
MAX_LAYERS = 64

RECORD_DTYPE = np.dtype([("event_id", "<u4"), ("mean_loss", "<f4"), ("sigma_i", "<f4"),
                         ("sigma_c", "<f4"), ("max_loss", "<f4")])
assert RECORD_DTYPE.itemsize == 20

_NAMES = {OK: "ARA_OK", EINVAL: "ARA_EINVAL", ERANGE: "ARA_ERANGE", EDUP: "ARA_EDUP",
          ENOMEM: "ARA_ENOMEM", ECUDA: "ARA_ECUDA", ECONVERGE: "ARA_ECONVERGE", ENCCL: "ARA_ENCCL"}

# every entry point declared in include/ara.h
EXPORTS = (
    "ara_last_error", "ara_version", "ara_ctx_create", "ara_ctx_destroy", "ara_ctx_synchronize",
    "ara_validate_portfolio", "ara_create_portfolio", "ara_portfolio_destroy", "ara_portfolio_info",
    "ara_load_yet",
    "ara_yet_refill", "ara_yet_refill_packed", "ara_yet_num_trials", "ara_yet_destroy", "ara_run", "ara_run_ep", "ara_last_run_timings", "ara_risk_measures_var", "ara_risk_measures_batch", "ara_exceedance_curve",
    "ara_risk_measures",
    "ara_sample_losses", "ara_draw_uniforms", "ara_normal_quantiles", "ara_beta_quantiles", "ara_prepare",
    "ara_yet_set_z", "ara_portfolio_set_z", "ara_last_run_launches", "ara_risk_measures_async",
)


class AraError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libara.so not built ({LIB_PATH}); run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
    L.ara_last_error.restype = C.c_char_p
    L.ara_version.restype = C.c_int
    L.ara_ctx_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
    L.ara_ctx_destroy.argtypes = [vp]; L.ara_ctx_destroy.restype = None
    L.ara_ctx_synchronize.argtypes = [vp]
    pf_args = [u32, u32, vp, vp, vp, u32, vp, vp, vp, vp]
    L.ara_validate_portfolio.argtypes = pf_args
    L.ara_create_portfolio.argtypes = [vp] + pf_args + [C.POINTER(vp)]
    L.ara_portfolio_destroy.argtypes = [vp]; L.ara_portfolio_destroy.restype = None
    L.ara_portfolio_info.argtypes = [vp, vp, vp, vp]
    L.ara_load_yet.argtypes = [vp, u64, u64, vp, u32, vp, vp, C.POINTER(vp)]
    L.ara_yet_refill.argtypes = [vp, vp, vp]
    L.ara_yet_refill_packed.argtypes = [vp, vp, u32, vp]
    L.ara_yet_num_trials.argtypes = [vp]; L.ara_yet_num_trials.restype = u64
    L.ara_yet_destroy.argtypes = [vp]; L.ara_yet_destroy.restype = None
    L.ara_run.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp]
    L.ara_run_ep.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, vp]
    L.ara_risk_measures.argtypes = [vp, vp, u32, u64, u32, i32, vp, u32, vp, vp]
    L.ara_risk_measures_var.argtypes = [vp, vp, u32, u64, u32, i32, vp, u32, vp, vp, vp]
    L.ara_exceedance_curve.argtypes = [vp, vp, u32, u64, u32, i32, vp]
    L.ara_risk_measures_batch.argtypes = [vp, vp, u32, u64, u32, vp, u32, vp, u32, vp, vp, vp]
    L.ara_risk_measures_async.argtypes = [vp, vp, u32, u64, u32, vp, u32, vp, u32, vp]
    L.ara_last_run_timings.argtypes = [vp, vp, vp, vp]
    L.ara_sample_losses.argtypes = [vp, u64, vp, vp, vp, u32, vp]
    L.ara_draw_uniforms.argtypes = [vp, u64, u64, vp, vp]
    L.ara_normal_quantiles.argtypes = [vp, u64, vp, vp]
    L.ara_beta_quantiles.argtypes = [vp, u64, vp, vp, vp, vp, vp]
    L.ara_prepare.argtypes = [vp, vp, vp, u32]
    L.ara_yet_set_z.argtypes = [vp, vp, u32, vp]
    L.ara_portfolio_set_z.argtypes = [vp, vp, vp]
    L.ara_last_run_launches.argtypes = [vp, vp, vp]
    for n in EXPORTS:            # fail loudly if an entry point is missing
        getattr(L, n)
    return L


lib = _load()


def last_error() -> str:
    return lib.ara_last_error().decode()


def _check(st):
    if st != OK:
        raise AraError(st, last_error())


def _p(a):
    """ctypes pointer for a numpy array, a torch tensor, an int address, or None."""
    if a is None:
        return None
    if isinstance(a, int):
        return C.c_void_p(a)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _current_stream_handle(device):
    import torch
    return torch.cuda.current_stream(device).cuda_stream


# ---------------------------------------------------------------------------
class Context:
    """ara_ctx: a device plus the CUDA stream all work is enqueued on."""

    def __init__(self, device: int = 0, stream=None):
        if stream is None:
            stream = _current_stream_handle(device)
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        self.device = device
        self.stream = stream
        h = C.c_void_p()
        _check(lib.ara_ctx_create(device, C.c_void_p(stream), C.byref(h)))
        self.h = h

    def synchronize(self):
        _check(lib.ara_ctx_synchronize(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib.ara_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _records(pf):
    recs = np.empty(len(pf["rec_event"]), RECORD_DTYPE)
    recs["event_id"] = pf["rec_event"]
    recs["mean_loss"] = pf["rec_mean"]
    recs["sigma_i"] = pf["rec_sigma_i"]
    recs["sigma_c"] = pf["rec_sigma_c"]
    recs["max_loss"] = pf["rec_max"]
    return recs


def _pf_arrays(pf):
    recs = _records(pf)
    eoff = np.ascontiguousarray(pf["elt_off"], np.uint64)
    et = pf.get("elt_terms")
    et = None if et is None else np.ascontiguousarray(np.asarray(et, np.float64).reshape(-1, 3))
    lprog = np.ascontiguousarray(pf["layer_prog"], np.uint32)
    loff = np.ascontiguousarray(pf["layer_elt_off"], np.uint64)
    lelts = np.ascontiguousarray(pf["layer_elts"], np.uint32)
    lt = np.ascontiguousarray(np.asarray(pf["layer_terms"], np.float64).reshape(-1, 4))
    keep = (recs, eoff, et, lprog, loff, lelts, lt)
    args = [int(pf["catalog_size"]), len(eoff) - 1, _p(eoff), _p(recs), _p(et), len(lprog),
            _p(lprog), _p(loff), _p(lelts), _p(lt)]
    return args, keep


def validate_portfolio(pf):
    """ara_validate_portfolio (host only); raises AraError."""
    args, _keep = _pf_arrays(pf)
    _check(lib.ara_validate_portfolio(*args))


class Portfolio:
    """ara_portfolio built from the flat-array portfolio dict (see aragen)."""

    def __init__(self, ctx: Context, pf):
        args, _keep = _pf_arrays(pf)
        h = C.c_void_p()
        _check(lib.ara_create_portfolio(ctx.h, *args, C.byref(h)))
        self.h, self.ctx = h, ctx
        self.n_layers = len(pf["layer_prog"])

    def set_z(self, z_event):
        """ara_portfolio_set_z: the z_(E) of every XELT record, in input record order."""
        z = np.ascontiguousarray(z_event, np.float32).ravel()
        _check(lib.ara_portfolio_set_z(self.ctx.h, self.h, _p(z)))

    def info(self):
        """dict(n_device_records, n_table_less, device_bytes) (ara_portfolio_info)."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.ara_portfolio_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"n_device_records": a.value, "n_table_less": b.value, "device_bytes": c.value}

    def close(self):
        if getattr(self, "h", None):
            lib.ara_portfolio_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Yet:
    """ara_yet: event ids (host numpy / pinned torch, or device torch)."""

    def __init__(self, ctx: Context, events, trial_off=None, fixed_len=0, first_trial=0,
                 n_trials=None, timestamps=None):
        off = None if trial_off is None else np.ascontiguousarray(trial_off, np.uint64)
        if n_trials is None:
            n_trials = len(off) - 1 if off is not None else (len(events) // fixed_len if fixed_len else 0)
        ts = None if timestamps is None else np.ascontiguousarray(timestamps, np.float32)
        h = C.c_void_p()
        _check(lib.ara_load_yet(ctx.h, int(n_trials), int(first_trial), _p(off),
                                int(fixed_len) if off is None else 0, _p(events), _p(ts), C.byref(h)))
        self.h, self.ctx = h, ctx
        self.n_trials = int(n_trials)
        self.first_trial = int(first_trial)

    @classmethod
    def from_dict(cls, ctx, yet, events=None):
        """From aragen.build_yet's dict (fixed length uses the compact form)."""
        ev = yet["events"] if events is None else events
        if yet.get("fixed_len"):
            return cls(ctx, ev, fixed_len=yet["fixed_len"], first_trial=yet.get("first_trial", 0),
                       n_trials=len(yet["trial_off"]) - 1)
        return cls(ctx, ev, trial_off=yet["trial_off"], first_trial=yet.get("first_trial", 0))

    def refill(self, events, ctx: "Context" = None):
        """ara_yet_refill: new event ids of the same shape, copied on ctx's stream
        (default: the context the YET was loaded with)."""
        _check(lib.ara_yet_refill((ctx or self.ctx).h, self.h, _p(events)))

    def set_z(self, z_prog):
        """ara_yet_set_z: the z_(Prog,E) of every occurrence, [n_programs][total events]."""
        z = np.ascontiguousarray(z_prog, np.float32)
        z2 = z.reshape(-1, z.shape[-1]) if z.ndim > 1 else z.reshape(1, -1)
        _check(lib.ara_yet_set_z(self.ctx.h, self.h, z2.shape[0], _p(z2)))

    def refill_packed(self, packed, bits: int, ctx: "Context" = None):
        """ara_yet_refill_packed: new event ids from their bit-packed words
        (aragen.pack_yet), staged and unpacked on the device, on ctx's stream."""
        _check(lib.ara_yet_refill_packed((ctx or self.ctx).h, self.h, int(bits), _p(packed)))

    def close(self):
        if getattr(self, "h", None):
            lib.ara_yet_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


RNG_FLAGS = {"g2": 0, "record": 32, "occurrence": 64, "supplied": 128}   # ARA_RNG_RECORD / _OCCURRENCE / _SUPPLIED


ASYNC = 256


def run(ctx: Context, pf: Portfolio, yet: Yet, seed: int, su: bool = True, debug: bool = False,
        ylt=None, exact: bool = False, wide_pairs: bool = False, rng: str = "g2", async_: bool = False):
    """ara_run; returns the device YLT [n_layers, n_trials] (and count/hash if debug).
    rng: "g2" (z_E per trial, occurrence, XELT), "record" (paper-literal z_E per
    XELT record), "occurrence" (z_E per occurrence shared by the XELTs)."""
    import torch
    dev = torch.device("cuda", ctx.device)
    if ylt is None:
        ylt = torch.empty((pf.n_layers, yet.n_trials), dtype=torch.float32, device=dev)
    cnt = hsh = None
    if debug:
        cnt = torch.zeros((pf.n_layers, yet.n_trials), dtype=torch.int32, device=dev)
        hsh = torch.zeros((pf.n_layers, yet.n_trials), dtype=torch.int64, device=dev)
    flags = (SU if su else 0) | (DEBUG_LOOKUP if debug else 0) | (EXACT if exact else 0) | \
        (WIDE_PAIRS if wide_pairs else 0) | RNG_FLAGS[rng] | (ASYNC if async_ else 0)
    _check(lib.ara_run(ctx.h, pf.h, yet.h, int(seed) & 0xFFFFFFFFFFFFFFFF, flags, _p(ylt), _p(cnt),
                       _p(hsh)))
    return (ylt, cnt, hsh) if debug else ylt


def run_ep(ctx: Context, pf: Portfolio, yet: Yet, seed: int, su: bool = True, debug: bool = False,
           ylt=None, occ_max=None, exact: bool = False, wide_pairs: bool = False, rng: str = "g2"):
    """ara_run_ep; returns (ylt, occ_max) device [n_layers, n_trials] (+ count/hash if debug).
    occ_max = the largest occurrence loss net of occurrence terms per (layer, trial): the OEP basis."""
    import torch
    dev = torch.device("cuda", ctx.device)
    shape = (pf.n_layers, yet.n_trials)
    if ylt is None:
        ylt = torch.empty(shape, dtype=torch.float32, device=dev)
    if occ_max is None:
        occ_max = torch.empty(shape, dtype=torch.float32, device=dev)
    cnt = hsh = None
    if debug:
        cnt = torch.zeros(shape, dtype=torch.int32, device=dev)
        hsh = torch.zeros(shape, dtype=torch.int64, device=dev)
    flags = (SU if su else 0) | (DEBUG_LOOKUP if debug else 0) | (EXACT if exact else 0) | \
        (WIDE_PAIRS if wide_pairs else 0) | RNG_FLAGS[rng]
    _check(lib.ara_run_ep(ctx.h, pf.h, yet.h, int(seed) & 0xFFFFFFFFFFFFFFFF, flags, _p(ylt), _p(occ_max),
                          _p(cnt), _p(hsh)))
    return (ylt, occ_max, cnt, hsh) if debug else (ylt, occ_max)


def prepare(ctx: Context, pf: Portfolio, yet: Yet, su: bool = True, debug: bool = False,
            wide_pairs: bool = False, async_: bool = False):
    """ara_prepare: allocate ara_run's scratch for (pf, yet) up front."""
    flags = (SU if su else 0) | (DEBUG_LOOKUP if debug else 0) | (WIDE_PAIRS if wide_pairs else 0) | \
        (ASYNC if async_ else 0)
    _check(lib.ara_prepare(ctx.h, pf.h, yet.h, flags))


def last_run_timings(ctx: Context):
    """ara_last_run_timings -> dict(compact_ms, sample_ms, redo_ms) of the last ara_run."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(lib.ara_last_run_timings(ctx.h, C.byref(a), C.byref(b), C.byref(c)))
    n, nb = C.c_uint32(), C.c_uint32()
    _check(lib.ara_last_run_launches(ctx.h, C.byref(n), C.byref(nb)))
    return {"compact_ms": a.value, "sample_ms": b.value, "redo_ms": c.value, "launches": n.value,
            "batches": nb.value}


def risk_measures(ctx: Context, ylt, n_layers: int, n_total: int, layer: int = 0,
                  rps=(100, 250, 500), n_shards: int = 1):
    """ara_risk_measures; returns (pml[n_rp], tvar[n_rp]) as numpy fp64."""
    r = np.ascontiguousarray(rps, np.float64)
    pml = np.empty(len(r)); tvar = np.empty(len(r))
    _check(lib.ara_risk_measures(ctx.h, _p(ylt), int(n_layers), int(n_total), int(n_shards),
                                 int(layer), _p(r), len(r), _p(pml), _p(tvar)))
    return pml, tvar


def risk_measures_var(ctx: Context, ylt, n_layers: int, n_total: int, layer: int = 0,
                      rps=(100, 250, 500), n_shards: int = 1):
    """ara_risk_measures_var; returns (pml[n_rp], tvar[n_rp], var[n_rp]) as numpy fp64."""
    r = np.ascontiguousarray(rps, np.float64)
    pml = np.empty(len(r)); tvar = np.empty(len(r)); var = np.empty(len(r))
    _check(lib.ara_risk_measures_var(ctx.h, _p(ylt), int(n_layers), int(n_total), int(n_shards),
                                     int(layer), _p(r), len(r), _p(pml), _p(tvar), _p(var)))
    return pml, tvar, var


def risk_measures_batch(ctx: Context, ylt, n_layers: int, n_total: int, layers, rps=(100, 250, 500),
                        n_shards: int = 1):
    """ara_risk_measures_batch; returns (pml, tvar, var), numpy fp64 [len(layers)][n_rp]."""
    r = np.ascontiguousarray(rps, np.float64)
    ls = np.ascontiguousarray(layers, np.int32)
    pml = np.empty((len(ls), len(r))); tvar = np.empty_like(pml); var = np.empty_like(pml)
    _check(lib.ara_risk_measures_batch(ctx.h, _p(ylt), int(n_layers), int(n_total), int(n_shards), _p(ls),
                                       len(ls), _p(r), len(r), _p(pml), _p(tvar), _p(var)))
    return pml, tvar, var


def risk_measures_async(ctx: Context, ylt, n_layers: int, n_total: int, layers, rps=(100, 250, 500),
                        n_shards: int = 1, out=None):
    """ara_risk_measures_async: the measures of every listed table enqueued on the
    context stream, no synchronisation; returns the device fp64 tensor
    [len(layers)][n_rp][3] of (PML, TVaR, VaR) they will be written to."""
    import torch
    r = np.ascontiguousarray(rps, np.float64)
    ls = np.ascontiguousarray(layers, np.int32)
    if out is None:
        out = torch.empty((len(ls), len(r), 3), dtype=torch.float64, device=ylt.device)
    elif not (isinstance(out, torch.Tensor) and out.dtype == torch.float64 and out.is_contiguous()
              and out.numel() >= 3 * len(ls) * len(r)):
        raise AraError(EINVAL, "out must be a contiguous float64 tensor of >= 3 * len(layers) * len(rps) elements")
    _check(lib.ara_risk_measures_async(ctx.h, _p(ylt), int(n_layers), int(n_total), int(n_shards), _p(ls),
                                       len(ls), _p(r), len(r), _p(out)))
    return out


def exceedance_curve(ctx: Context, ylt, n_layers: int, n_total: int, layer: int = 0, n_shards: int = 1,
                     out=None):
    """ara_exceedance_curve: device fp32 [n_total], the losses sorted descending
    (rank i has exceedance probability i/(N+1))."""
    import torch
    if out is None:
        out = torch.empty(int(n_total), dtype=torch.float32, device=ylt.device)
    _check(lib.ara_exceedance_curve(ctx.h, _p(ylt), int(n_layers), int(n_total), int(n_shards), int(layer),
                                    _p(out)))
    return out


def sample_losses(ctx: Context, records, z_prog, z_event, exact: bool = False):
    """ara_sample_losses: device loss draws for (record, z_P, z_E) triples."""
    recs = np.ascontiguousarray(records, RECORD_DTYPE)
    zp = np.ascontiguousarray(z_prog, np.float32)
    ze = np.ascontiguousarray(z_event, np.float32)
    out = np.empty(len(recs), np.float32)
    _check(lib.ara_sample_losses(ctx.h, len(recs), _p(recs), _p(zp), _p(ze), EXACT if exact else 0,
                                 _p(out)))
    return out


def draw_uniforms(ctx: Context, seed: int, ctr):
    """ara_draw_uniforms: U(lane0(Philox(seed, ctr))) for ctr rows (i, k, id, tag)."""
    c = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    out = np.empty(len(c), np.float32)
    _check(lib.ara_draw_uniforms(ctx.h, int(seed) & 0xFFFFFFFFFFFFFFFF, len(c), _p(c), _p(out)))
    return out


def normal_quantiles(ctx: Context, bits):
    """ara_normal_quantiles: Phi^-1(U(x)) of 32-bit Philox words x, as the kernels take it."""
    b = np.ascontiguousarray(bits, np.uint32).ravel()
    out = np.empty(len(b), np.float32)
    _check(lib.ara_normal_quantiles(ctx.h, len(b), _p(b), _p(out)))
    return out


def beta_quantiles(ctx: Context, alpha, beta, v):
    """ara_beta_quantiles: (x, 1 - x) with I_x(alpha, beta) = Phi(v), by the
    device's fp64 solve (row a6 on its own)."""
    a = np.ascontiguousarray(alpha, np.float64).ravel()
    b = np.ascontiguousarray(np.broadcast_to(beta, a.shape), np.float64).ravel()
    w = np.ascontiguousarray(np.broadcast_to(v, a.shape), np.float64).ravel()
    x = np.empty(len(a), np.float64)
    y = np.empty(len(a), np.float64)
    _check(lib.ara_beta_quantiles(ctx.h, len(a), _p(a), _p(b), _p(w), _p(x), _p(y)))
    return x, y
