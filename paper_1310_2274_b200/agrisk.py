"""AGRISK01: a little-endian binary (and CSV) file format for the inputs and
outputs of the hot path -- YET, XELT set, portfolio, YLT -- so that a user's
data can be stored and loaded into the dicts ``ara.Portfolio`` / ``ara.Yet``
take.  Storage plumbing only ("invented -- artifact
plumbing"): no step of the method is computed here.

The paper's data model is carried in full, including the draws it
stores with the inputs (reading G30): z_(Prog,E) per YET occurrence and
program and z_(E) per XELT record, both optional.

Binary layout (all little-endian, fixed width, no compression):

    header   magic "AGRISK01" (8 B) | kind u8 | format_version u16 | counts u64[4]
    YET       (kind 1) counts: n_trials, n_occurrences, n_programs (z_prog rows), first_trial
              trial_off u64[n+1] | event_id u32[m] | timestamp f32[m] | z_prog f32[n_programs][m]
    XELT set  (kind 2) counts: n_elts, n_records, has_z (0/1), has_terms (0/1)
              elt_off u64[n_elts+1] | event_id u32[r] | mean, sigma_i, sigma_c, max f32[r] each
              | z_e f32[r] (has_z) | terms f64[n_elts][3] (retention, limit, share; has_terms)
    PORTFOLIO (kind 3) counts: n_layers, n_slots, catalog_size, 0
              layer_prog u32[L] | layer_elt_off u64[L+1] | layer_elts u32[slots] | terms f64[L][4]
    YLT       (kind 4) counts: n_layers, n_trials, first_trial, 0
              rows (trial_id u64, loss f64) [n_layers][n_trials]

Reading checks the magic, kind and version and every size; a violation
raises ``AgriskError`` carrying the byte offset where it was detected.
Binary round trips are bit-exact; CSV round trips render floats with 17
significant digits (bit-exact for f64, and for f32 read back as f32).
"""
from __future__ import annotations

import csv
import io
import struct

import numpy as np

MAGIC = b"AGRISK01"
VERSION = 1
KIND_YET, KIND_XELT, KIND_PORTFOLIO, KIND_YLT = 1, 2, 3, 4
_HDR = struct.Struct("<8sBH4Q")          # 8 + 1 + 2 + 32 = 43 bytes
HEADER_BYTES = _HDR.size


class AgriskError(ValueError):
    """A structured load error: message and the byte offset where it was detected."""

    def __init__(self, msg, offset):
        super().__init__(f"{msg} (byte offset {offset})")
        self.offset = offset


# ---------------------------------------------------------------------------
class _Reader:
    def __init__(self, data: bytes):
        self.b = data
        self.o = 0

    def header(self, kind):
        if len(self.b) < HEADER_BYTES:
            raise AgriskError("truncated header", len(self.b))
        magic, k, ver, *counts = _HDR.unpack_from(self.b, 0)
        if magic != MAGIC:
            raise AgriskError(f"bad magic {magic!r}", 0)
        if ver != VERSION:
            raise AgriskError(f"format_version {ver} != {VERSION}", 9)
        if k != kind:
            raise AgriskError(f"kind {k} != {kind}", 8)
        self.o = HEADER_BYTES
        return counts

    def array(self, dtype, n):
        dt = np.dtype(dtype).newbyteorder("<")
        nb = dt.itemsize * int(n)
        if self.o + nb > len(self.b):
            raise AgriskError(f"truncated stream: need {nb} bytes of {dt}", self.o)
        a = np.frombuffer(self.b, dt, int(n), self.o).astype(dt.newbyteorder("="))
        self.o += nb
        return a

    def end(self):
        if self.o != len(self.b):
            raise AgriskError(f"{len(self.b) - self.o} trailing bytes", self.o)


def _header(kind, *counts):
    c = list(counts) + [0] * (4 - len(counts))
    return _HDR.pack(MAGIC, kind, VERSION, *[int(x) for x in c])


def _le(a, dtype):
    return np.ascontiguousarray(a, np.dtype(dtype).newbyteorder("<")).tobytes()


def _check_offsets(off, n_items, total, where, what):
    if off[0] != 0 or np.any(np.diff(off.astype(np.int64)) < 0) or off[-1] != total:
        raise AgriskError(f"{what} offsets are not monotone from 0 to {total}", where)


# ---- YET -------------------------------------------------------------------
def yet_to_bytes(yet) -> bytes:
    off = np.asarray(yet["trial_off"], np.uint64)
    ev = np.asarray(yet["events"], np.uint32)
    ts = np.asarray(yet.get("timestamps", np.zeros(ev.size, np.float32)), np.float32)
    zp = yet.get("z_prog")
    zp = np.zeros((0, ev.size), np.float32) if zp is None else np.asarray(zp, np.float32)
    if zp.ndim == 1:
        zp = zp.reshape(1, -1)
    return (_header(KIND_YET, off.size - 1, ev.size, zp.shape[0], yet.get("first_trial", 0)) +
            _le(off, "u8") + _le(ev, "u4") + _le(ts, "f4") + _le(zp, "f4"))


def yet_from_bytes(data: bytes):
    r = _Reader(data)
    n, m, n_prog, first = r.header(KIND_YET)
    o0 = r.o
    off = r.array("u8", n + 1)
    _check_offsets(off, n, m, o0, "trial")
    ev = r.array("u4", m)
    ts = r.array("f4", m)
    zp = r.array("f4", n_prog * m).reshape(n_prog, m)
    r.end()
    out = {"trial_off": off, "events": ev, "timestamps": ts, "first_trial": int(first)}
    if n_prog:
        out["z_prog"] = zp
    return out


# ---- XELT set ----------------------------------------------------------------
_REC = ("rec_event", "rec_mean", "rec_sigma_i", "rec_sigma_c", "rec_max")


def xelts_to_bytes(pf) -> bytes:
    off = np.asarray(pf["elt_off"], np.uint64)
    R = int(off[-1])
    ze = pf.get("rec_z_event")
    et = pf.get("elt_terms")
    out = [_header(KIND_XELT, off.size - 1, R, ze is not None, et is not None), _le(off, "u8"),
           _le(pf["rec_event"], "u4")]
    out += [_le(pf[k], "f4") for k in _REC[1:]]
    if ze is not None:
        out.append(_le(ze, "f4"))
    if et is not None:
        out.append(_le(np.asarray(et, np.float64).reshape(-1, 3), "f8"))
    return b"".join(out)


def xelts_from_bytes(data: bytes):
    r = _Reader(data)
    n_elts, R, has_z, has_terms = r.header(KIND_XELT)
    o0 = r.o
    off = r.array("u8", n_elts + 1)
    _check_offsets(off, n_elts, R, o0, "XELT record")
    out = {"elt_off": off, "rec_event": r.array("u4", R)}
    for k in _REC[1:]:
        out[k] = r.array("f4", R)
    out["rec_z_event"] = r.array("f4", R) if has_z else None
    out["elt_terms"] = r.array("f8", 3 * n_elts).reshape(n_elts, 3) if has_terms else None
    r.end()
    return out


# ---- portfolio ---------------------------------------------------------------
def portfolio_to_bytes(pf) -> bytes:
    lp = np.asarray(pf["layer_prog"], np.uint32)
    loff = np.asarray(pf["layer_elt_off"], np.uint64)
    return (_header(KIND_PORTFOLIO, lp.size, loff[-1], pf["catalog_size"]) + _le(lp, "u4") + _le(loff, "u8") +
            _le(pf["layer_elts"], "u4") + _le(np.asarray(pf["layer_terms"], np.float64).reshape(-1, 4), "f8"))


def portfolio_from_bytes(data: bytes):
    r = _Reader(data)
    L, S, C, _ = r.header(KIND_PORTFOLIO)
    lp = r.array("u4", L)
    o0 = r.o
    loff = r.array("u8", L + 1)
    _check_offsets(loff, L, S, o0, "layer")
    out = {"catalog_size": int(C), "layer_prog": lp, "layer_elt_off": loff, "layer_elts": r.array("u4", S),
           "layer_terms": r.array("f8", 4 * L).reshape(L, 4)}
    r.end()
    return out


# ---- YLT -----------------------------------------------------------------------
_ROW = np.dtype([("trial", "<u8"), ("loss", "<f8")])


def ylt_to_bytes(ylt, first_trial=0) -> bytes:
    y = np.atleast_2d(np.asarray(ylt, np.float64))
    L, N = y.shape
    rows = np.empty((L, N), _ROW)
    rows["trial"] = np.arange(first_trial, first_trial + N, dtype=np.uint64)[None, :]
    rows["loss"] = y
    return _header(KIND_YLT, L, N, first_trial) + rows.tobytes()


def ylt_from_bytes(data: bytes):
    r = _Reader(data)
    L, N, first, _ = r.header(KIND_YLT)
    if r.o + _ROW.itemsize * L * N > len(data):
        raise AgriskError("truncated stream: YLT rows", r.o)
    rows = np.frombuffer(data, _ROW, L * N, r.o).reshape(L, N)
    r.o += _ROW.itemsize * L * N
    r.end()
    if L * N and not np.array_equal(rows["trial"], np.broadcast_to(np.arange(first, first + N, dtype=np.uint64), (L, N))):
        raise AgriskError("YLT trial ids are not first_trial .. first_trial + N - 1", HEADER_BYTES)
    return {"ylt": rows["loss"].astype(np.float64), "first_trial": int(first)}


# ---- files -----------------------------------------------------------------------
def write(path, kind, obj, **kw):
    enc = {KIND_YET: yet_to_bytes, KIND_XELT: xelts_to_bytes, KIND_PORTFOLIO: portfolio_to_bytes,
           KIND_YLT: ylt_to_bytes}[kind]
    with open(path, "wb") as f:
        f.write(enc(obj, **kw))


def read(path, kind):
    dec = {KIND_YET: yet_from_bytes, KIND_XELT: xelts_from_bytes, KIND_PORTFOLIO: portfolio_from_bytes,
           KIND_YLT: ylt_from_bytes}[kind]
    with open(path, "rb") as f:
        return dec(f.read())


def merge_portfolio(xelts, portfolio):
    """The flat portfolio dict ``ara.Portfolio`` takes, from a loaded XELT set and portfolio."""
    out = dict(xelts)
    out.update(portfolio)
    return out


# ---- CSV (SPEC S:478-479 schemas; floats with 17 significant digits) -----------
def _g(x):
    return repr(float(x)) if np.isfinite(x) else ("inf" if x > 0 else "-inf" if x < 0 else "nan")


def yet_to_csv(yet) -> str:
    s = io.StringIO()
    w = csv.writer(s, lineterminator="\n")
    zp = yet.get("z_prog")
    zp2 = None if zp is None else np.asarray(zp, np.float32)
    if zp2 is not None and zp2.ndim == 1:
        zp2 = zp2.reshape(1, -1)
    n_prog = 0 if zp2 is None else zp2.shape[0]
    w.writerow(["trial_id", "event_id", "timestamp"] + [f"z_prog_e_{p}" for p in range(n_prog)])
    off = np.asarray(yet["trial_off"], np.uint64)
    ts = yet.get("timestamps", np.zeros(len(yet["events"]), np.float32))
    first = int(yet.get("first_trial", 0))
    for t in range(off.size - 1):
        for o in range(int(off[t]), int(off[t + 1])):
            w.writerow([first + t, int(yet["events"][o]), _g(ts[o])] +
                       ([_g(zp2[p, o]) for p in range(n_prog)] if n_prog else []))
    return s.getvalue()


def yet_from_csv(text: str, n_trials=None, first_trial=None):
    """(Trials without occurrences have no rows: pass first_trial / n_trials
    to keep leading / trailing empty trials.)"""
    rows = list(csv.reader(io.StringIO(text)))
    hdr, rows = rows[0], rows[1:]
    n_prog = len(hdr) - 3
    tid = np.array([int(r[0]) for r in rows], np.int64)
    first = int(first_trial if first_trial is not None else (tid[0] if tid.size else 0))
    n = int(n_trials if n_trials is not None else (tid[-1] - first + 1 if tid.size else 0))
    counts = np.bincount(tid - first, minlength=n) if tid.size else np.zeros(n, np.int64)
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(counts, out=off[1:])
    out = {"trial_off": off, "events": np.array([int(r[1]) for r in rows], np.uint32),
           "timestamps": np.array([float(r[2]) for r in rows], np.float32), "first_trial": first}
    if n_prog:
        out["z_prog"] = np.array([[float(r[3 + p]) for r in rows] for p in range(n_prog)], np.float32)
    return out


def ylt_to_csv(ylt, first_trial=0) -> str:
    y = np.atleast_2d(np.asarray(ylt, np.float64))
    lines = ["layer,trial_id,loss"]
    for l in range(y.shape[0]):
        lines += [f"{l},{first_trial + t},{_g(y[l, t])}" for t in range(y.shape[1])]
    return "\n".join(lines) + "\n"


def ylt_from_csv(text: str):
    rows = list(csv.reader(io.StringIO(text)))[1:]
    L = 1 + max((int(r[0]) for r in rows), default=-1)
    first = min((int(r[1]) for r in rows), default=0)
    N = len(rows) // max(L, 1)
    y = np.zeros((L, N))
    for r in rows:
        y[int(r[0]), int(r[1]) - first] = float(r[2])
    return {"ylt": y, "first_trial": first}
