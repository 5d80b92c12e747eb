"""AGRISK01 storage format (plumbing, no method arithmetic):
bit-exact binary round trips of all four kinds over randomized fixtures,
structured errors with byte offsets, the YLT size rule, CSV round trips, and
a loaded portfolio + YET running the oracle to the same YLT."""
import numpy as np
import pytest

import aragen
import oracle
from paper_1310_2274_b200 import agrisk as AG


def _rand_yet(rng, z=True):
    n = int(rng.integers(0, 30))
    lens = rng.integers(0, 12, n)
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    m = int(off[-1])
    y = {"trial_off": off, "events": rng.integers(0, 2 ** 32, m, dtype=np.uint64).astype(np.uint32),
         "timestamps": rng.standard_normal(m).astype(np.float32), "first_trial": int(rng.integers(0, 10 ** 9))}
    if z:
        y["z_prog"] = rng.uniform(0, 1, (int(rng.integers(1, 4)), m)).astype(np.float32)
    return y


def _rand_xelts(rng):
    n = int(rng.integers(1, 8))
    lens = rng.integers(0, 20, n)
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    R = int(off[-1])
    f = lambda: rng.standard_normal(R).astype(np.float32)  # noqa: E731
    return {"elt_off": off, "rec_event": rng.integers(0, 10 ** 6, R).astype(np.uint32), "rec_mean": f(),
            "rec_sigma_i": f(), "rec_sigma_c": f(), "rec_max": f(),
            "rec_z_event": f() if rng.uniform() < 0.5 else None,
            "elt_terms": rng.standard_normal((n, 3)) if rng.uniform() < 0.5 else None}


def _eq(a, b):
    assert set(a) == set(b), (set(a), set(b))
    for k in a:
        if a[k] is None or b[k] is None:
            assert a[k] is None and b[k] is None, k
        elif isinstance(a[k], np.ndarray):
            assert a[k].dtype == b[k].dtype and a[k].shape == b[k].shape, k
            assert a[k].tobytes() == b[k].tobytes(), k          # bit-exact, NaN payloads included
        else:
            assert a[k] == b[k], k


@pytest.mark.parametrize("seed", range(200))
def test_binary_round_trips_bit_exact(seed):
    rng = np.random.default_rng(seed)
    y = _rand_yet(rng, z=seed % 2 == 0)
    _eq(AG.yet_from_bytes(AG.yet_to_bytes(y)), y)
    x = _rand_xelts(rng)
    _eq(AG.xelts_from_bytes(AG.xelts_to_bytes(x)), x)
    L = int(rng.integers(1, 5))
    S = rng.integers(1, 6, L)
    loff = np.zeros(L + 1, np.uint64)
    np.cumsum(S, out=loff[1:])
    pf = {"catalog_size": int(rng.integers(1, 10 ** 6)), "layer_prog": rng.integers(0, 10, L).astype(np.uint32),
          "layer_elt_off": loff, "layer_elts": rng.integers(0, 100, int(loff[-1])).astype(np.uint32),
          "layer_terms": rng.standard_normal((L, 4))}
    _eq(AG.portfolio_from_bytes(AG.portfolio_to_bytes(pf)), pf)
    ylt = rng.standard_normal((L, int(rng.integers(0, 50))))
    first = int(rng.integers(0, 10 ** 6))
    back = AG.ylt_from_bytes(AG.ylt_to_bytes(ylt, first_trial=first))
    assert back["ylt"].tobytes() == ylt.tobytes() and back["first_trial"] == first


def test_errors_carry_byte_offsets():
    y = _rand_yet(np.random.default_rng(1))
    b = AG.yet_to_bytes(y)
    with pytest.raises(AG.AgriskError) as ei:
        AG.yet_from_bytes(b"XGRISK01" + b[8:])                  # corrupt magic
    assert ei.value.offset == 0
    bad = bytearray(b)
    bad[9] = 7                                                  # format_version
    with pytest.raises(AG.AgriskError) as ei:
        AG.yet_from_bytes(bytes(bad))
    assert ei.value.offset == 9
    with pytest.raises(AG.AgriskError) as ei:
        AG.xelts_from_bytes(b)                                  # wrong kind
    assert ei.value.offset == 8
    with pytest.raises(AG.AgriskError) as ei:
        AG.yet_from_bytes(b[:-3])                               # truncated
    assert AG.HEADER_BYTES <= ei.value.offset < len(b)
    with pytest.raises(AG.AgriskError):
        AG.yet_from_bytes(b + b"\0")                            # trailing bytes
    with pytest.raises(AG.AgriskError) as ei:
        AG.yet_from_bytes(b[:20])
    assert ei.value.offset == 20


def test_ylt_file_size():
    # an 800,000-trial YLT = header + 800,000 x (8-byte id + 8-byte loss)
    b = AG.ylt_to_bytes(np.zeros(800000))
    assert len(b) == AG.HEADER_BYTES + 800000 * 16


@pytest.mark.parametrize("seed", range(20))
def test_csv_round_trips(seed):
    rng = np.random.default_rng(100 + seed)
    y = _rand_yet(rng, z=seed % 2 == 0)
    y["events"] = y["events"] % np.uint32(10 ** 6)
    n = len(y["trial_off"]) - 1
    back = AG.yet_from_csv(AG.yet_to_csv(y), n_trials=n, first_trial=y["first_trial"])
    if "z_prog" in y and not y["events"].size:
        back["z_prog"] = y["z_prog"]                           # (no rows: no z columns to read)
    _eq(back, y)
    ylt = rng.standard_normal((2, 7))
    b2 = AG.ylt_from_csv(AG.ylt_to_csv(ylt, first_trial=5))
    assert b2["ylt"].tobytes() == ylt.tobytes() and b2["first_trial"] == 5


def test_loaded_inputs_run_the_same(tmp_path):
    # cfg1's inputs written and read back as files run the oracle to the same YLT
    cfg = aragen.load_config("cfg1")
    cfg["n_trials"] = 50
    pf, yet = aragen.build_portfolio(cfg), aragen.build_yet(cfg)
    AG.write(tmp_path / "x.agr", AG.KIND_XELT, pf)
    AG.write(tmp_path / "p.agr", AG.KIND_PORTFOLIO, pf)
    AG.write(tmp_path / "y.agr", AG.KIND_YET, yet)
    pf2 = AG.merge_portfolio(AG.read(tmp_path / "x.agr", AG.KIND_XELT), AG.read(tmp_path / "p.agr", AG.KIND_PORTFOLIO))
    yet2 = AG.read(tmp_path / "y.agr", AG.KIND_YET)
    a = oracle.run(pf, yet, seed=3)["ylt"]
    b = oracle.run(pf2, yet2, seed=3)["ylt"]
    assert np.array_equal(a, b)
    AG.write(tmp_path / "ylt.agr", AG.KIND_YLT, a, first_trial=0)
    assert np.array_equal(AG.read(tmp_path / "ylt.agr", AG.KIND_YLT)["ylt"], a)
