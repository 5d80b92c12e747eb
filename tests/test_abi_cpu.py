"""CPU checks of the C-ABI library: it loads, exports every entry point
include/ara.h declares, its host-side validation (ara_validate_portfolio)
rejects what S:126-177 says is invalid, and without a GPU it fails loudly
(no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import aragen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ara():
    from paper_1310_2274_b200 import build
    build.build()
    from paper_1310_2274_b200 import ara as A
    return A


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ara.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ara_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(ara):
    import ctypes
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(ara.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ara.EXPORTS)
    assert ara.lib.ara_version() >= 100


def test_library_is_sm100a(ara):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", ara.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(ara):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import ctypes
    h = ctypes.c_void_p()
    st = ara.lib.ara_ctx_create(0, None, ctypes.byref(h))
    assert st == ara.ECUDA
    assert "no CUDA device" in ara.last_error()


def base_pf():
    cfg = aragen.load_config("cfg1")
    cfg.update(n_layers=2, elts_per_layer=2, records_per_elt=50, catalog=200,
               layer_terms=[[1e5, 5e6, 1e6, 1e8], [2e5, 5e6, 1e6, 1e8]])
    return aragen.build_portfolio(cfg)


def test_validate_ok(ara):
    ara.validate_portfolio(base_pf())


@pytest.mark.parametrize("mutate,code,needle", [
    (lambda p: p["rec_event"].__setitem__(3, 200), "ERANGE", "catalog_size"),
    (lambda p: p["rec_event"].__setitem__(4, p["rec_event"][3]), "EDUP", "duplicate event"),
    (lambda p: p["rec_mean"].__setitem__(5, p["rec_max"][5] * 2), "EINVAL", "mean <= max"),
    (lambda p: p["rec_sigma_i"].__setitem__(5, -1.0), "EINVAL", "sigmas >= 0"),
    (lambda p: p["rec_max"].__setitem__(5, 0.0), "EINVAL", "max > 0"),
    (lambda p: p["rec_mean"].__setitem__(5, np.nan), "EINVAL", "finite"),
    (lambda p: p["layer_elts"].__setitem__(1, 0), "EDUP", "duplicate XELT"),
    (lambda p: p["layer_elts"].__setitem__(1, 9), "ERANGE", "n_elts"),
    (lambda p: p["layer_terms"].__setitem__((0, 1), 0.0), "EINVAL", "limits > 0"),
    (lambda p: p["layer_terms"].__setitem__((1, 2), -1.0), "EINVAL", "retentions >= 0"),
    (lambda p: p.__setitem__("layer_elt_off", np.array([0, 0, 4], np.uint64)), "EINVAL", "covers no XELT"),
    (lambda p: p.__setitem__("catalog_size", 0), "EINVAL", "catalog_size"),
    (lambda p: p.__setitem__("elt_terms", np.array([[0, 1e5, 1.5]] * 4)), "EINVAL", "share"),
    (lambda p: p["layer_prog"].__setitem__(1, 256), "EINVAL", "program 256"),
])
def test_validate_rejects(ara, mutate, code, needle):
    pf = base_pf()
    mutate(pf)
    with pytest.raises(ara.AraError) as ei:
        ara.validate_portfolio(pf)
    assert ei.value.code == getattr(ara, code)
    assert needle in str(ei.value)


def test_validate_limits(ara):
    pf = base_pf()
    n = 4097                                  # > ARA_MAX_PORTFOLIO_LAYERS
    pf2 = dict(pf)
    pf2["layer_prog"] = np.zeros(n, np.uint32)
    pf2["layer_elt_off"] = np.arange(n + 1, dtype=np.uint64)
    pf2["layer_elts"] = np.zeros(n, np.uint32)
    pf2["layer_terms"] = np.tile([1.0, 1e6, 0.0, 1e9], (n, 1))
    with pytest.raises(ara.AraError, match="n_layers"):
        ara.validate_portfolio(pf2)
    ok = dict(pf)
    ok["elt_terms"] = np.array([[0.0, np.inf, 1.0]] * 4)
    ara.validate_portfolio(ok)
    ok["layer_terms"] = np.array([[0.0, np.inf, 0.0, np.inf]] * 2)
    ara.validate_portfolio(ok)
    # 65 layers (more than one kernel group) are valid; a layer over > 224 XELTs is not
    pf3 = dict(pf)
    pf3["layer_prog"] = np.zeros(65, np.uint32)
    pf3["layer_elt_off"] = np.arange(66, dtype=np.uint64)
    pf3["layer_elts"] = np.zeros(65, np.uint32)
    pf3["layer_terms"] = np.tile([1.0, 1e6, 0.0, 1e9], (65, 1))
    ara.validate_portfolio(pf3)
