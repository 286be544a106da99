"""The C-ABI library loads and exports every symbol include/rsw.h declares; host-only logic and
argument validation work without a GPU (no compute calls here)."""
import ctypes
import re
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1303_6615_b200 import build
    import paper_1303_6615_b200 as rsw
    build.build()
    return rsw, rsw.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "rsw.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(\w+)\s*\([^;{]*\)\s*;", src)) - {"if", "while"})


def test_exports_every_declared_symbol(lib):
    rsw, L = lib
    names = header_functions()
    assert len(names) >= 17, names
    for name in names:
        assert hasattr(L, name), name
    assert sorted(rsw.EXPORTS) == names


def test_shard_range(lib):
    rsw, _ = lib
    assert rsw.shard_range(4096, 3, 8) == (1536, 2048)
    assert rsw.shard_range(8, 0, 1) == (0, 8)
    with pytest.raises(rsw.RSWError):
        rsw.shard_range(10, 0, 4)  # not divisible


def test_flops_per_unit(lib):
    rsw, _ = lib
    # F_N and F_step values for C1 / C5
    assert rsw.flops_per_unit(64, "nonlinear") == 6964
    assert rsw.flops_per_unit(64, "etdrk4") == 31816
    assert rsw.flops_per_unit(1024, "nonlinear") == 172404
    assert rsw.flops_per_unit(1024, "etdrk4") == 751176
    assert rsw.flops_per_unit(1024, "strang") == 362592
    assert rsw.flops_per_unit(512, "sample") == 85362


def test_validation_before_any_launch(lib):
    rsw, L = lib
    bad = [rsw._Params(0.0, 1.0, 0.0, 64), rsw._Params(1e-2, 1.0, -1.0, 64), rsw._Params(1e-2, 1.0, 0.0, 100),
           rsw._Params(1e-2, 1.0, 0.0, 2048), rsw._Params(float("nan"), 1.0, 0.0, 64)]
    buf = ctypes.c_void_p(1)
    for p in bad:
        rc = L.rsw_fine_propagate(ctypes.byref(p), 0, 0, 0.1, 0.01, 1, buf, buf, None)
        assert rc == rsw.RSW_ERR_CONFIG
        assert L.rsw_last_error()
    good = rsw._Params(1e-2, 1.0, 0.0, 64)
    assert L.rsw_fine_propagate(ctypes.byref(good), 0, 0, 0.1, 0.2, 1, buf, buf, None) == rsw.RSW_ERR_CONFIG
    assert L.rsw_fine_propagate(ctypes.byref(good), 7, 0, 0.1, 0.01, 1, buf, buf, None) == rsw.RSW_ERR_CONFIG
    assert L.rsw_averaged_rhs(ctypes.byref(good), 0.05, 1, 1, buf, ctypes.c_void_p(2), None) == rsw.RSW_ERR_CONFIG
    assert L.rsw_nonlinear(ctypes.byref(good), 1, buf, buf, None) == rsw.RSW_ERR_CONFIG  # aliasing
    cfg = rsw._PararealConfig(0.125, 1e-3, 0.05, 0.0, 32, 8, 9, 0, 0)  # max_iters > n_slices
    r = (ctypes.c_double * 9)()
    it = ctypes.c_int32()
    assert L.parareal_iterate(ctypes.byref(good), ctypes.byref(cfg), buf, buf, r, ctypes.byref(it), None,
                              None) == rsw.RSW_ERR_CONFIG
    assert L.rsw_fine_propagate(ctypes.byref(good), 0, 0, 0.1, 0.01, 0, None, None, None) == rsw.RSW_OK
