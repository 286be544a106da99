"""ctypes loader for the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this module.  The product package
(``paper_1303_6615_b200``) never imports it, and it never imports the product.

Every function takes/returns numpy arrays in the shared state layout
``float64[batch, 3, n//2 + 1, 2]`` (fields v1, v2, h; wavenumbers k = 0..n/2; re, im).
See ``rsw_oracle.c`` for the paper citations of each computation.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_ERR_CONFIG, ORC_NOT_CONVERGED, ORC_ERR_DIVERGED = 0, 1, 2, 3
FINE_ETDRK4, FINE_STRANG, FINE_IFRK4 = 0, 1, 2
COARSE_RK4, COARSE_MIDPOINT, COARSE_STRANG = 0, 1, 2
FLAG_LINEAR_ONLY = 1


class OrcParams(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("F", ctypes.c_double), ("mu", ctypes.c_double),
                ("n", ctypes.c_int32)]


class OrcPararealConfig(ctypes.Structure):
    _fields_ = [("dT", ctypes.c_double), ("dt", ctypes.c_double), ("T0", ctypes.c_double),
                ("tol", ctypes.c_double), ("M", ctypes.c_int32), ("n_slices", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("fine_scheme", ctypes.c_int32),
                ("coarse_scheme", ctypes.c_int32)]


def build(force: bool = False) -> str:
    """Compile the oracle with the plain C toolchain (gcc -O2 -fopenmp, no fast-math)."""
    src = os.path.join(_HERE, "rsw_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-B" if force else "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        P = ctypes.POINTER(OrcParams)
        L.oracle_fine_propagate.argtypes = [P, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_int32, dp, dp]
        L.oracle_nonlinear.argtypes = [P, ctypes.c_int32, dp, dp]
        L.oracle_averaged_rhs.argtypes = [P, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, dp, dp]
        L.oracle_coarse_propagate.argtypes = [P, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_int32, ctypes.c_int32, dp, dp]
        L.oracle_parareal.argtypes = [P, ctypes.POINTER(OrcPararealConfig), dp, dp, dp,
                                      ctypes.POINTER(ctypes.c_int32), dp, dp]
        L.oracle_dft_forward.argtypes = [ctypes.c_int32, dp, dp]
        L.oracle_dft_inverse.argtypes = [ctypes.c_int32, dp, dp]
        L.oracle_phi.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_double, dp]
        L.oracle_mode_eigen.argtypes = [ctypes.c_double, ctypes.c_double, dp, dp]
        L.oracle_mode_matrix.argtypes = [P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, dp]
        L.oracle_weights.argtypes = [ctypes.c_int32, dp]
        L.oracle_rel_l2.argtypes = [ctypes.c_int32, dp, dp]
        L.oracle_rel_l2.restype = ctypes.c_double
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _params(eps, F, mu, n) -> OrcParams:
    return OrcParams(float(eps), float(F), float(mu), int(n))


def _states(u: np.ndarray, n: int) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    assert u.shape[-3:] == (3, n // 2 + 1, 2), u.shape
    return u


def _check(rc: int, ok=(ORC_OK,)):
    if rc not in ok:
        raise RuntimeError(f"oracle returned status {rc}")
    return rc


def num_threads() -> int:
    return lib().oracle_num_threads()


def nonlinear(u, eps, F, mu, n):
    u = _states(u, n)
    out = np.empty_like(u)
    nb = u.size // (3 * (n // 2 + 1) * 2)
    _check(lib().oracle_nonlinear(ctypes.byref(_params(eps, F, mu, n)), nb, _ptr(u), _ptr(out)))
    return out


def fine_propagate(u, eps, F, mu, n, dT, dt, scheme=FINE_ETDRK4, flags=0):
    u = _states(u, n)
    out = np.empty_like(u)
    nb = u.size // (3 * (n // 2 + 1) * 2)
    _check(lib().oracle_fine_propagate(ctypes.byref(_params(eps, F, mu, n)), scheme, flags,
                                       dT, dt, nb, _ptr(u), _ptr(out)))
    return out


def averaged_rhs(u, eps, F, mu, n, T0, M):
    u = _states(u, n)
    out = np.empty_like(u)
    nb = u.size // (3 * (n // 2 + 1) * 2)
    _check(lib().oracle_averaged_rhs(ctypes.byref(_params(eps, F, mu, n)), T0, M, nb,
                                     _ptr(u), _ptr(out)))
    return out


def coarse_propagate(u, eps, F, mu, n, dT, T0, M, scheme=COARSE_RK4):
    u = _states(u, n)
    out = np.empty_like(u)
    nb = u.size // (3 * (n // 2 + 1) * 2)
    _check(lib().oracle_coarse_propagate(ctypes.byref(_params(eps, F, mu, n)), scheme, dT, T0, M,
                                         nb, _ptr(u), _ptr(out)))
    return out


def parareal(u0, eps, F, mu, n, *, dT, dt, T0, M, n_slices, max_iters, tol=0.0,
             fine_scheme=FINE_ETDRK4, coarse_scheme=COARSE_RK4, want_FG=False):
    """Returns dict(U=[S+1,...], resid=[iters], iters=int, status=int[, F, G])."""
    u0 = _states(u0, n).reshape(3, n // 2 + 1, 2).copy()
    S = n_slices
    U = np.zeros((S + 1, 3, n // 2 + 1, 2))
    resid = np.zeros(max(max_iters, 1))
    it = ctypes.c_int32(0)
    F_out = np.zeros((S, 3, n // 2 + 1, 2)) if want_FG else None
    G_out = np.zeros((S, 3, n // 2 + 1, 2)) if want_FG else None
    cfg = OrcPararealConfig(dT, dt, T0, tol, M, S, max_iters, fine_scheme, coarse_scheme)
    rc = lib().oracle_parareal(ctypes.byref(_params(eps, F, mu, n)), ctypes.byref(cfg), _ptr(u0),
                               _ptr(U), _ptr(resid), ctypes.byref(it),
                               _ptr(F_out) if want_FG else None, _ptr(G_out) if want_FG else None)
    _check(rc, ok=(ORC_OK, ORC_NOT_CONVERGED))
    out = dict(U=U, resid=resid[: it.value].copy(), iters=it.value, status=rc)
    if want_FG:
        out["F"], out["G"] = F_out, G_out
    return out


def dft_forward(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    X = np.empty((n // 2 + 1, 2))
    lib().oracle_dft_forward(n, _ptr(x), _ptr(X))
    return X[:, 0] + 1j * X[:, 1]


def dft_inverse(X, n):
    Xr = np.ascontiguousarray(np.stack([np.real(X), np.imag(X)], -1), dtype=np.float64)
    x = np.empty(n)
    lib().oracle_dft_inverse(n, _ptr(Xr), _ptr(x))
    return x


def phi(j, z):
    out = np.empty(2)
    lib().oracle_phi(j, float(np.real(z)), float(np.imag(z)), _ptr(out))
    return complex(out[0], out[1])


def mode_eigen(k, F):
    lam = np.empty(3)
    V = np.empty((3, 3, 2))
    lib().oracle_mode_eigen(float(k), float(F), _ptr(lam), _ptr(V))
    return lam, V[..., 0] + 1j * V[..., 1]


MATRIX = dict(E=0, E2=1, Q=2, f1=3, f2=4, f3=5, expL=6)


def mode_matrix(which, k, h, eps, F, mu, n=64):
    out = np.empty((3, 3, 2))
    lib().oracle_mode_matrix(ctypes.byref(_params(eps, F, mu, n)), float(k), float(h),
                             MATRIX[which], _ptr(out))
    return out[..., 0] + 1j * out[..., 1]


def weights(M):
    w = np.empty(M)
    lib().oracle_weights(M, _ptr(w))
    return w


def rel_l2(n, a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return lib().oracle_rel_l2(n, _ptr(a), _ptr(b))
