"""B200-native hot path of the asymptotic parareal method for 1-D rotating shallow water
(arxiv 1303.6615): a thin ctypes binding over librsw.so (include/rsw.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of librsw.so.  There
is no CPU fallback — if the library is missing or the device is not a GPU, calls raise.

States are torch.float64 CUDA tensors shaped (..., 3, n//2 + 1, 2) (fields v1, v2, h; wavenumbers
k = 0..n/2; re, im).  Work is enqueued on torch's current CUDA stream.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

from . import inputs  # noqa: F401  (seeded generators; no method arithmetic)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSW_LIB") or os.path.join(_HERE, "librsw.so")

RSW_OK, RSW_ERR_CONFIG, RSW_NOT_CONVERGED, RSW_ERR_DIVERGED, RSW_ERR_CUDA, RSW_ERR_NCCL = range(6)
FINE_ETDRK4, FINE_STRANG, FINE_IFRK4 = 0, 1, 2
COARSE_RK4, COARSE_MIDPOINT, COARSE_STRANG = 0, 1, 2
SCHEDULE_AUTO, SCHEDULE_BULK, SCHEDULE_PIPELINED = 0, 1, 2
FLAG_LINEAR_ONLY = 1

# names exported by include/rsw.h (checked by tests/test_capi_load.py)
EXPORTS = [
    "rsw_nonlinear", "rsw_fine_propagate", "rsw_averaged_rhs", "rsw_coarse_propagate",
    "parareal_iterate", "parareal_iterate_ex", "rsw_shard_range", "rsw_nccl_unique_id",
    "rsw_comm_init", "rsw_comm_destroy", "rsw_fp64_peak", "rsw_flops_per_unit", "rsw_last_error",
    "rsw_shutdown", "rsw_check_states", "parareal_resume", "rsw_device_topology",
    "rsw_triad_coefficients",
]


class RSWError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rsw status {status}: {msg}")
        self.status = status


class _Params(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("F", ctypes.c_double), ("mu", ctypes.c_double),
                ("n", ctypes.c_int32)]


class _PararealConfig(ctypes.Structure):
    _fields_ = [("dT", ctypes.c_double), ("dt", ctypes.c_double), ("T0", ctypes.c_double),
                ("tol", ctypes.c_double), ("M", ctypes.c_int32), ("n_slices", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("fine_scheme", ctypes.c_int32),
                ("coarse_scheme", ctypes.c_int32), ("schedule", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("fine_ms", ctypes.c_double), ("comm_ms", ctypes.c_double),
                ("coarse_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("fine_slice_steps", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("pipelined", ctypes.c_int32), ("sweep0_ms", ctypes.c_double), ("lag_ms", ctypes.c_double),
                ("fine_task_ms", ctypes.c_double), ("coarse_groups", ctypes.c_int32),
                ("group_ctas", ctypes.c_int32), ("die_aware", ctypes.c_int32), ("coarse_triad", ctypes.c_int32)]


@dataclasses.dataclass(frozen=True)
class Params:
    eps: float
    F: float
    mu: float
    n: int

    def _c(self) -> _Params:
        return _Params(float(self.eps), float(self.F), float(self.mu), int(self.n))


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load librsw.so (build it first with paper_1303_6615_b200.build.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RSWError(RSW_ERR_CUDA, f"{path} not built; run `python -m paper_1303_6615_b200.build`")
    L = ctypes.CDLL(path)
    vp, dp, i32, u32, dbl = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
    P = ctypes.POINTER(_Params)
    L.rsw_check_states.argtypes = [P, i32, dp, vp]
    L.rsw_nonlinear.argtypes = [P, i32, dp, dp, vp]
    L.rsw_fine_propagate.argtypes = [P, i32, u32, dbl, dbl, i32, dp, dp, vp]
    L.rsw_averaged_rhs.argtypes = [P, dbl, i32, i32, dp, dp, vp]
    L.rsw_coarse_propagate.argtypes = [P, i32, dbl, dbl, i32, i32, dp, dp, vp]
    L.rsw_triad_coefficients.argtypes = [P, dbl, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.parareal_iterate.argtypes = [P, ctypes.POINTER(_PararealConfig), dp, dp,
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32), vp, vp]
    L.parareal_iterate_ex.argtypes = L.parareal_iterate.argtypes + [dp, dp, ctypes.POINTER(_Stats)]
    L.parareal_resume.argtypes = [P, ctypes.POINTER(_PararealConfig), dp, dp, i32, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(i32), vp, vp, dp, dp, ctypes.POINTER(_Stats)]
    L.rsw_shard_range.argtypes = [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.rsw_nccl_unique_id.argtypes = [vp]
    L.rsw_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.rsw_comm_destroy.argtypes = [vp]
    L.rsw_fp64_peak.argtypes = [ctypes.POINTER(ctypes.c_double), vp]
    L.rsw_device_topology.argtypes = [ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.rsw_flops_per_unit.argtypes = [i32, i32]
    L.rsw_flops_per_unit.restype = ctypes.c_double
    L.rsw_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("rsw_flops_per_unit", "rsw_last_error", "rsw_shutdown"):
            getattr(L, name).restype = ctypes.c_int
    L.rsw_shutdown.restype = None
    _lib = L
    return L


def _check(rc: int, ok=(RSW_OK,)) -> int:
    if rc not in ok:
        raise RSWError(rc, load().rsw_last_error().decode(errors="replace"))
    return rc


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _state_arg(t, n: int):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise RSWError(RSW_ERR_CONFIG, "states must be contiguous float64 CUDA tensors")
    if tuple(t.shape[-3:]) != (3, n // 2 + 1, 2):
        raise RSWError(RSW_ERR_CONFIG, f"state shape {tuple(t.shape)} != (..., 3, {n // 2 + 1}, 2)")
    return ctypes.c_void_p(t.data_ptr()), t.numel() // (3 * (n // 2 + 1) * 2)


def check_states(p: Params, u):
    """Layout check on the device (R10: modes k > n/3 zero; R16: Im û_0 zero); raises RSWError
    (RSW_ERR_CONFIG) on a violation.  Synchronises the current stream."""
    a, nb = _state_arg(u, p.n)
    _check(load().rsw_check_states(ctypes.byref(p._c()), nb, a, _stream()))


def device_topology() -> dict:
    """SMs per die of the current device and whether the die-homing probe succeeded."""
    d = (ctypes.c_int32 * 2)()
    ok = ctypes.c_int32(0)
    _check(load().rsw_device_topology(d, ctypes.byref(ok)))
    return dict(die_sms=[d[0], d[1]], probed=bool(ok.value))


def nonlinear(p: Params, u, validate: bool = True):
    """N(u) for a batch of states (paper operator table, sign R1)."""
    import torch
    a, nb = _state_arg(u, p.n)
    if validate:
        check_states(p, u)
    out = torch.empty_like(u)
    _check(load().rsw_nonlinear(ctypes.byref(p._c()), nb, a, ctypes.c_void_p(out.data_ptr()), _stream()))
    return out


def fine_propagate(p: Params, u, dT: float, dt: float, scheme: int = FINE_ETDRK4, flags: int = 0, out=None,
                   validate: bool = True):
    """F: each state advanced by dT with ceil(dT/dt - 1e-9) ETDRK4 / Strang / IF-RK4 steps (R9)."""
    import torch
    a, nb = _state_arg(u, p.n)
    out = torch.empty_like(u) if out is None else out
    _, nbo = _state_arg(out, p.n)
    if nbo != nb or out.device != u.device:
        raise RSWError(RSW_ERR_CONFIG, "out must hold as many states as u, on the same device")
    if validate:
        check_states(p, u)
    _check(load().rsw_fine_propagate(ctypes.byref(p._c()), scheme, flags, dT, dt, nb, a,
                                     ctypes.c_void_p(out.data_ptr()), _stream()))
    return out


def averaged_rhs(p: Params, u, T0: float, M: int, validate: bool = True):
    """N̄ for a batch of states (Alg.1; R4, R5)."""
    import torch
    a, nb = _state_arg(u, p.n)
    if validate:
        check_states(p, u)
    out = torch.empty_like(u)
    _check(load().rsw_averaged_rhs(ctypes.byref(p._c()), T0, M, nb, a, ctypes.c_void_p(out.data_ptr()),
                                   _stream()))
    return out


def triad_coefficients(p: Params, T0: float, M: int):
    """Triad coefficients W' of N̄ (host computation; rsw.h rsw_triad_coefficients): one
    float64 per coefficient in the library's block layout, for the contraction in the rotated frame."""
    import numpy as np
    cnt = ctypes.c_int64(0)
    _check(load().rsw_triad_coefficients(ctypes.byref(p._c()), T0, M, None, ctypes.byref(cnt)))
    out = np.empty(cnt.value, dtype=np.float64)
    _check(load().rsw_triad_coefficients(ctypes.byref(p._c()), T0, M,
                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cnt)))
    return out


def coarse_propagate(p: Params, u, dT: float, T0: float, M: int, scheme: int = COARSE_RK4, validate: bool = True):
    """G for a batch of states (Alg.2; R3, R6)."""
    import torch
    a, nb = _state_arg(u, p.n)
    if validate:
        check_states(p, u)
    out = torch.empty_like(u)
    _check(load().rsw_coarse_propagate(ctypes.byref(p._c()), scheme, dT, T0, M, nb, a,
                                       ctypes.c_void_p(out.data_ptr()), _stream()))
    return out


class Comm:
    """Library-owned NCCL communicator, bootstrapped through torch.distributed."""

    def __init__(self, rank: int, world: int, id_bytes: bytes):
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(id_bytes, 128)
        _check(load().rsw_comm_init(buf, rank, world, ctypes.byref(h)))
        self.handle, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load().rsw_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls) -> "Comm":
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.frombuffer(bytearray(cls.unique_id()), dtype=torch.uint8).clone()
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0)
        return cls(rank, world, bytes(t.cpu().tolist()))

    def close(self):
        if self.handle:
            load().rsw_comm_destroy(self.handle)
            self.handle = None


def shard_range(n_slices: int, rank: int, world: int):
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    _check(load().rsw_shard_range(n_slices, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def parareal_iterate(p: Params, u0, *, dT, dt, T0, M, n_slices, max_iters, tol=0.0,
                     fine_scheme=FINE_ETDRK4, coarse_scheme=COARSE_RK4, comm: Comm | None = None,
                     U=None, want_FG=False, allow_diverged=False, schedule=None):
    """Asymptotic parareal (Eq. HMM parareal iteration P:428-430, Alg.4).
    Returns dict(U, resid, iters, status, stats[, F, G])."""
    import torch
    a, nb = _state_arg(u0, p.n)
    if u0.dim() != 3 or nb != 1:
        raise RSWError(RSW_ERR_CONFIG, f"u0 must be one state of shape (3, {p.n // 2 + 1}, 2)")
    shape = (n_slices + 1, 3, p.n // 2 + 1, 2)
    if U is None:
        U = torch.empty(shape, dtype=torch.float64, device=u0.device)
    else:
        _state_arg(U, p.n)
        if tuple(U.shape) != shape or U.device != u0.device:
            raise RSWError(RSW_ERR_CONFIG, f"U must be a contiguous float64 tensor of shape {shape} on {u0.device}")
    F = torch.empty((n_slices,) + shape[1:], dtype=torch.float64, device=u0.device) if want_FG else None
    G = torch.empty_like(F) if want_FG else None
    resid = (ctypes.c_double * max(max_iters, 1))()
    it = ctypes.c_int32(0)
    st = _Stats()
    if schedule is None:
        schedule = SCHEDULE_AUTO
    cfg = _PararealConfig(dT, dt, T0, tol, M, n_slices, max_iters, fine_scheme, coarse_scheme, schedule)
    rc = load().parareal_iterate_ex(ctypes.byref(p._c()), ctypes.byref(cfg), a, ctypes.c_void_p(U.data_ptr()),
                                    resid, ctypes.byref(it), comm.handle if comm else None, _stream(),
                                    ctypes.c_void_p(F.data_ptr()) if want_FG else None,
                                    ctypes.c_void_p(G.data_ptr()) if want_FG else None, ctypes.byref(st))
    _check(rc, ok=(RSW_OK, RSW_NOT_CONVERGED) + ((RSW_ERR_DIVERGED,) if allow_diverged else ()))
    out = dict(U=U, resid=[resid[i] for i in range(it.value)], iters=it.value, status=rc,
               stats=dict(fine_ms=st.fine_ms, comm_ms=st.comm_ms, coarse_ms=st.coarse_ms,
                          total_ms=st.total_ms, fine_slice_steps=st.fine_slice_steps,
                          kernel_launches=st.kernel_launches, pipelined=bool(st.pipelined),
                          sweep0_ms=st.sweep0_ms, lag_ms=st.lag_ms, fine_task_ms=st.fine_task_ms,
                          coarse_groups=st.coarse_groups, group_ctas=st.group_ctas, die_aware=bool(st.die_aware),
                          coarse_triad=bool(st.coarse_triad)))
    if want_FG:
        out["F"], out["G"] = F, G
    return out


def parareal_resume(p: Params, U, G, k_done: int, *, dT, dt, T0, M, n_slices, max_iters, tol=0.0,
                    fine_scheme=FINE_ETDRK4, coarse_scheme=COARSE_RK4, comm: Comm | None = None, want_FG=False,
                    allow_diverged=False):
    """Continue a parareal iteration from the checkpoint {U = U^k_done, G = G(U^k_done_n)} (the U and G of
    a parareal_iterate(..., want_FG=True) call) up to max_iters (bulk schedule).  U is updated in place.
    Returns dict(U, resid (of the iterations run here), iters (total), status, stats[, F, G])."""
    import torch
    shape = (n_slices + 1, 3, p.n // 2 + 1, 2)
    _state_arg(U, p.n)
    _state_arg(G, p.n)
    if tuple(U.shape) != shape or tuple(G.shape) != (n_slices,) + shape[1:] or U.device != G.device:
        raise RSWError(RSW_ERR_CONFIG, f"U must be {shape} and G {(n_slices,) + shape[1:]} on one device")
    F_o = torch.empty_like(G) if want_FG else None
    G_o = torch.empty_like(G) if want_FG else None
    nres = max(max_iters - k_done, 1)
    resid = (ctypes.c_double * nres)()
    it = ctypes.c_int32(0)
    st = _Stats()
    cfg = _PararealConfig(dT, dt, T0, tol, M, n_slices, max_iters, fine_scheme, coarse_scheme, SCHEDULE_BULK)
    rc = load().parareal_resume(ctypes.byref(p._c()), ctypes.byref(cfg), ctypes.c_void_p(U.data_ptr()),
                                ctypes.c_void_p(G.data_ptr()), int(k_done), resid, ctypes.byref(it),
                                comm.handle if comm else None, _stream(),
                                ctypes.c_void_p(F_o.data_ptr()) if want_FG else None,
                                ctypes.c_void_p(G_o.data_ptr()) if want_FG else None, ctypes.byref(st))
    _check(rc, ok=(RSW_OK, RSW_NOT_CONVERGED) + ((RSW_ERR_DIVERGED,) if allow_diverged else ()))
    out = dict(U=U, resid=[resid[i] for i in range(it.value - k_done)], iters=it.value, status=rc,
               stats=dict(fine_ms=st.fine_ms, comm_ms=st.comm_ms, coarse_ms=st.coarse_ms, total_ms=st.total_ms,
                          fine_slice_steps=st.fine_slice_steps, kernel_launches=st.kernel_launches))
    if want_FG:
        out["F"], out["G"] = F_o, G_o
    return out


def fp64_peak_tflops() -> float:
    v = ctypes.c_double()
    _check(load().rsw_fp64_peak(ctypes.byref(v), _stream()))
    return v.value


def flops_per_unit(n: int, which: str) -> float:
    return load().rsw_flops_per_unit(n, dict(nonlinear=0, etdrk4=1, strang=2, sample=3, triad=4)[which])
