"""Seeded synthetic inputs and workload configurations.

This module holds NO arithmetic of the method: it only draws initial states with numpy's PCG64
and lists the BASELINE.json workload parameters.  Both the CUDA path (through the tests and
bench.py) and the CPU oracle consume exactly these float64 arrays, bit-identically.

State layout: float64[..., 3, n//2 + 1, 2] — fields (v1, v2, h), wavenumbers k = 0..n/2, (re, im),
with the normalised forward transform û_k = (1/n) Σ_j u_j e^{-ikx_j}, x_j = 2πj/n.  Modes with
k > n//3 (2/3 rule) and Im(û_0) are zero.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    n: int                  # grid points = FFT length
    eps: float
    F: float
    mu: float
    T: float
    n_slices: int
    dt: float               # fine step (dt_eff = dT / ceil(dT/dt - 1e-9), R9)
    T0: float               # averaging window, physical units (R4)
    M: int                  # quadrature points (M-1 effective samples, R5)
    max_iters: int
    tol: float = 0.0        # 0: run exactly max_iters
    fine_scheme: int = 0    # 0 ETDRK4, 1 Strang
    coarse_scheme: int = 0  # 0 RK4, 1 midpoint
    n_states: int = 0       # C4 only: batch of independent states

    @property
    def dT(self) -> float:
        return self.T / self.n_slices

    @property
    def K(self) -> int:
        return self.n // 3

    @property
    def m_fine(self) -> int:
        return int(math.ceil(self.dT / self.dt - 1e-9))

    @property
    def dt_eff(self) -> float:
        return self.dT / self.m_fine

    @property
    def state_shape(self):
        return (3, self.n // 2 + 1, 2)

    def params(self):
        return dict(eps=self.eps, F=self.F, mu=self.mu, n=self.n)


# BASELINE.json configs[0..4].
C1 = Workload("C1", n=64, eps=1e-2, F=1.0, mu=1e-4, T=1.0, n_slices=8, dt=1e-3, T0=0.05, M=32,
              max_iters=4)
C2 = Workload("C2", n=128, eps=1e-2, F=1.0, mu=1e-4, T=8.0, n_slices=64, dt=5e-4, T0=0.05, M=64,
              max_iters=64, tol=1e-6)
C3 = Workload("C3", n=256, eps=1e-3, F=1.0, mu=1e-5, T=16.0, n_slices=512, dt=1e-4, T0=0.01,
              M=128, max_iters=5)
C4 = Workload("C4", n=512, eps=1e-3, F=1.0, mu=0.0, T=1.0, n_slices=1, dt=1.0, T0=0.01, M=256,
              max_iters=0, n_states=4096)
C5 = Workload("C5", n=1024, eps=1e-4, F=1.0, mu=1e-6, T=32.0, n_slices=4096, dt=2e-5, T0=0.002,
              M=256, max_iters=6)
WORKLOADS = {w.name: w for w in (C1, C2, C3, C4, C5)}


def _gaussian_hat(n: int) -> np.ndarray:
    """Half spectrum of g(x) = exp(-4(x-π)^2) on x_j = 2πj/n, masked to k <= n//3."""
    x = 2.0 * np.pi * np.arange(n) / n
    g = np.exp(-4.0 * (x - np.pi) ** 2)
    gh = np.fft.rfft(g) / n
    gh[n // 3 + 1:] = 0.0
    gh[0] = gh[0].real
    return gh


def _pack(c: np.ndarray) -> np.ndarray:
    out = np.zeros(c.shape + (2,))
    out[..., 0] = c.real
    out[..., 1] = c.imag
    return out


def initial_state(w: Workload, seed: int = 0) -> np.ndarray:
    """The configuration's initial state(s), SURVEY.md §8(d) draw layout."""
    n, nh = w.n, w.n // 2 + 1
    rng = np.random.default_rng(seed)
    if w.name in ("C1", "C2"):
        z = rng.standard_normal((9, 2))
        c = np.zeros((3, nh), complex)
        c[2] = _gaussian_hat(n)
        c[2, 1:9] += 1e-3 * (z[1:9, 0] + 1j * z[1:9, 1])
        c[2, 0] += 1e-3 * z[0, 0]
        return _pack(c)
    if w.name in ("C3", "C5"):
        kmax = 32 if w.name == "C3" else 64
        z = rng.standard_normal((3, kmax + 1, 2))
        c = np.zeros((3, nh), complex)
        k = np.arange(1, kmax + 1)
        for f in range(3):
            c[f, 1:kmax + 1] = (1.0 + k) ** -3 * (z[f, 1:, 0] + 1j * z[f, 1:, 1])
        c[2, 0] = z[2, 0, 0]
        c[2] += _gaussian_hat(n)
        return _pack(c)
    if w.name == "C4":
        return random_states(n, w.n_states, seed=seed, kmax=w.K, zero_mean_uv=True)
    raise KeyError(w.name)


def paper_initial_state(n: int) -> np.ndarray:
    """The paper's initial condition (Eq. initial condition 1-1): v1 = v2 = 0,
    h = c1 (e^{-4(x-π/2)^2} sin(3(x-π/2)) + e^{-2(x-π)^2} sin(8(x-π))) + c0 with c0, c1 chosen so that
    ∫h = 0 and max|h| = 1 (on the grid; P:1151 writes "c1 and c2", read as c1, c0 — R17)."""
    x = 2.0 * np.pi * np.arange(n) / n
    g = (np.exp(-4.0 * (x - np.pi / 2) ** 2) * np.sin(3.0 * (x - np.pi / 2))
         + np.exp(-2.0 * (x - np.pi) ** 2) * np.sin(8.0 * (x - np.pi)))
    g = g - g.mean()
    h = g / np.abs(g).max()
    c = np.zeros((3, n // 2 + 1), complex)
    c[2] = np.fft.rfft(h) / n
    c[2, n // 3 + 1:] = 0.0
    c[2, 0] = 0.0
    return _pack(c)


# The paper's experiments as parareal workloads; grid n = 128 (not stated in the
# paper; SPEC's default).  T = number of slices x ΔT with the paper's slice counts.
PAPER_EXPERIMENTS = {
    "eps1e-2": dict(eps=1e-2, dT=0.5, dt=1.0 / 2500, n_slices=1250, T0=1.5, M=450,
                    standard_dT=(4e-2, 5e-2)),                      # P:1196-1234 (T0 = 150 ε, R4/R17)
    "eps1e-1": dict(eps=1e-1, dT=0.3, dt=1.0 / 250, n_slices=150, T0=0.5, M=10,
                    standard_dT=(0.1, 0.2)),
    "eps1": dict(eps=1.0, dT=0.3, dt=1.0 / 200, n_slices=60, T0=0.3, M=10,
                 standard_dT=(0.3, 0.4)),
}


def random_states(n: int, batch: int, seed: int = 0, kmax: int | None = None,
                  decay: float = 3.0, zero_mean_uv: bool = True, scale: float = 1.0) -> np.ndarray:
    """û_{b,f,k} = scale (1+k)^-decay (z0 + i z1), k = 1..kmax;  k = 0: v1, v2 = 0, h = z (C4 recipe)."""
    nh = n // 2 + 1
    kmax = n // 3 if kmax is None else min(kmax, n // 3)
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((batch, 3, kmax + 1, 2))
    c = np.zeros((batch, 3, nh), complex)
    k = np.arange(1, kmax + 1)
    c[:, :, 1:kmax + 1] = scale * (1.0 + k) ** -decay * (z[:, :, 1:, 0] + 1j * z[:, :, 1:, 1])
    c[:, 2, 0] = scale * z[:, 2, 0, 0]
    if not zero_mean_uv:
        c[:, 0, 0] = scale * z[:, 0, 0, 0]
        c[:, 1, 0] = scale * z[:, 1, 0, 0]
    return _pack(c)
