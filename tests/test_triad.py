"""Triad form of the averaged nonlinearity (P:1113-1118 with Alg.1's quadrature).

CPU tests: the library's host-built triad coefficients W (rsw_triad_coefficients, no GPU involved)
contracted with the eigen coordinates of a state in plain numpy must reproduce the oracle's
M-sample quadrature N̄ (oracle.averaged_rhs: naive DFT, eigendecomposition) to round-off — the
exchange of the quadrature sum with the triad sum is exact for the dealiased product (K = n/3)."""
import numpy as np
import pytest

import oracle
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs


def triad_nbar(W, u, n, F, eps, T0):
    """N̄ (primitive half spectrum) from the triad table in the layout and rotated frame rsw.h documents."""
    K = n // 3
    s = np.sqrt(0.5)
    uc = u[..., 0] + 1j * u[..., 1]
    ks = np.arange(-K, K + 1)
    aks = np.abs(ks)
    a = ks / np.sqrt(F)
    om = np.sqrt(1 + a * a)
    p, q = 1 / (np.sqrt(2) * om), 1 / om
    uh = np.where(ks >= 0, uc[:, aks], np.conj(uc[:, aks]))  # û(κ), κ = -K..K (real fields)
    t = p * (uh[1] - 1j * a * uh[2])
    isu0 = 1j * s * uh[0]
    y = np.array([t + isu0, q * (uh[2] - 1j * a * uh[1]), t - isu0])  # (c-, c0, c+) = R^H û
    tc = 0.5 * T0 / eps
    y = y * np.array([np.exp(1j * om * tc), np.ones_like(om), np.exp(-1j * om * tc)])  # c'^α = c^α e^{-iαωτ_c}
    # the coefficient of entry (γ, α, β) is real when (γ = 0) == (β = 0), else i times the stored value
    unit = np.array([[1, 1j, 1], [1j, 1, 1j], [1, 1j, 1]])[:, None, :]  # [γ][1][β]
    out = np.zeros((3, n // 2 + 1), complex)
    off = 0
    for kap in range(K + 1):
        nk = 2 * K + 1 - kap
        blk = W[off:off + 18 * nk].reshape(3, 2, 3, nk) * unit[..., None]
        off += 18 * nk
        i = np.arange(nk)
        k1, k2 = kap - K + i, K - i
        c = np.einsum("gabi,ai,bi->g", blk, y[[0, 2]][:, k1 + K], y[:, k2 + K])
        om_k = np.sqrt(1 + kap * kap / F)
        c = c * np.exp(1j * np.array([-1, 0, 1]) * om_k * tc)  # back: × e^{iγωτ_c}
        ak, pk, qk = kap / np.sqrt(F), 1 / (np.sqrt(2) * om_k), 1 / om_k
        d, e = c[2] - c[0], c[2] + c[0]
        out[:, kap] = [1j * s * d, pk * e + 1j * ak * qk * c[1], qk * c[1] + 1j * ak * pk * e]
    assert off == W.size
    return out


@pytest.mark.parametrize("n,M,cfg", [(16, 8, "C1"), (64, 32, "C1"), (128, 64, "C2"), (256, 128, "C3"), (512, 32, "C4")])
def test_triad_table_reproduces_quadrature(n, M, cfg):
    w = getattr(inputs, cfg)
    p = rsw.Params(w.eps, w.F, w.mu, n)
    W = rsw.triad_coefficients(p, w.T0, M)
    K = n // 3
    assert W.size == 18 * sum(2 * K + 1 - k for k in range(K + 1))
    u = inputs.random_states(n, 2, seed=5)
    ref = oracle.averaged_rhs(u, w.eps, w.F, w.mu, n, w.T0, M)
    for b in range(2):
        refc = ref[b, ..., 0] + 1j * ref[b, ..., 1]
        out = triad_nbar(W, u[b], n, w.F, w.eps, w.T0)
        assert np.abs(out - refc).max() <= 1e-13 * np.abs(refc).max()


def test_triad_table_errors():
    p = rsw.Params(0.01, 1.0, 1e-4, 2048)
    with pytest.raises(rsw.RSWError):
        rsw.triad_coefficients(p, 0.05, 32)  # n > 1024
    with pytest.raises(rsw.RSWError):
        rsw.triad_coefficients(rsw.Params(0.01, 1.0, 1e-4, 64), 0.05, 1)  # M < 2
