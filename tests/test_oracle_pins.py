"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU needed).

Each test is chosen so that a plausible mistake in the oracle (a dropped term, a wrong sign or
index, a transposed operand) fails one of them.  Nothing here re-types the oracle's own formula:
the references are brute force, closed forms, library routines (numpy.fft, scipy.linalg.expm,
scipy.integrate.quad, mpmath), invariants and textbook reductions.  DESIGN.md §4 maps each oracle
function to its pins.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.integrate
import scipy.linalg

from paper_1303_6615_b200 import inputs
from tests.helpers import rel_l2

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cplx(u):
    return u[..., 0] + 1j * u[..., 1]


def pack(c):
    return np.ascontiguousarray(np.stack([c.real, c.imag], -1))


def L_hat(k, F):
    """L̂(k) from the operator table P:1082-1085 with ∂x -> ik."""
    a = k / math.sqrt(F)
    return np.array([[0, -1, 1j * a], [1, 0, 0], [1j * a, 0, 0]], dtype=complex)


def A_mat(k, eps, F, mu):
    """A = -L̂/ε + D̂, D̂ = -μk^4 (Eq. full eqn P:49 moved to the RHS; R2, R3)."""
    return -L_hat(k, F) / eps - mu * k ** 4 * np.eye(3)


# ------------------------------------------------------------------------------------- DFT
def test_dft_brute_force_definition(orc):
    n = 16
    x = np.random.default_rng(0).standard_normal(n)
    X = orc.dft_forward(x)
    j = np.arange(n)
    for k in range(n // 2 + 1):
        ref = sum(x[jj] * complex(math.cos(2 * math.pi * jj * k / n), -math.sin(2 * math.pi * jj * k / n))
                  for jj in j) / n
        assert abs(X[k] - ref) < 1e-15


@pytest.mark.parametrize("n", [16, 64, 256])
def test_dft_vs_numpy_and_roundtrip(orc, n):
    x = np.random.default_rng(n).standard_normal(n)
    X = orc.dft_forward(x)
    assert np.abs(X - np.fft.rfft(x) / n).max() < 1e-14
    Xb = X.copy()
    x2 = orc.dft_inverse(Xb, n)
    assert np.abs(x2 - x).max() < 1e-13 * np.abs(x).max()  # S:64 round trip
    assert np.abs(x2 - np.fft.irfft(X * n, n)).max() < 1e-13


# -------------------------------------------------------------------------------- N(u)
def _convolution_N(u, n):
    """Brute-force O(K^2) truncated convolution of N(u) = -(v1 v1x, v1 v2x, (h v1)x) over the
    signed spectrum |k| <= K (exact for the 2/3-rule pseudo-spectral product, R10)."""
    K = n // 3
    c = cplx(u)

    def full(f, k):
        return c[f, k] if k >= 0 else np.conj(c[f, -k])

    out = np.zeros((3, n // 2 + 1), complex)
    for k in range(K + 1):
        s1 = s2 = s3 = 0.0
        for k1 in range(-K, K + 1):
            k2 = k - k1
            if abs(k2) > K:
                continue
            s1 += full(0, k1) * 1j * k2 * full(0, k2)   # v1 * ∂x v1
            s2 += full(0, k1) * 1j * k2 * full(1, k2)   # v1 * ∂x v2
            s3 += full(2, k1) * full(0, k2)             # h v1
        out[0, k], out[1, k], out[2, k] = -s1, -s2, -1j * k * s3
    return out


@pytest.mark.parametrize("n", [16, 32, 64])
def test_nonlinear_equals_truncated_convolution(orc, n):
    u = inputs.random_states(n, 1, seed=5, decay=0.5, zero_mean_uv=False)[0]
    got = cplx(orc.nonlinear(u, 1e-2, 1.0, 0.0, n))
    ref = _convolution_N(u, n)
    assert np.abs(got - ref).max() < 1e-13 * np.abs(ref).max()


def test_nonlinear_sin_closed_form(orc):
    """v1 = sin x, v2 = h = 0  ->  N1 = -sin x cos x = -½ sin 2x."""
    n = 32
    c = np.zeros((3, n // 2 + 1), complex)
    c[0, 1] = -0.5j  # sin x = (e^{ix} - e^{-ix})/(2i)
    got = cplx(orc.nonlinear(pack(c), 1.0, 1.0, 0.0, n))
    ref = np.zeros_like(c)
    ref[0, 2] = -0.5 * (-0.5j)  # -½ sin 2x
    assert np.abs(got - ref).max() < 1e-15


def test_nonlinear_constant_state_and_mean_h(orc):
    n = 64
    c = np.zeros((3, n // 2 + 1), complex)
    c[:, 0] = [0.3, -1.2, 2.0]
    assert np.abs(orc.nonlinear(pack(c), 1.0, 1.0, 0.0, n)).max() < 1e-14
    u = inputs.random_states(n, 4, seed=1, zero_mean_uv=False)
    out = orc.nonlinear(u, 1.0, 1.0, 0.0, n)
    assert np.abs(out[:, 2, 0, :]).max() < 1e-15  # ĥ_0 of ∂x(h v1) vanishes
    assert np.all(out[:, :, n // 3 + 1:, :] == 0.0)  # 2/3 rule


# ----------------------------------------------------------------------- eigenstructure
@pytest.mark.parametrize("k,F", [(0, 1.0), (1, 1.0), (7, 1.0), (40, 2.5)])
def test_dispersion_relation(orc, k, F):
    """ω_k^α = α √(1 + k²/F);  H = iL̂ = V diag(λ) V^H with V unitary."""
    lam, V = orc.mode_eigen(k, F)
    w = math.sqrt(1 + k * k / F)
    assert np.allclose(lam, [-w, 0.0, w], atol=1e-13 * w)
    H = 1j * L_hat(k, F)
    assert np.abs(V.conj().T @ V - np.eye(3)).max() < 1e-14
    assert np.abs(H @ V - V @ np.diag(lam)).max() < 1e-13 * w


def test_golden_paper_values(orc):
    with open(os.path.join(GOLDEN, "paper_values.json")) as f:
        g = json.load(f)
    for item in g["dispersion"]:
        lam, _ = orc.mode_eigen(item["k"], item["F"])
        assert abs(lam[2] - item["omega"]) < 1e-13, item


# ----------------------------------------------------------------------------- φ-functions
def _phi_mp(j, z):
    import mpmath
    with mpmath.workdps(150):
        z = mpmath.mpc(z.real, z.imag)
        if j == 0:
            r = mpmath.exp(z)
        else:
            s = mpmath.exp(z) - sum(z ** m / mpmath.factorial(m) for m in range(j))
            r = s / z ** j
        return complex(r)


@pytest.mark.parametrize("z", [1e-12, -1e-8, 1e-4, 2e-4, 0.02, -0.5, 0.99, 1.0, 1.5, 20.0, -30.0,
                               0.1 + 2j, 5j, -0.3 + 0.7j, -2e-3 - 0.25j])
@pytest.mark.parametrize("j", [0, 1, 2, 3])
def test_phi_vs_mpmath(orc, j, z):
    z = complex(z)
    ref = _phi_mp(j, z)
    got = orc.phi(j, z)
    assert abs(got - ref) <= 4e-15 * abs(ref), (got, ref)


# ---------------------------------------------------------------- matrix functions f(hA)
def _phi_blocks(X):
    """φ1, φ2, φ3 of a 3x3 matrix via the augmented-matrix exponential (Higham / Sidje):
    expm([[X, I, 0, 0], [0, 0, I, 0], [0, 0, 0, I], [0, 0, 0, 0]]) top row = [e^X, φ1, φ2, φ3]."""
    Z = np.zeros((12, 12), complex)
    Z[:3, :3] = X
    Z[:3, 3:6] = Z[3:6, 6:9] = Z[6:9, 9:12] = np.eye(3)
    E = scipy.linalg.expm(Z)
    return E[:3, :3], E[:3, 3:6], E[:3, 6:9], E[:3, 9:12]


@pytest.mark.parametrize("k", [0, 1, 5, 21])
@pytest.mark.parametrize("eps,mu,h", [(1e-2, 1e-4, 1e-3), (1.0, 1e-4, 0.01), (1e-4, 1e-6, 2e-5)])
def test_etdrk4_matrices_vs_expm(orc, k, eps, mu, h):
    A = A_mat(k, eps, 1.0, mu)
    E, p1, p2, p3 = _phi_blocks(h * A)
    E2, q1, _, _ = _phi_blocks(0.5 * h * A)
    ref = dict(E=E, E2=E2, Q=0.5 * h * q1, f1=h * (p1 - 3 * p2 + 4 * p3), f2=h * (2 * p2 - 4 * p3),
               f3=h * (4 * p3 - p2))
    for name, R in ref.items():
        got = orc.mode_matrix(name, k, h, eps, 1.0, mu)
        assert np.abs(got - R).max() <= 1e-12 * max(np.abs(R).max(), 1e-300), name


@pytest.mark.parametrize("k,tau", [(0, 0.7), (3, -12.5), (30, 200.0)])
def test_expL_vs_expm(orc, k, tau):
    got = orc.mode_matrix("expL", k, tau, 1.0, 1.0, 0.0)
    assert np.abs(got - scipy.linalg.expm(tau * L_hat(k, 1.0))).max() < 1e-12 * (1 + abs(tau) * k)


# ------------------------------------------------------------------------- fine propagators
def test_linear_only_exact(orc):
    """N ≡ 0: u(T) = e^{TA} u(0) per mode (scipy expm), for every fine scheme."""
    n, eps, mu, T = 64, 1e-2, 1e-4, 0.05
    u = inputs.random_states(n, 2, seed=4, zero_mean_uv=False)
    for scheme in (0, 1, 2):
        got = cplx(orc.fine_propagate(u, eps, 1.0, mu, n, T, 1e-3, scheme, flags=1))
        c = cplx(u)
        for k in range(n // 3 + 1):
            ref = (scipy.linalg.expm(T * A_mat(k, eps, 1.0, mu)) @ c[:, :, k].T).T
            assert np.abs(got[:, :, k] - ref).max() < 1e-12


def test_k0_textbook_rotation(orc):
    """A constant-in-x state keeps N ≡ 0; the k=0 flow is the inertial rotation
    v1(t) = v1 cos(t/ε) + v2 sin(t/ε), v2(t) = v2 cos(t/ε) - v1 sin(t/ε), h const."""
    n, eps, T = 32, 0.05, 0.37
    c = np.zeros((3, n // 2 + 1), complex)
    c[:, 0] = [0.4, -0.9, 1.3]
    got = cplx(orc.fine_propagate(pack(c), eps, 1.0, 1e-3, n, T, 1e-2, 0))[:, 0]
    th = T / eps
    ref = [0.4 * math.cos(th) - 0.9 * math.sin(th), -0.9 * math.cos(th) - 0.4 * math.sin(th), 1.3]
    assert np.abs(got - ref).max() < 1e-13


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_mean_height_conserved(orc, scheme):
    w = inputs.C1
    u = inputs.initial_state(w, seed=2)
    out = orc.fine_propagate(u, w.eps, w.F, w.mu, w.n, 0.05, w.dt, scheme)
    assert abs(out[2, 0, 0] - u[2, 0, 0]) < 1e-15
    assert out[2, 0, 1] == 0.0


def _conv_rate(orc, scheme, eps, mu, T, n=64, base=4):
    # base: coarsest number of steps; the reference uses base*64 steps
    u = inputs.random_states(n, 1, seed=9, kmax=8, scale=0.3)[0]
    ref = orc.fine_propagate(u, eps, 1.0, mu, n, T, T / (base * 64), scheme)
    errs = [rel_l2(orc.fine_propagate(u, eps, 1.0, mu, n, T, T / (base * 2 ** i), scheme), ref, n)
            for i in range(3)]
    return [errs[i] / errs[i + 1] for i in range(2)]


@pytest.mark.parametrize("eps,mu", [(1.0, 1e-4), (1e-2, 1e-4)])
def test_etdrk4_fourth_order(orc, eps, mu):
    # asymptotic regime needs dt < ε: 64..256 steps over T = 0.125 at ε = 1e-2
    rates = _conv_rate(orc, 0, eps, mu, T=0.5 if eps == 1.0 else 0.125, base=4 if eps == 1.0 else 64)
    assert all(13.0 < r < 19.5 for r in rates), rates


def test_strang_second_order(orc):
    rates = _conv_rate(orc, 1, 1.0, 1e-4, T=0.5)
    assert all(3.5 < r < 4.6 for r in rates), rates


def _rk4(f, u, h):
    k1 = f(u)
    k2 = f(u + 0.5 * h * k1)
    k3 = f(u + 0.5 * h * k2)
    k4 = f(u + h * k3)
    return u + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)


def test_etdrk4_reduces_to_rk4(orc):
    """ε -> ∞, μ = 0: A = 0, φ_j = 1/j!, and ETDRK4 is classical RK4 on u' = N(u)."""
    n, h = 32, 0.01
    u = inputs.random_states(n, 1, seed=3, scale=0.5)[0]
    f = lambda x: orc.nonlinear(x, 1e30, 1.0, 0.0, n)
    ref = _rk4(f, u, h)
    got = orc.fine_propagate(u, 1e30, 1.0, 0.0, n, h, h, 0)
    assert rel_l2(got, ref, n) < 1e-14


# integrating-factor baseline (RK4 on v = e^{-tA} u)
@pytest.mark.parametrize("eps,mu", [(1.0, 1e-4), (1e-2, 1e-4)])
def test_ifrk4_fourth_order(orc, eps, mu):
    # IF methods reach their asymptotic rate later than ETDRK4 when h max|λ| = h ω_max / ε is large
    # (the transformed nonlinearity oscillates at the fast frequencies): at ε = 1e-2, n = 64 the
    # rates are 80.6 (h ω/ε = 4.1, pre-asymptotic), then 16.7, 16.1, 14.8 (measured)
    rates = _conv_rate(orc, 2, eps, mu, T=0.5 if eps == 1.0 else 0.125, base=4 if eps == 1.0 else 128)
    assert all(13.0 < r < 19.5 for r in rates), rates


def test_ifrk4_reduces_to_rk4(orc):
    """ε -> ∞, μ = 0: the integrating factor is the identity and IF-RK4 is classical RK4."""
    n, h = 32, 0.01
    u = inputs.random_states(n, 1, seed=3, scale=0.5)[0]
    f = lambda x: orc.nonlinear(x, 1e30, 1.0, 0.0, n)
    got = orc.fine_propagate(u, 1e30, 1.0, 0.0, n, h, h, 2)
    assert rel_l2(got, _rk4(f, u, h), n) < 1e-14


def test_ifrk4_solves_the_same_equation(orc):
    """IF-RK4 and ETDRK4 converge to the same trajectory (a wrong transform direction or sign in
    the integrating factor would converge elsewhere): both at small steps agree to O(h^4)."""
    n, eps, mu, T = 64, 1e-2, 1e-4, 0.05
    u = inputs.random_states(n, 1, seed=11, kmax=8, scale=0.3)[0]
    a = orc.fine_propagate(u, eps, 1.0, mu, n, T, T / 512, 2)
    b = orc.fine_propagate(u, eps, 1.0, mu, n, T, T / 2048, 0)
    assert rel_l2(a, b, n) < 1e-11
    # and they are different methods: at a large step they differ well above round-off
    a4 = orc.fine_propagate(u, eps, 1.0, mu, n, T, T / 8, 2)
    b4 = orc.fine_propagate(u, eps, 1.0, mu, n, T, T / 8, 0)
    assert rel_l2(a4, b4, n) > 1e-9


# --------------------------------------------------------------------------- averaging
def test_weights_kernel_moments(orc):
    """w_m >= 0, Σw = 1, w_0 = 0, symmetric; its second central moment converges to that of
    ρ(s) = exp(-1/(s(1-s))) computed by scipy quad."""
    M = 64
    w = orc.weights(M)
    s = np.arange(M) / M
    assert w[0] == 0.0 and np.all(w >= 0) and abs(w.sum() - 1) < 1e-15
    assert abs((w * s).sum() - 0.5) < 1e-15
    rho = lambda x: math.exp(-1.0 / (x * (1 - x)))
    Z = scipy.integrate.quad(rho, 0, 1, epsabs=0, epsrel=1e-13)[0]
    m2 = scipy.integrate.quad(lambda x: rho(x) * (x - 0.5) ** 2, 0, 1, epsabs=0, epsrel=1e-13)[0] / Z
    assert abs((w * (s - 0.5) ** 2).sum() - m2) < 1e-12
    assert abs(1 / Z - 142.25037577709585) < 1e-9  # ||ρ||_1 normalisation constant C
    assert np.array_equal(orc.weights(2), [0.0, 1.0])


def test_average_reduces_to_N_without_scale_separation(orc):
    """ε -> ∞: e^{±τ L̂} = I, Σ w = 1, so N̄(v) = N(v)."""
    n = 32
    u = inputs.random_states(n, 2, seed=8)
    got = orc.averaged_rhs(u, 1e30, 1.0, 0.0, n, 0.05, 16)
    ref = orc.nonlinear(u, 1e30, 1.0, 0.0, n)
    assert rel_l2(got, ref, n).max() < 1e-14


def test_average_homogeneity_and_constants(orc):
    n = 32
    u = inputs.random_states(n, 1, seed=2)
    a = orc.averaged_rhs(u, 1e-2, 1.0, 0.0, n, 0.05, 24)
    b = orc.averaged_rhs(2.0 * u, 1e-2, 1.0, 0.0, n, 0.05, 24)
    assert rel_l2(b, 4.0 * a, n).max() < 1e-14  # N̄(2u) = 4 N̄(u)
    c = np.zeros((1, 3, n // 2 + 1, 2))
    c[0, :, 0, 0] = [0.5, 0.2, 1.0]
    # a constant state is not constant under e^{-τL̂} (inertial rotation) but stays x-independent
    assert np.abs(orc.averaged_rhs(c, 1e-2, 1.0, 0.0, n, 0.05, 24)).max() < 1e-15


def test_average_slow_mode_projection(orc):
    """For v in the α=0 (geostrophic) eigenspace, e^{-τL̂} v = v, so the α=0 component of N̄(v)
    equals that of N(v) exactly; closed-form eigenvector r^0 = (0, ia, 1)/ω."""
    n = 32
    K = n // 3
    rng = np.random.default_rng(4)
    c = np.zeros((3, n // 2 + 1), complex)
    for k in range(1, K + 1):
        w = math.sqrt(1 + k * k)
        amp = (rng.standard_normal() + 1j * rng.standard_normal()) / (1 + k) ** 2
        c[:, k] = amp * np.array([0, 1j * k, 1]) / w
    u = pack(c)[None]
    Nbar = cplx(orc.averaged_rhs(u, 1e-2, 1.0, 0.0, n, 0.05, 32))[0]
    Nu = cplx(orc.nonlinear(u, 1e-2, 1.0, 0.0, n))[0]
    for k in range(1, K + 1):
        r0 = np.array([0, 1j * k, 1]) / math.sqrt(1 + k * k)
        assert abs(r0.conj() @ Nbar[:, k] - r0.conj() @ Nu[:, k]) < 1e-14


def test_average_converges_in_M(orc):
    n = 64
    u = inputs.random_states(n, 1, seed=6)
    prev, diffs = None, []
    for M in (16, 32, 64, 128):
        cur = orc.averaged_rhs(u, 1e-2, 1.0, 0.0, n, 0.05, M)
        if prev is not None:
            diffs.append(rel_l2(cur, prev, n)[0])
        prev = cur
    assert diffs[0] > diffs[1] > diffs[2] and diffs[2] < 1e-9, diffs  # super-algebraic


# ---------------------------------------------------------------------------- coarse step
def test_coarse_reduces_to_rk4(orc):
    """ε -> ∞, μ = 0: G(u) = one RK4 step of size ΔT on u' = N(u) (Alg.2 with R6)."""
    n, dT = 32, 0.02
    u = inputs.random_states(n, 1, seed=12, scale=0.5)[0]
    f = lambda x: orc.nonlinear(x, 1e30, 1.0, 0.0, n)
    got = orc.coarse_propagate(u, 1e30, 1.0, 0.0, n, dT, 0.05, 16)
    assert rel_l2(got, _rk4(f, u, dT), n) < 1e-14


def test_coarse_midpoint_reduces(orc):
    n, dT = 32, 0.02
    u = inputs.random_states(n, 1, seed=13, scale=0.5)[0]
    f = lambda x: orc.nonlinear(x, 1e30, 1.0, 0.0, n)
    got = orc.coarse_propagate(u, 1e30, 1.0, 0.0, n, dT, 0.05, 16, scheme=1)
    assert rel_l2(got, u + dT * f(u + 0.5 * dT * f(u)), n) < 1e-14


def test_coarse_linear_part_exact(orc):
    """With N ≡ 0 (a constant state) G(u) = e^{-(ΔT/ε)L̂} e^{ΔT D̂} u = the exact linear flow."""
    n, eps, dT = 32, 1e-2, 0.125
    c = np.zeros((3, n // 2 + 1), complex)
    c[:, 0] = [0.4, -0.9, 1.3]
    got = cplx(orc.coarse_propagate(pack(c), eps, 1.0, 1e-4, n, dT, 0.05, 32))[:, 0]
    ref = scipy.linalg.expm(dT * A_mat(0, eps, 1.0, 1e-4)) @ c[:, 0]
    assert np.abs(got - ref).max() < 1e-13


def test_coarse_approximates_fine(orc):
    """φ - φ̄ -> 0 as ε -> 0 with T0/ε large: the asymptotic coarse step
    tracks the fine solution over ΔT ≫ ε better than the linear flow alone, and improves as ε
    halves.  A wrong sign of the back-transform (R3) gives O(1) errors; a wrong conjugation sign
    or a missing weight normalisation also fails the margins below."""
    w = inputs.C1
    u = inputs.initial_state(w)
    errs = []
    for eps in (0.005, 0.0025):
        G = orc.coarse_propagate(u, eps, w.F, w.mu, w.n, w.dT, 60 * eps, 480)
        F = orc.fine_propagate(u, eps, w.F, w.mu, w.n, w.dT, eps / 10)
        lin = orc.fine_propagate(u, eps, w.F, w.mu, w.n, w.dT, eps / 10, flags=1)
        errs.append((rel_l2(G, F, w.n), rel_l2(lin, F, w.n)))
    (g1, l1), (g2, l2) = errs
    assert g1 < 0.8 * l1 and g2 < 0.6 * l2 and g2 < 0.8 * g1, errs


# ---------------------------------------------------------------------------- parareal
def test_parareal_exact_after_S_iterations(orc):
    """Telescoping identity: U^k_n equals the serial fine solution for n <= k."""
    w = inputs.C1
    u0 = inputs.initial_state(w)
    ser = [u0]
    for _ in range(w.n_slices):
        ser.append(orc.fine_propagate(ser[-1], w.eps, w.F, w.mu, w.n, w.dT, w.dt))
    ser = np.stack(ser)
    for k in (2, w.n_slices):
        r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                         max_iters=k)
        assert np.array_equal(r["U"][0], u0)
        assert rel_l2(r["U"][1:k + 1], ser[1:k + 1], w.n).max() < 1e-13


def test_parareal_converges_and_stops(orc):
    w = inputs.C1
    u0 = inputs.initial_state(w)
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                     max_iters=8, tol=5e-4)
    res = r["resid"]
    assert all(res[i + 1] < 0.3 * res[i] for i in range(len(res) - 1)), res
    assert r["iters"] == 4 and res[-1] < 5e-4 <= res[-2] and r["status"] == 0


def test_standard_parareal_exact_after_S(orc):
    """NEXT-1, standard parareal with a Strang coarse solver: the same telescoping
    identity holds (U^S_n = serial fine), and the coarse step is one Strang step of the full eqn."""
    w = inputs.C1
    u0 = inputs.initial_state(w)
    S = 4
    ser = [u0]
    for _ in range(S):
        ser.append(orc.fine_propagate(ser[-1], w.eps, w.F, w.mu, w.n, w.dT, w.dt))
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=S,
                     coarse_scheme=2)
    assert rel_l2(r["U"][1:], np.stack(ser[1:]), w.n).max() < 1e-13
    g = orc.coarse_propagate(u0, w.eps, w.F, w.mu, w.n, w.dT, w.T0, w.M, scheme=2)
    assert rel_l2(g, orc.fine_propagate(u0, w.eps, w.F, w.mu, w.n, w.dT, w.dT, scheme=1), w.n) == 0.0


# ---------------------------------------------------------------- residual norm and D half-steps
def _grid(u, n):
    """Physical grid values of a half-spectrum state (numpy.fft.irfft; û_k = (1/n) Σ u_j e^{-ikx_j})."""
    c = cplx(np.asarray(u))
    return np.fft.irfft(c * n, n=n, axis=-1)


def test_residual_is_physical_relative_l2(orc):
    """R12 (Alg.4): r_k = max_{n=1..S} ||U^k_n - U^{k-1}_n||_2 / ||U^k_n||_2 with the L2 norm
    taken over the 3 fields ON THE GRID.  Recomputed here from the oracle's own iterates (runs with
    max_iters = k-1 and k) through numpy.fft.irfft, with no Parseval weights: a residual with unit
    weights, with the denominator U^{k-1}, or with the max taken without slice S fails."""
    w = inputs.C1
    n = w.n
    u0 = inputs.initial_state(w)
    run = lambda k: orc.parareal(u0, w.eps, w.F, w.mu, n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                                 n_slices=w.n_slices, max_iters=k)
    runs = [run(k) for k in range(0, 5)]
    argmax_at_S = 0
    for k in range(1, 5):
        new, old = _grid(runs[k]["U"][1:], n), _grid(runs[k - 1]["U"][1:], n)
        num = np.sqrt(((new - old) ** 2).sum(axis=(-1, -2)))
        den = np.sqrt((new ** 2).sum(axis=(-1, -2)))
        rs = num / den
        # the difference U^k - U^{k-1} cancels ~4 digits at k = 4 (r_4 ~ 1.5e-4), so the grid and the
        # half-spectrum evaluations agree to ~1e-12 relative, not to the 1e-16 of the states
        assert abs(runs[k]["resid"][k - 1] - rs.max()) <= 1e-11 * rs.max(), (k, runs[k]["resid"], rs)
        # the history of the longer run agrees with the shorter ones (same iterates)
        assert np.array_equal(runs[4]["resid"][:k], runs[k]["resid"])
        argmax_at_S += int(np.argmax(rs) == w.n_slices - 1)
        # the pin is sharp: the alternative readings differ from r_k by far more than 1e-13
        den_old = np.sqrt((old ** 2).sum(axis=(-1, -2)))
        assert abs((num / den_old).max() - rs.max()) > 1e-9 * rs.max()
    # slice S attains the max in at least one iteration, so dropping it from the max is caught
    assert argmax_at_S >= 1


def test_residual_weights_are_parseval(orc):
    """The half-spectrum norm the oracle uses equals the grid L2 (Parseval, P:571 / R12): checked on
    its rel_l2 entry against irfft, for random states with a non-zero k = n/2-adjacent spectrum."""
    n = 64
    a = inputs.random_states(n, 2, seed=21)
    ga, gb = _grid(a[0], n), _grid(a[1], n)
    ref = np.sqrt(((ga - gb) ** 2).sum() / (gb ** 2).sum())
    assert abs(orc.rel_l2(n, a[0], a[1]) - ref) < 1e-14 * ref
    # unit weights would give a different value on these states
    d = cplx(a[0] - a[1])
    unit = np.sqrt((np.abs(d) ** 2).sum() / (np.abs(cplx(a[1])) ** 2).sum())
    assert abs(unit - ref) > 1e-3 * ref


def test_coarse_D_half_steps_without_nonlinearity(orc):
    """Alg.2: G = e^{-(ΔT/ε)L̂} e^{(ΔT/2)D̂} RK4_N̄ e^{(ΔT/2)D̂}.  With ε -> ∞
    (L̂/ε -> 0) and v1 ≡ 0 (N ≡ 0, so N̄ ≡ 0) the RK4 stage is the identity and G(u) = e^{-μk⁴ΔT} u
    per mode: a dropped, doubled or un-halved D half-step fails."""
    n, dT, mu = 32, 0.05, 0.3
    rng = np.random.default_rng(5)
    c = np.zeros((3, n // 2 + 1), complex)
    K = n // 3
    c[1:, 1:K + 1] = rng.standard_normal((2, K)) + 1j * rng.standard_normal((2, K))
    c[1:, 0] = rng.standard_normal(2)
    for scheme in (0, 1):
        got = cplx(orc.coarse_propagate(pack(c), 1e30, 1.0, mu, n, dT, 0.05, 16, scheme=scheme))
        k = np.arange(n // 2 + 1)
        ref = c * np.exp(-mu * k ** 4 * dT)[None, :]
        assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max(), scheme


def test_coarse_D_half_steps_around_rk4(orc):
    """The same composition on a general state: D½ ∘ RK4_N ∘ D½ (ε -> ∞, μ > 0), built from
    oracle.nonlinear and numpy.exp(-μk⁴ΔT/2).  Putting both half-steps before (or after) the RK4
    step, or using a full step on one side, changes the result by O(μk⁴ΔT · ΔT N)."""
    n, dT, mu = 32, 0.05, 0.02
    u = inputs.random_states(n, 1, seed=14, scale=0.5)[0]
    k = np.arange(n // 2 + 1)
    dh = np.exp(-mu * k ** 4 * dT / 2)[None, :, None]
    f = lambda x: orc.nonlinear(x, 1e30, 1.0, mu, n)
    ref = dh * _rk4(f, dh * u, dT)
    got = orc.coarse_propagate(u, 1e30, 1.0, mu, n, dT, 0.05, 16)
    assert rel_l2(got, ref, n) < 1e-14
    # the alternative placements differ measurably on this state
    alt = _rk4(f, dh * dh * u, dT)
    assert rel_l2(alt, ref, n) > 1e-6
    refm = dh * ((dh * u) + dT * f(dh * u + 0.5 * dT * f(dh * u)))
    gotm = orc.coarse_propagate(u, 1e30, 1.0, mu, n, dT, 0.05, 16, scheme=1)
    assert rel_l2(gotm, refm, n) < 1e-14
