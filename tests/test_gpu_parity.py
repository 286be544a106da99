"""GPU (librsw.so, sm_100a) vs CPU oracle parity on identical seeded inputs:
relative weighted L2 (R12) <= 1e-10 per state / slice endpoint / iterate, identical iteration
counts.  Every call goes through the C-ABI (paper_1303_6615_b200 is a ctypes binding)."""
import numpy as np
import pytest
import torch

from paper_1303_6615_b200 import inputs
from tests.helpers import rel_l2, to_np

pytestmark = pytest.mark.gpu
TOL = 1e-10


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def P(rsw, eps, F, mu, n):
    return rsw.Params(eps, F, mu, n)


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 512, 1024])
def test_nonlinear(rsw_gpu, orc, n):
    u = inputs.random_states(n, 3, seed=n, decay=1.0)  # odd batch: exercises the dummy pair slot
    got = to_np(rsw_gpu.nonlinear(P(rsw_gpu, 1e-2, 1.0, 1e-4, n), dev(u)))
    ref = orc.nonlinear(u, 1e-2, 1.0, 1e-4, n)
    err = rel_l2(got, ref, n)
    assert err.max() < 1e-12, err
    assert np.all(got[:, :, n // 3 + 1:, :] == 0.0)
    assert np.all(got[:, :, 0, 1] == 0.0)


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_fine_c1(rsw_gpu, orc, scheme):
    w = inputs.C1
    u = np.stack([inputs.initial_state(w, seed=s) for s in range(5)])
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u), w.dT, w.dt, scheme))
    ref = orc.fine_propagate(u, w.eps, w.F, w.mu, w.n, w.dT, w.dt, scheme)
    err = rel_l2(got, ref, w.n)
    assert err.max() < TOL, err


@pytest.mark.parametrize("scheme", [0, 1, 2])
@pytest.mark.parametrize("n,eps,mu,dt,steps", [(128, 1e-2, 1e-4, 5e-4, 40), (256, 1e-3, 1e-5, 1e-4, 25),
                                               (512, 1e-3, 1e-5, 1e-4, 6), (1024, 1e-4, 1e-6, 2e-5, 4)])
def test_fine_sizes(rsw_gpu, orc, scheme, n, eps, mu, dt, steps):
    u = inputs.random_states(n, 3, seed=7, kmax=min(64, n // 3))
    dT = steps * dt * 0.99  # non-integer dT/dt: ceil rule R9
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, eps, 1.0, mu, n), dev(u), dT, dt, scheme))
    ref = orc.fine_propagate(u, eps, 1.0, mu, n, dT, dt, scheme)
    err = rel_l2(got, ref, n)
    assert err.max() < TOL, err


@pytest.mark.parametrize("n", [64, 256])
def test_fine_throughput_layout(rsw_gpu, orc, n):
    """n <= 256 with more than 2 pairs per SM runs 3N/R threads per pair (fewer pairs: twice that);
    601 slices (301 pairs, the last with a dummy slice) take the throughput layout."""
    S = 601
    u = inputs.random_states(n, S, seed=17, kmax=min(32, n // 3))
    eps, mu, dt = 1e-2, 1e-4, 2e-4
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, eps, 1.0, mu, n), dev(u), 2 * dt, dt, 0))
    idx = np.r_[0:4, 297:305, S - 4:S]  # both layouts' tails and the dummy-slice pair
    ref = orc.fine_propagate(u[idx], eps, 1.0, mu, n, 2 * dt, dt, 0)
    err = rel_l2(got[idx], ref, n)
    assert err.max() < TOL, err


@pytest.mark.parametrize("S", [1, 5, 7])
def test_fine_pair_groups_tail(rsw_gpu, orc, S):
    """n = 1024 runs two pair-groups per CTA: S = 1 (one group with a dummy slice), 5 (the second
    CTA's second group idle), 7 (last pair with a dummy slice) against the oracle."""
    n, eps, mu, dt = 1024, 1e-4, 1e-6, 2e-5
    u = inputs.random_states(n, S, seed=13, kmax=64)
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, eps, 1.0, mu, n), dev(u), 2 * dt, dt, 0))
    ref = orc.fine_propagate(u, eps, 1.0, mu, n, 2 * dt, dt, 0)
    err = rel_l2(got, ref, n)
    assert err.max() < TOL, err


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_fine_linear_only(rsw_gpu, orc, scheme):
    n = 128
    u = inputs.random_states(n, 4, seed=3)
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, 1e-2, 1.0, 1e-4, n), dev(u), 0.1, 1e-3, scheme,
                                       flags=rsw_gpu.FLAG_LINEAR_ONLY))
    ref = orc.fine_propagate(u, 1e-2, 1.0, 1e-4, n, 0.1, 1e-3, scheme, flags=1)
    assert rel_l2(got, ref, n).max() < 1e-12


def test_fine_in_place(rsw_gpu, orc):
    w = inputs.C1
    u = np.stack([inputs.initial_state(w, seed=s) for s in range(3)])
    t = dev(u)
    rsw_gpu.fine_propagate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), t, w.dT, w.dt, 0, out=t)
    ref = orc.fine_propagate(u, w.eps, w.F, w.mu, w.n, w.dT, w.dt, 0)
    assert rel_l2(to_np(t), ref, w.n).max() < TOL


@pytest.mark.parametrize("n,eps,T0,M", [(16, 1e-2, 0.05, 8), (32, 1e-2, 0.05, 16), (64, 1e-2, 0.05, 32),
                                        (128, 1e-2, 0.05, 64), (256, 1e-3, 0.01, 128), (512, 1e-3, 0.01, 256),
                                        (1024, 1e-4, 0.002, 16)])
@pytest.mark.parametrize("form", ["triad", "quadrature"])
def test_averaged_rhs(rsw_gpu, orc, n, eps, T0, M, form, monkeypatch):
    """Both evaluations of N̄ (triad form for n <= 512, else / RSW_COARSE_TRIAD=0 the
    per-sample pseudo-spectral kernel) against the oracle's Alg.1 quadrature."""
    if form == "quadrature":
        monkeypatch.setenv("RSW_COARSE_TRIAD", "0")
    nb = 3 if n < 512 else 2
    u = inputs.random_states(n, nb, seed=11)
    got = to_np(rsw_gpu.averaged_rhs(P(rsw_gpu, eps, 1.0, 1e-5, n), dev(u), T0, M))
    ref = orc.averaged_rhs(u, eps, 1.0, 1e-5, n, T0, M)
    assert rel_l2(got, ref, n).max() < TOL


@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("wname", ["C1", "C3"])
def test_coarse(rsw_gpu, orc, scheme, wname):
    w = inputs.WORKLOADS[wname]
    u = np.stack([inputs.initial_state(w, seed=s) for s in range(2)])
    got = to_np(rsw_gpu.coarse_propagate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u), w.dT, w.T0, w.M, scheme))
    ref = orc.coarse_propagate(u, w.eps, w.F, w.mu, w.n, w.dT, w.T0, w.M, scheme)
    assert rel_l2(got, ref, w.n).max() < TOL


@pytest.mark.parametrize("n", [512, 1024])
def test_coarse_large_n(rsw_gpu, orc, n):
    """Coarse step at the radix-16 sizes (512 = 2.16.16, 1024 = 4.16.16) with a small sample count."""
    u = inputs.random_states(n, 2, seed=31, kmax=64)
    eps, mu, dT, T0, M = 1e-4, 1e-6, 0.0078125, 0.002, 8
    got = to_np(rsw_gpu.coarse_propagate(P(rsw_gpu, eps, 1.0, mu, n), dev(u), dT, T0, M, 0))
    ref = orc.coarse_propagate(u, eps, 1.0, mu, n, dT, T0, M, 0)
    assert rel_l2(got, ref, n).max() < TOL


def _parareal_both(rsw, orc, w, seed=0, max_iters=None, tol=None):
    u0 = inputs.initial_state(w, seed=seed)
    mi = w.max_iters if max_iters is None else max_iters
    tl = w.tol if tol is None else tol
    g = rsw.parareal_iterate(P(rsw, w.eps, w.F, w.mu, w.n), dev(u0), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                             n_slices=w.n_slices, max_iters=mi, tol=tl, want_FG=True)
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                     max_iters=mi, tol=tl, want_FG=True)
    return g, r


@pytest.mark.parametrize("k", [0, 1, 2, 4])
def test_parareal_c1_every_iterate(rsw_gpu, orc, k):
    w = inputs.C1
    g, r = _parareal_both(rsw_gpu, orc, w, max_iters=k)
    assert g["iters"] == r["iters"] == k
    err = rel_l2(to_np(g["U"]), r["U"], w.n)
    assert err[1:].max() < TOL, err
    assert np.array_equal(to_np(g["U"])[0], inputs.initial_state(w))
    if k:
        assert np.allclose(g["resid"], r["resid"], rtol=1e-8, atol=0)
        assert rel_l2(to_np(g["F"]), r["F"], w.n).max() < TOL


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_parareal_c1_seeds(rsw_gpu, orc, seed):
    g, r = _parareal_both(rsw_gpu, orc, inputs.C1, seed=seed)
    assert rel_l2(to_np(g["U"]), r["U"], 64)[1:].max() < TOL
    assert np.allclose(g["resid"], r["resid"], rtol=1e-8, atol=0)


def test_parareal_c1_strang_midpoint(rsw_gpu, orc):
    w = inputs.C1
    u0 = inputs.initial_state(w)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=3, fine_scheme=1, coarse_scheme=1)
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u0), **kw)
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, **kw)
    assert rel_l2(to_np(g["U"]), r["U"], w.n)[1:].max() < TOL


# ------------------------------------------------------------------ full-size parity (fixtures)
GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def _fixture(name):
    import os
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"missing oracle fixture {name}: run tests/golden/make_oracle_fixtures.py")
    return np.load(path)


def test_parareal_c2_identical_iteration_count(rsw_gpu):
    """C2: parareal to tol 1e-6 stops at the same k as the oracle, same residuals and iterate."""
    ref = _fixture("oracle_C2.npz")
    w = inputs.C2
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(inputs.initial_state(w)), dT=w.dT,
                                 dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol)
    assert g["iters"] == int(ref["iters"]) == 11
    assert g["status"] == 0
    assert np.allclose(g["resid"], ref["resid"], rtol=1e-8, atol=0)
    assert rel_l2(to_np(g["U"]), ref["U"], w.n)[1:].max() < TOL


def test_parareal_c3_bench_configuration(rsw_gpu):
    """C3 whole solve in bench.py's launch configuration: residual history of every iterate and the
    final U (every 8th slice and the last) against the oracle's full run."""
    ref = _fixture("oracle_C3.npz")
    w = inputs.C3
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(inputs.initial_state(w)), dT=w.dT,
                                 dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters)
    assert g["iters"] == int(ref["iters"]) == 5
    assert np.allclose(g["resid"], ref["resid"], rtol=1e-8, atol=0)
    err = rel_l2(to_np(g["U"])[ref["idx"]], ref["U"], w.n)
    assert err[1:].max() < TOL, err.max()


@pytest.mark.parametrize("k", [1, 2])
def test_parareal_c5_prefix(rsw_gpu, k):
    """C5 at full size (4096 slices, n = 1024): the first 8 slices of U^k equal the oracle's
    self-contained 8-slice problem (U^k_n depends only on slices < n).  C5 iterates blow up further
    down the chain, so the guard may report divergence; the prefix is still checked."""
    ref = _fixture("oracle_C5_prefix8.npz")[f"U{k}"]
    w = inputs.C5
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(inputs.initial_state(w)), dT=w.dT,
                                 dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=k,
                                 allow_diverged=True)
    assert rel_l2(to_np(g["U"])[1:9], ref[1:9], w.n).max() < TOL


@pytest.mark.parametrize("form", ["triad", "quadrature"])
def test_averaged_rhs_c4_full_size_sampled(rsw_gpu, orc, form, monkeypatch):
    """C4 at full size (4096 states, n = 512, M = 256) in the bench's launch configurations (triad form,
    and the per-sample kernel beside it); the oracle evaluates sampled states one by one (first and
    last pair, a pair in the middle)."""
    if form == "quadrature":
        monkeypatch.setenv("RSW_COARSE_TRIAD", "0")
    w = inputs.C4
    u = inputs.initial_state(w)
    assert u.shape[0] == 4096
    got = to_np(rsw_gpu.averaged_rhs(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u), w.T0, w.M))
    idx = np.array([0, 1, 2047, 2048, 4094, 4095])
    ref = orc.averaged_rhs(u[idx], w.eps, w.F, w.mu, w.n, w.T0, w.M)
    assert rel_l2(got[idx], ref, w.n).max() < TOL


def test_fine_c5_full_size_sampled(rsw_gpu, orc):
    """The bench's fine_c5 launch: the C5 fine sweep over 4096 slices (n = 1024, 391 ETDRK4 steps, two
    pair-groups per CTA); the oracle propagates the first and the last slice one by one."""
    w = inputs.C5
    u = inputs.random_states(w.n, w.n_slices, seed=0, kmax=64)
    got = to_np(rsw_gpu.fine_propagate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u), w.dT, w.dt, 0))
    idx = np.array([0, w.n_slices - 1])
    ref = orc.fine_propagate(u[idx], w.eps, w.F, w.mu, w.n, w.dT, w.dt, 0)
    assert rel_l2(got[idx], ref, w.n).max() < TOL


def test_parareal_c5_full_size_identities(rsw_gpu):
    """C5 at full size (4096 slices, n = 1024) through properties that hold at any size, on the GPU's
    own arrays (no oracle input comes from the CUDA path): the k = 0 sweep is the coarse chain
    U^0_{n+1} = G(U^0_n); the first iteration's update U^1_{n+1} = G(U^1_n) + (F(U^0_n) - G(U^0_n))
    holds bitwise; U_0 is never modified; r_1 recomputed on the host (R12)."""
    w = inputs.C5
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = inputs.initial_state(w)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, want_FG=True, allow_diverged=True)
    r0 = rsw_gpu.parareal_iterate(p, dev(u0), max_iters=0, **kw)
    r1 = rsw_gpu.parareal_iterate(p, dev(u0), max_iters=1, **kw)
    U0, G0 = to_np(r0["U"]), to_np(r0["G"])
    U1, F0, G1 = to_np(r1["U"]), to_np(r1["F"]), to_np(r1["G"])
    assert np.isfinite(U1).all()
    assert np.array_equal(U0[1:], G0)
    assert np.array_equal(U1[1:], G1 + (F0 - G0))
    assert np.array_equal(U1[0], u0) and np.array_equal(U0[0], u0)
    r_host = rel_l2(U0[1:], U1[1:], w.n).max()
    assert r1["iters"] == 1 and abs(r1["resid"][0] - r_host) <= 1e-10 * r_host


# ------------------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_world_bitwise(rsw_gpu, world, monkeypatch):
    """Sharding the fine sweep over P (virtual) ranks leaves every iterate bitwise unchanged."""
    w = inputs.C3
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2)
    u0 = dev(inputs.initial_state(w))
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    monkeypatch.delenv("RSW_VIRTUAL_WORLD", raising=False)
    a = to_np(rsw_gpu.parareal_iterate(p, u0, **kw)["U"])
    monkeypatch.setenv("RSW_VIRTUAL_WORLD", str(world))
    b = to_np(rsw_gpu.parareal_iterate(p, u0, **kw)["U"])
    assert np.array_equal(a, b)


def test_determinism(rsw_gpu):
    w = inputs.C1
    u = dev(np.stack([inputs.initial_state(w, seed=s) for s in range(4)]))
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    f1, f2 = to_np(rsw_gpu.fine_propagate(p, u, w.dT, w.dt)), to_np(rsw_gpu.fine_propagate(p, u, w.dT, w.dt))
    assert np.array_equal(f1, f2)
    a1, a2 = to_np(rsw_gpu.averaged_rhs(p, u, w.T0, w.M)), to_np(rsw_gpu.averaged_rhs(p, u, w.T0, w.M))
    assert np.array_equal(a1, a2)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=3)
    assert np.array_equal(to_np(rsw_gpu.parareal_iterate(p, u[0], **kw)["U"]),
                          to_np(rsw_gpu.parareal_iterate(p, u[0], **kw)["U"]))


def test_edge_sizes(rsw_gpu, orc):
    """Single slice (dummy pair slot), odd slice counts, one-slice parareal, max_iters = 0, empty batch."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    for nb in (1, 3):
        u = np.stack([inputs.initial_state(w, seed=s) for s in range(nb)])
        got = to_np(rsw_gpu.fine_propagate(p, dev(u), 0.01, w.dt))
        assert rel_l2(got, orc.fine_propagate(u, w.eps, w.F, w.mu, w.n, 0.01, w.dt), w.n).max() < TOL
    u0 = inputs.initial_state(w)
    for S, k in ((1, 1), (3, 2), (8, 0)):
        g = rsw_gpu.parareal_iterate(p, dev(u0), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=k)
        r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=k)
        assert g["iters"] == r["iters"] == k
        assert rel_l2(to_np(g["U"]), r["U"], w.n)[1:].max() < TOL
    empty = rsw_gpu.fine_propagate(p, dev(np.zeros((0,) + w.state_shape)), w.dT, w.dt)
    assert empty.shape[0] == 0


@pytest.mark.parametrize("schedule", ["bulk", "pipelined"])
@pytest.mark.parametrize("fault", ["nan", "overflow"])
def test_divergence_guard_fault_injection(rsw_gpu, schedule, fault):
    """Fault injection: a NaN in one retained mode of u0, or an amplitude that overflows in
    the first N-evals, must end the solve with RSW_ERR_DIVERGED (non-finite or > 1e6 residual)
    under both schedules — never a hang on the pipelined schedule's sentinel hand-off."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = inputs.initial_state(w)
    if fault == "nan":
        u0[2, 3, 0] = np.nan
    else:
        u0 = u0 * 1e150
    sched = rsw_gpu.SCHEDULE_BULK if schedule == "bulk" else rsw_gpu.SCHEDULE_PIPELINED
    g = rsw_gpu.parareal_iterate(p, dev(u0), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                                 max_iters=3, schedule=sched, allow_diverged=True)
    assert g["status"] == rsw_gpu.RSW_ERR_DIVERGED
    # the library stays usable after the guard fired
    ok = rsw_gpu.parareal_iterate(p, dev(inputs.initial_state(w)), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                                  n_slices=w.n_slices, max_iters=1, schedule=sched)
    assert ok["status"] == rsw_gpu.RSW_OK and np.isfinite(to_np(ok["U"])).all()


@pytest.mark.parametrize("M", [2, 3, 5])
def test_small_M(rsw_gpu, orc, M):
    """M = 2 (one effective sample), odd M (unpaired last sample)."""
    w = inputs.C1
    u = inputs.random_states(w.n, 2, seed=M)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    got = to_np(rsw_gpu.averaged_rhs(p, dev(u), w.T0, M))
    assert rel_l2(got, orc.averaged_rhs(u, w.eps, w.F, w.mu, w.n, w.T0, M), w.n).max() < TOL
    g = to_np(rsw_gpu.coarse_propagate(p, dev(u), w.dT, w.T0, M))
    assert rel_l2(g, orc.coarse_propagate(u, w.eps, w.F, w.mu, w.n, w.dT, w.T0, M), w.n).max() < TOL


def test_fp64_peak_probe(rsw_gpu):
    v = rsw_gpu.fp64_peak_tflops()
    assert 10.0 < v < 45.0  # B200 FP64: 148 SMs x 64 FMA/clk x 2 x <= 1.965 GHz = 37.2 TFLOP/s


# ------------------------------------------------------ NEXT-1: standard parareal, Strang coarse
@pytest.mark.parametrize("k", [1, 3])
def test_standard_parareal_strang_coarse(rsw_gpu, orc, k):
    """Standard parareal: coarse = one Strang step of size ΔT on the full equation."""
    w = inputs.C1
    u0 = inputs.initial_state(w)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=k, coarse_scheme=2)
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u0), want_FG=True, **kw)
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, want_FG=True, **kw)
    assert rel_l2(to_np(g["U"]), r["U"], w.n)[1:].max() < TOL
    assert rel_l2(to_np(g["G"]), r["G"], w.n).max() < TOL
    assert np.allclose(g["resid"], r["resid"], rtol=1e-8, atol=0)
    gc = to_np(rsw_gpu.coarse_propagate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(u0[None]), w.dT, w.T0, w.M, 2))
    assert rel_l2(gc, orc.coarse_propagate(u0[None], w.eps, w.F, w.mu, w.n, w.dT, w.T0, w.M, 2), w.n).max() < TOL


# ------------------------------------------------ NEXT-2: the paper's experiments (truncated)
@pytest.mark.parametrize("name,coarse", [("eps1e-1", 1), ("eps1e-1", 2), ("eps1", 1)])
def test_paper_experiment_prefix(rsw_gpu, orc, name, coarse):
    """The paper's IC and parameters, first 12 slices, 2 iterations:
    GPU = oracle for the paper's midpoint slow solver (Alg.2) and for standard parareal."""
    cfg = inputs.PAPER_EXPERIMENTS[name]
    n = 64
    u0 = inputs.paper_initial_state(n)
    dT = cfg["dT"] if coarse != 2 else cfg["standard_dT"][0]
    kw = dict(dT=dT, dt=cfg["dt"], T0=cfg["T0"], M=cfg["M"], n_slices=12, max_iters=2, coarse_scheme=coarse)
    g = rsw_gpu.parareal_iterate(P(rsw_gpu, cfg["eps"], 1.0, 1e-4, n), dev(u0), **kw)
    r = orc.parareal(u0, cfg["eps"], 1.0, 1e-4, n, **kw)
    assert rel_l2(to_np(g["U"]), r["U"], n)[1:].max() < TOL
    assert np.allclose(g["resid"], r["resid"], rtol=1e-8, atol=0)


# ---- pipelined schedule (NEXT-3): same arithmetic as the bulk schedule, so results are bitwise equal
@pytest.mark.parametrize("wname,fine_scheme,coarse_scheme", [("C1", 0, 0), ("C1", 1, 1), ("C1", 2, 0), ("C2", 0, 0)])
def test_pipelined_schedule_bitwise_equals_bulk(rsw_gpu, wname, fine_scheme, coarse_scheme):
    w = getattr(inputs, wname)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol,
              fine_scheme=fine_scheme, coarse_scheme=coarse_scheme, want_FG=True)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert b["stats"]["pipelined"] and not a["stats"]["pipelined"]
    assert a["iters"] == b["iters"] and a["resid"] == b["resid"]
    assert torch.equal(a["U"], b["U"])
    assert torch.equal(a["F"], b["F"]) and torch.equal(a["G"], b["G"])


@pytest.mark.parametrize("gc,ng", [(32, 4), (16, 6), (64, 2)])
def test_pipelined_group_layouts_bitwise(rsw_gpu, gc, ng, monkeypatch):
    """C3 (the bench workload, 2 iterations) under several coarse-group layouts: per-pair partials
    and a fixed reduction order make the result independent of how the sweeps are spread."""
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    monkeypatch.setenv("RSW_PIPE_GC", str(gc))
    monkeypatch.setenv("RSW_PIPE_NG", str(ng))
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])


def test_pipelined_die_placement_bitwise(rsw_gpu, monkeypatch):
    """C3 (2 iterations): the pipelined schedule with die-aware coarse groups (each group's CTAs on one
    die, its exchange arrays in L2 pages homed there) and without the placement
    (RSW_NO_DIE_AWARE=1: groups from the global ticket, same homed arena) give bitwise the bulk result;
    the stats report the layout that ran."""
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    monkeypatch.setenv("RSW_NO_DIE_AWARE", "1")
    c = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert not c["stats"]["die_aware"]
    assert b["stats"]["coarse_groups"] >= 1 and b["stats"]["group_ctas"] >= 1
    for r in (b, c):
        assert r["resid"] == a["resid"] and torch.equal(r["U"], a["U"])
    print("die-aware placement:", b["stats"]["die_aware"], "groups", b["stats"]["coarse_groups"], "x",
          b["stats"]["group_ctas"])


def test_pipelined_many_sample_pairs_layout(rsw_gpu):
    """The paper's eps = 1e-2 experiment's coarse setting (n = 128, M = 450: 225 sample pairs per stage)
    with 4 iterations on a truncated chain: the layout cost model picks up to 8 pairs per coarse CTA,
    and the die placement must not shrink the groups past that (PIPE_CFG) — the regression was an
    invalid launch configuration.  Bitwise equal to bulk."""
    cfg = inputs.PAPER_EXPERIMENTS["eps1e-2"]
    p = P(rsw_gpu, cfg["eps"], 1.0, 1e-4, 128)
    u0 = dev(inputs.paper_initial_state(128))
    kw = dict(dT=cfg["dT"], dt=cfg["dt"] * 10, T0=cfg["T0"], M=cfg["M"], n_slices=24, max_iters=4, allow_diverged=True)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert b["stats"]["pipelined"]
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
    print("layout:", b["stats"]["coarse_groups"], "x", b["stats"]["group_ctas"], "die_aware", b["stats"]["die_aware"])


def test_device_topology(rsw_gpu):
    """the die-homing probe splits the SMs into two dies (a B200 is two dies of 74 SMs
    less the floorswept ones) and finds the page hash on every chunk; the split covers every SM."""
    import torch
    t = rsw_gpu.device_topology()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert sum(t["die_sms"]) == sms
    assert t["probed"], t
    assert min(t["die_sms"]) >= sms // 3
    print("dies:", t)


def test_check_states_layout(rsw_gpu):
    """§8(b): an input with a non-zero mode k > n/3 (R10) or Im û_0 != 0 (R16) is RSW_ERR_CONFIG —
    through rsw_check_states, through parareal_iterate's own device check of u0, and through the
    binding's default check before the asynchronous entry points."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u = inputs.random_states(w.n, 3, seed=1)
    rsw_gpu.check_states(p, dev(u))
    hi = u.copy()
    hi[1, 2, w.n // 3 + 1, 0] = 1e-3
    im0 = u.copy()
    im0[2, 0, 0, 1] = 0.5
    for bad in (hi, im0):
        with pytest.raises(rsw_gpu.RSWError) as e:
            rsw_gpu.check_states(p, dev(bad))
        assert e.value.status == rsw_gpu.RSW_ERR_CONFIG
        with pytest.raises(rsw_gpu.RSWError) as e:
            rsw_gpu.fine_propagate(p, dev(bad), w.dT, w.dt)
        assert e.value.status == rsw_gpu.RSW_ERR_CONFIG
    for k in (1, 2):
        bad0 = hi[1] if k == 1 else im0[2]
        for sched in (rsw_gpu.SCHEDULE_BULK, rsw_gpu.SCHEDULE_AUTO):
            with pytest.raises(rsw_gpu.RSWError) as e:
                rsw_gpu.parareal_iterate(p, dev(bad0), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                                         max_iters=1, schedule=sched)
            assert e.value.status == rsw_gpu.RSW_ERR_CONFIG
    # the library stays usable
    g = rsw_gpu.parareal_iterate(p, dev(u[0]), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=1)
    assert g["status"] == rsw_gpu.RSW_OK


def test_auto_schedule_falls_back_to_bulk(rsw_gpu, monkeypatch):
    """AUTO must run the bulk schedule when the pipelined kernel cannot hold the
    configuration (M/2 = 1250 sample pairs > 8 per coarse CTA x 148 co-resident CTAs); an explicit
    PIPELINED request fails with RSW_ERR_CONFIG.  With M/2 = 500 pairs the coarse groups are re-sized
    (8 pairs per CTA) and the pipelined schedule runs, bitwise equal to bulk.  (The sample-pair limits
    belong to the M-sample quadrature sweeps; the triad sweeps have none, see
    test_triad_any_M_runs_pipelined.)"""
    monkeypatch.setenv("RSW_COARSE_TRIAD", "0")
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    for M, pipelined in ((2500, False), (1000, True)):
        kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=M, n_slices=w.n_slices, max_iters=2)
        a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_AUTO, **kw)
        b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
        assert a["stats"]["pipelined"] == pipelined
        assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
        if not pipelined:
            with pytest.raises(rsw_gpu.RSWError) as e:
                rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
            assert e.value.status == rsw_gpu.RSW_ERR_CONFIG


@pytest.mark.parametrize("schedule", ["bulk", "pipelined"])
def test_two_streams_share_the_workspace_safely(rsw_gpu, schedule):
    """two parareal_iterate calls issued back to back on different streams (no stats, so the
    first returns with its copies out of the workspace still queued) must not corrupt each other:
    the library orders every call after the previous user of the workspace."""
    import ctypes
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    sch = rsw_gpu.SCHEDULE_BULK if schedule == "bulk" else rsw_gpu.SCHEDULE_PIPELINED
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2, schedule=sch)
    u0 = [dev(inputs.initial_state(w, seed=s)) for s in (0, 1)]
    ref = [rsw_gpu.parareal_iterate(p, u, **kw)["U"].clone() for u in u0]
    L = rsw_gpu.load()
    cfg = rsw_gpu._PararealConfig(w.dT, w.dt, w.T0, 0.0, w.M, w.n_slices, 2, 0, 0, sch)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [torch.full_like(ref[0], float("nan")) for _ in range(2)]
    res = [(ctypes.c_double * 2)() for _ in range(2)]
    its = [ctypes.c_int32() for _ in range(2)]
    torch.cuda.synchronize()
    for i in range(2):
        rc = L.parareal_iterate(ctypes.byref(p._c()), ctypes.byref(cfg), ctypes.c_void_p(u0[i].data_ptr()),
                                ctypes.c_void_p(out[i].data_ptr()), res[i], ctypes.byref(its[i]), None,
                                ctypes.c_void_p(streams[i].cuda_stream))
        assert rc == rsw_gpu.RSW_OK
    torch.cuda.synchronize()
    for i in range(2):
        assert torch.equal(out[i], ref[i])


def test_comm_world1_runs_the_nccl_exchange(rsw_gpu):
    """a6 through the library on one GPU: a real NCCL communicator of world size 1 (rsw_nccl_unique_id,
    rsw_comm_init, the in-place ncclAllGather of parareal_iterate) gives the bulk schedule's iterates
    bitwise."""
    import os
    import socket
    import torch.distributed as dist
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2)
    ref = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", torch.cuda.current_device()))
    comm = None
    try:
        comm = rsw_gpu.Comm.from_torch_distributed()
        g = rsw_gpu.parareal_iterate(p, u0, comm=comm, **kw)
        assert not g["stats"]["pipelined"]
        assert g["resid"] == ref["resid"] and torch.equal(g["U"], ref["U"])
    finally:
        if comm:
            comm.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("wname,max_iters,tol", [("C3", 2, 0.0), ("C2", 64, 1e-6)])
def test_pipelined_push_to_peer_mirror(rsw_gpu, wname, max_iters, tol, monkeypatch):
    """Multi-GPU pipelined schedule on one GPU (RSW_PIPE_MIRROR=1): every finished fine pair is ALSO
    pushed into a same-GPU "peer" copy of F (NVLink-store code path: copy, system fence, system-scope
    release of the peer's done flag).  The pushed copy must equal F bitwise and every pair of the
    iterations used must be released; the solve itself is unchanged (bitwise equal to bulk)."""
    w = getattr(inputs, wname)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=max_iters, tol=tol, want_FG=True)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    monkeypatch.setenv("RSW_PIPE_MIRROR", "1")
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert b["stats"]["pipelined"]
    assert a["iters"] == b["iters"] and a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
    assert torch.equal(a["F"], b["F"])  # b["F"] is the pushed (mirror) copy


@pytest.mark.parametrize("wname", ["C3", "C1"])
def test_bulk_fine_kernel_stores_to_peer_mirror(rsw_gpu, wname, monkeypatch):
    """Multi-GPU bulk schedule on one GPU (RSW_BULK_MIRROR=1): the fine kernel also stores every slice's
    endpoint into a same-GPU "peer" copy of F (the fused compute + exchange path that replaces the
    all-gather: NVLink stores from the fine epilogue, system fence).  The stored copy equals F bitwise
    and the solve is unchanged."""
    w = getattr(inputs, wname)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2, want_FG=True,
              schedule=rsw_gpu.SCHEDULE_BULK)
    a = rsw_gpu.parareal_iterate(p, u0, **kw)
    monkeypatch.setenv("RSW_BULK_MIRROR", "1")
    b = rsw_gpu.parareal_iterate(p, u0, **kw)
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
    assert torch.equal(a["F"], b["F"])  # b["F"] is the stored (mirror) copy


def test_pipelined_long_fine_task_outlives_the_watchdog_limit(rsw_gpu, monkeypatch):
    """a dependency wait may legitimately last one whole fine solve.  With the watchdog limit
    lowered to 100 ms (RSW_WATCHDOG_MS) and fine tasks of ~150k steps (several times the limit), the
    pipelined solve must still complete — the waits time out only without progress anywhere (the fine
    workers' heartbeat) — and equal the bulk schedule bitwise."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dT / 150000, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=1)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    monkeypatch.setenv("RSW_WATCHDOG_MS", "100")
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert b["stats"]["fine_task_ms"] > 300.0, b["stats"]  # each task lasted several watchdog limits
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])


@pytest.mark.parametrize("wname,k_ckpt", [("C3", 2), ("C2", 6)])
def test_checkpoint_resume_bitwise(rsw_gpu, wname, k_ckpt):
    """Checkpoint / resume: the {U^k, G(U^k_n), k} of a run stopped after k iterations (any
    schedule) continued with parareal_resume gives the uninterrupted run bitwise — iterates, residual
    history, and (C2) the tolerance stop at the same iteration."""
    w = getattr(inputs, wname)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, tol=w.tol)
    full = rsw_gpu.parareal_iterate(p, u0, max_iters=w.max_iters, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    part = rsw_gpu.parareal_iterate(p, u0, max_iters=k_ckpt, want_FG=True, **kw)  # AUTO: pipelined
    assert part["iters"] == k_ckpt
    U, G = part["U"].clone(), part["G"].clone()
    res = rsw_gpu.parareal_resume(p, U, G, k_ckpt, max_iters=w.max_iters, **kw)
    assert res["iters"] == full["iters"]
    assert part["resid"] + res["resid"] == full["resid"]
    assert torch.equal(res["U"], full["U"])


def test_runner_cli_and_checkpoint(rsw_gpu, tmp_path):
    """The command-line runner (python -m paper_1303_6615_b200): a 2-iteration C1 run writing a checkpoint,
    then a resumed run to 4 iterations — JSON reports and the final U equal the direct 4-iteration solve."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_1303_6615_b200", "--preset", "C1", *a],
                                    capture_output=True, text=True, timeout=300, cwd=root)
    r1 = run("--max-iter", "2", "--checkpoint", str(tmp_path / "ck.npz"), "--output", str(tmp_path / "r1.json"))
    assert r1.returncode == 0, r1.stderr[-2000:]
    r2 = run("--max-iter", "4", "--resume", str(tmp_path / "ck.npz"), "--save-U", str(tmp_path / "U.npy"),
             "--output", str(tmp_path / "r2.json"))
    assert r2.returncode == 0, r2.stderr[-2000:]
    j1, j2 = (json.load(open(tmp_path / f)) for f in ("r1.json", "r2.json"))
    w = inputs.C1
    ref = rsw_gpu.parareal_iterate(P(rsw_gpu, w.eps, w.F, w.mu, w.n), dev(inputs.initial_state(w)), dT=w.dT, dt=w.dt,
                                   T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=4)
    assert j1["iterations"] == 2 and j2["iterations"] == 4 and j2["status"] == "ok"
    assert j1["residuals"] + j2["residuals"] == ref["resid"]
    assert np.array_equal(np.load(tmp_path / "U.npy"), to_np(ref["U"]))


def test_repeatability_soak(rsw_gpu):
    """Stand-in for racecheck (compute-sanitizer is unavailable on this pool): the lock-free protocols
    (pipelined sentinel hand-offs, task claiming, in-place FFT passes with one barrier each, TMEM
    slots) must give bitwise-identical results run after run under varying timing."""
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=2)
    ref = rsw_gpu.parareal_iterate(p, u0, **kw)
    for _ in range(8):
        r = rsw_gpu.parareal_iterate(p, u0, **kw)
        assert r["resid"] == ref["resid"] and torch.equal(r["U"], ref["U"])
    p5 = P(rsw_gpu, 1e-4, 1.0, 1e-6, 1024)
    u5 = dev(inputs.random_states(1024, 600, seed=21, kmax=64))
    f_ref = rsw_gpu.fine_propagate(p5, u5, 4e-5, 2e-5, 0)
    p4 = P(rsw_gpu, 1e-3, 1.0, 0.0, 512)
    u4 = dev(inputs.random_states(512, 600, seed=22))
    a_ref = rsw_gpu.averaged_rhs(p4, u4, 0.01, 32)
    for _ in range(4):
        assert torch.equal(rsw_gpu.fine_propagate(p5, u5, 4e-5, 2e-5, 0), f_ref)
        assert torch.equal(rsw_gpu.averaged_rhs(p4, u4, 0.01, 32), a_ref)


def test_pipelined_rejects_unsupported(rsw_gpu):
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, 512)
    u0 = dev(inputs.random_states(512, 1, seed=0)[0])
    with pytest.raises(rsw_gpu.RSWError):
        rsw_gpu.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=4, max_iters=1,
                                 schedule=rsw_gpu.SCHEDULE_PIPELINED)


def test_parareal_c1_ifrk4_fine(rsw_gpu, orc):
    """Asymptotic parareal with the integrating-factor fine solver (NEXT-4) vs the oracle."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = inputs.initial_state(w)
    g = rsw_gpu.parareal_iterate(p, dev(u0), dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                                 max_iters=3, fine_scheme=rsw_gpu.FINE_IFRK4)
    r = orc.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                     max_iters=3, fine_scheme=2)
    assert rel_l2(to_np(g["U"]), r["U"], w.n)[1:].max() < TOL
    assert np.allclose(g["resid"], r["resid"], rtol=1e-8, atol=0)


# ------------------------------------------------------ triad form of N̄ in the coarse sweeps
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_triad_sweeps_match_oracle_and_quadrature(rsw_gpu, orc, name, monkeypatch):
    """The triad coarse sweeps (default for n <= 256) and the M-sample quadrature sweeps
    (RSW_COARSE_TRIAD=0) both match the oracle's parareal iterates; the iteration count of the
    tolerance-driven C2 run is the oracle's; bulk and pipelined triad runs agree bitwise."""
    w = getattr(inputs, name)
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = inputs.initial_state(w)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol)
    ref = orc.parareal(u0, w.eps, w.F, w.mu, w.n, **kw) if name == "C1" else _fixture("oracle_C2.npz")
    runs = {}
    for triad in ("1", "0"):
        monkeypatch.setenv("RSW_COARSE_TRIAD", triad)
        for sched in (rsw_gpu.SCHEDULE_BULK, rsw_gpu.SCHEDULE_PIPELINED):
            g = rsw_gpu.parareal_iterate(p, dev(u0), schedule=sched, **kw)
            assert g["stats"]["coarse_triad"] == (triad == "1")
            assert g["iters"] == int(ref["iters"])
            assert rel_l2(to_np(g["U"]), ref["U"], w.n)[1:].max() < TOL
            runs[(triad, sched)] = g
    for triad in ("1", "0"):
        a, b = runs[(triad, rsw_gpu.SCHEDULE_BULK)], runs[(triad, rsw_gpu.SCHEDULE_PIPELINED)]
        assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])


def test_triad_any_M_runs_pipelined(rsw_gpu, orc):
    """The triad sweeps carry no sample pairs, so M = 2500 (beyond the quadrature layout's limit) runs
    pipelined, bitwise equal to bulk and within tolerance of the oracle's coarse propagator."""
    w = inputs.C1
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=2500, n_slices=w.n_slices, max_iters=2)
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_AUTO, **kw)
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    assert a["stats"]["pipelined"] and a["stats"]["coarse_triad"]
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
    u = inputs.random_states(w.n, 2, seed=11)
    g = to_np(rsw_gpu.coarse_propagate(p, dev(u), w.dT, w.T0, 2500))
    assert rel_l2(g, orc.coarse_propagate(u, w.eps, w.F, w.mu, w.n, w.dT, w.T0, 2500), w.n).max() < TOL


def test_triad_global_table_layout_bitwise(rsw_gpu, monkeypatch):
    """A coarse layout whose owned coefficient blocks do not fit shared memory (C3 with 11 CTAs per
    group: 8 owned modes, ~290 KB of coefficients for rank 0) reads the global table instead: the same
    values, bitwise equal to the bulk sweep (which holds its blocks in shared memory)."""
    w = inputs.C3
    p = P(rsw_gpu, w.eps, w.F, w.mu, w.n)
    u0 = dev(inputs.initial_state(w))
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=64, max_iters=2)
    b = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_BULK, **kw)
    monkeypatch.setenv("RSW_PIPE_GC", "11")
    monkeypatch.setenv("RSW_PIPE_NG", "2")
    a = rsw_gpu.parareal_iterate(p, u0, schedule=rsw_gpu.SCHEDULE_PIPELINED, **kw)
    assert a["stats"]["group_ctas"] == 11
    assert a["resid"] == b["resid"] and torch.equal(a["U"], b["U"])
