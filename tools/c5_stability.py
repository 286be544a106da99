"""Oracle-only evidence for the behaviour of the C5 parareal iteration.

Runs Alg.4 on a prefix of BASELINE configs[4] (C5: n = 1024, eps = 1e-4, mu = 1e-6,
dT = 0.0078125, dt = 2e-5, T0 = 0.002, M = 256), driving ONLY the CPU oracle's propagators
(oracle.fine_propagate, oracle.coarse_propagate) from this script, and records the per-slice
relative L2 change r_k(n) = ||U^k_n - U^{k-1}_n|| / ||U^k_n|| (R12) for k = 1..K, for
  * the configuration's initial state (C5 recipe), and
  * the same state at half amplitude (the advective coarse-step stability number dT k |v1| halves).
Writes docs/c5_stability.json.  No value comes from the CUDA path.

  python tools/c5_stability.py [--slices 32] [--iters 6]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402


def rel(a, b, n):
    w = np.full(n // 2 + 1, 2.0)
    w[0] = w[-1] = 1.0
    d = (((a - b) ** 2) * w[:, None]).sum(axis=(-1, -2, -3))
    r = ((a ** 2) * w[:, None]).sum(axis=(-1, -2, -3))
    return np.sqrt(d / r)


def run(u0, w, S, K, log):
    kw = dict(eps=w.eps, F=w.F, mu=w.mu, n=w.n)
    U = np.zeros((S + 1,) + u0.shape)
    G = np.zeros((S,) + u0.shape)
    U[0] = u0
    t = time.time()
    for s in range(S):  # k = 0: U_{n+1} = G(U_n)
        G[s] = oracle.coarse_propagate(U[s], dT=w.dT, T0=w.T0, M=w.M, **kw)
        U[s + 1] = G[s]
    log(f"  k=0 sweep {time.time() - t:.0f}s")
    out = []
    for k in range(1, K + 1):
        t = time.time()
        F = oracle.fine_propagate(np.ascontiguousarray(U[:S]), dT=w.dT, dt=w.dt, **kw)  # parfor n
        Uold = U.copy()
        for s in range(S):  # serial sweep
            g = oracle.coarse_propagate(U[s], dT=w.dT, T0=w.T0, M=w.M, **kw)
            U[s + 1] = g + (F[s] - G[s])
            G[s] = g
        rk = rel(U[1:], Uold[1:], w.n)
        finite = bool(np.isfinite(U).all())
        out.append({"k": k, "r_per_slice": [float(x) for x in rk], "r_k": float(np.max(rk)), "finite": finite,
                    "max_abs_v1_grid": float(np.abs(np.fft.irfft((U[:, 0, :, 0] + 1j * U[:, 0, :, 1]) * w.n,
                                                                   n=w.n, axis=-1)).max())})
        log(f"  k={k}: r_k {np.max(rk):.3e}  r(n=1) {rk[0]:.3e}  r(n=S) {rk[-1]:.3e}  {time.time() - t:.0f}s")
        if not finite:
            break
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", type=int, default=32)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--out", default=os.path.join(ROOT, "docs", "c5_stability.json"))
    a = ap.parse_args()
    oracle.build()
    w = inputs.C5
    u0 = inputs.initial_state(w)
    res = {"config": "C5 (BASELINE configs[4]) prefix", "slices": a.slices, "n": w.n, "eps": w.eps, "mu": w.mu,
           "dT": w.dT, "dt_eff": w.dt_eff, "m_fine": w.m_fine, "T0": w.T0, "M": w.M,
           "source": "tools/c5_stability.py: oracle.fine_propagate / oracle.coarse_propagate only", "runs": {}}
    log = lambda s: print(s, flush=True)
    for name, scale in (("amplitude x1 (C5 initial state)", 1.0), ("amplitude x0.5", 0.5)):
        log(f"{name}:")
        res["runs"][name] = run(u0 * scale, w, a.slices, a.iters, log)
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
