"""NEXT-2: the paper's three RSW experiments on the GPU path, with the paper's initial
condition, mu = 1e-4, F = 1, grid n = 128.  For each ε: the asymptotic parareal
(averaged coarse step with the paper's midpoint rule, Alg.2, and with RK4; ΔT, T0, M̄
from the paper) and the standard parareal with a Strang coarse
solver at the paper's two smaller ΔT, iterations k = 0..5, against the serial fine
(ETDRK4) reference at the slice boundaries.  Error = max_n relative L∞ on the grid.
The paper's figures are placeholders, so this reproduces the experiments, not its numbers.

  python tools/paper_experiments.py [--out docs/paper_experiments.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

N_GRID, MU, F = 128, 1e-4, 1.0


def grid(U):
    c = U[..., 0] + 1j * U[..., 1]
    return np.fft.irfft(c * N_GRID, N_GRID, axis=-1)  # [.., 3, n]


def serial_reference(p, u0, dT, dt, S):
    ref = [u0]
    x = u0[None].contiguous()
    for _ in range(S):
        x = rsw.fine_propagate(p, x, dT, dt)
        ref.append(x[0])
    return torch.stack(ref).cpu().numpy()


def max_rel_linf(U, R):
    g, r = grid(U), grid(R)
    num = np.abs(g - r).reshape(len(g), -1).max(axis=1)
    den = np.abs(r).reshape(len(r), -1).max(axis=1)
    return float((num / den)[1:].max())


def run(name, cfg, kmax=5):
    p = rsw.Params(cfg["eps"], F, MU, N_GRID)
    u0 = torch.from_numpy(inputs.paper_initial_state(N_GRID)).cuda()
    T = cfg["n_slices"] * cfg["dT"]
    out = {"eps": cfg["eps"], "T": T, "grid": N_GRID}
    t = time.time()
    cache = {}

    def ref_for(dT):
        S = int(round(T / dT))
        if S not in cache:
            # the serial fine solution sampled every ΔT_min, coarser grids reuse it
            cache[S] = serial_reference(p, u0, dT, cfg["dt"], S)
        return cache[S]

    # the paper's slow solver is the midpoint rule (Alg.2); BASELINE's RK4 is run beside it
    runs = ([("asymptotic_midpoint(paper Alg.2)", cfg["dT"], 1), ("asymptotic_rk4", cfg["dT"], 0)]
            + [(f"standard_strang_dT={d:g}", d, 2) for d in cfg["standard_dT"]])
    for label, dT, coarse in runs:
        S = int(round(T / dT))
        R = ref_for(dT)
        errs, resid = [], []
        for k in range(kmax + 1):
            r = rsw.parareal_iterate(p, u0, dT=dT, dt=cfg["dt"], T0=cfg["T0"], M=cfg["M"], n_slices=S,
                                     max_iters=k, coarse_scheme=coarse, allow_diverged=True)
            errs.append(max_rel_linf(r["U"].cpu().numpy(), R))
            resid = r["resid"]
        out[label] = {"dT": dT, "slices": S, "fine_steps_per_slice": int(np.ceil(dT / cfg["dt"] - 1e-9)),
                      "max_rel_linf_error_k0..k5": errs, "residuals": resid}
        print(name, label, ["%.2e" % e for e in errs], flush=True)
    out["wall_s"] = time.time() - t
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "docs", "paper_experiments.json"))
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    res = {}
    for name, cfg in inputs.PAPER_EXPERIMENTS.items():
        if a.only and name != a.only:
            continue
        res[name] = run(name, cfg)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
