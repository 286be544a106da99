"""NEXT-2: the paper's three RSW experiments on the GPU path, with the paper's initial
condition, mu = 1e-4, F = 1, grid n = 128.  For each ε: the asymptotic parareal
(averaged coarse step with the paper's midpoint rule, Alg.2, and with RK4; ΔT, T0, M̄
from the paper) and the standard parareal with a Strang coarse
solver at the paper's two smaller ΔT, iterations k = 0..5, against the serial fine
(ETDRK4) reference at the slice boundaries.  Error = max_n relative L∞ on the grid.
The paper's figures are placeholders, so this reproduces the experiments, not its numbers.

NEXT-4 (--serial): the paper's serial-accuracy comparison: each serial
integrator of the full equation — ETDRK4, the integrating-factor method (IF-RK4) and Strang splitting
— at Δt = ε/m over the whole interval, error (same metric) against an ETDRK4 solution at Δt = ε/100,
and the largest Δt whose error is at most the asymptotic parareal's error after 5 iterations.

  python tools/paper_experiments.py [--out docs/paper_experiments.json]
  python tools/paper_experiments.py --serial [--out docs/paper_serial_accuracy.json]
  python tools/paper_experiments.py --speedup            (measured B200 times -> docs/paper_speedup.json)
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


def serial_reference(p, u0, dT, dt, S, scheme=0):
    ref = [u0]
    x = u0[None].contiguous()
    for _ in range(S):
        x = rsw.fine_propagate(p, x, dT, dt, scheme)
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


def timed_ms(fn, reps=2):
    fn()  # warm-up (tables, workspace)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def speedup(name, cfg, errors, kmax=5):
    """Measured B200 speedups of the paper's experiment (NEXT-1 / NEXT-2 on the GPU): the serial fine
    ETDRK4 solve of the whole interval (one launch, T/Δt steps) against each parareal variant after
    k = 1..kmax iterations (default schedule: pipelined for the averaged coarse solvers, bulk for the
    Strang coarse solver), with the accuracies of docs/paper_experiments.json beside them."""
    p = rsw.Params(cfg["eps"], F, MU, N_GRID)
    u0 = torch.from_numpy(inputs.paper_initial_state(N_GRID)).cuda()
    T = cfg["n_slices"] * cfg["dT"]
    x = u0[None].contiguous()
    t_serial = timed_ms(lambda: rsw.fine_propagate(p, x, T, cfg["dt"], 0, validate=False), reps=1)
    out = {"eps": cfg["eps"], "T": T, "serial_fine_ms": t_serial,
           "serial_fine_steps": int(np.ceil(T / cfg["dt"] - 1e-9)), "variants": {}}
    runs = ([("asymptotic_midpoint(paper Alg.2)", cfg["dT"], 1), ("asymptotic_rk4", cfg["dT"], 0)]
            + [(f"standard_strang_dT={d:g}", d, 2) for d in cfg["standard_dT"]])
    for label, dT, coarse in runs:
        S = int(round(T / dT))
        rows = []
        for k in range(1, kmax + 1):
            res = {}

            def solve():
                res["r"] = rsw.parareal_iterate(p, u0, dT=dT, dt=cfg["dt"], T0=cfg["T0"], M=cfg["M"], n_slices=S,
                                                max_iters=k, coarse_scheme=coarse, allow_diverged=True)
            ms = timed_ms(solve)
            err = errors.get(label, {}).get("max_rel_linf_error_k0..k5", [None] * (kmax + 1))[k]
            rows.append({"k": k, "ms": ms, "speedup_vs_serial_fine": t_serial / ms, "max_rel_linf_error": err,
                         "pipelined": bool(res["r"]["stats"]["pipelined"])})
            print(name, label, k, f"{ms:.2f} ms", f"speedup {t_serial / ms:.1f}", err, flush=True)
        out["variants"][label] = {"dT": dT, "slices": S, "iterations": rows}
    return out


SERIAL_SCHEMES = {"ETDRK4": 0, "IF-RK4": 2, "Strang": 1}


def serial_accuracy(name, cfg, targets, divisors=(5, 10, 20, 25, 50)):
    p = rsw.Params(cfg["eps"], F, MU, N_GRID)
    u0 = torch.from_numpy(inputs.paper_initial_state(N_GRID)).cuda()
    eps, dT, S = cfg["eps"], cfg["dT"], cfg["n_slices"]
    t = time.time()
    ref = serial_reference(p, u0, dT, eps / 100, S, 0)
    out = {"eps": eps, "T": S * dT, "reference": "ETDRK4, dt = eps/100", "targets": targets, "schemes": {}}
    for sname, sch in SERIAL_SCHEMES.items():
        errs = {}
        for m in divisors:
            U = serial_reference(p, u0, dT, eps / m, S, sch)
            e = max_rel_linf(U, ref)
            errs[f"eps/{m}"] = e if np.isfinite(e) else None
            print(name, sname, f"dt=eps/{m}", "%.2e" % e, flush=True)
        best = {}
        for tname, tval in targets.items():
            ok = [m for m in divisors if errs[f"eps/{m}"] is not None and errs[f"eps/{m}"] <= tval]
            best[tname] = f"eps/{min(ok)}" if ok else None
        out["schemes"][sname] = {"max_rel_linf_error": errs, "largest_dt_reaching": best}
    out["wall_s"] = time.time() - t
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "docs", "paper_experiments.json"))
    ap.add_argument("--only", default="")
    ap.add_argument("--serial", action="store_true")
    ap.add_argument("--speedup", action="store_true", help="measured B200 times -> docs/paper_speedup.json")
    a = ap.parse_args()
    res = {}
    if a.speedup:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        prev = json.load(open(os.path.join(root, "docs", "paper_experiments.json")))
        for name, cfg in inputs.PAPER_EXPERIMENTS.items():
            if a.only and name != a.only:
                continue
            res[name] = speedup(name, cfg, prev[name])
        with open(os.path.join(root, "docs", "paper_speedup.json"), "w") as f:
            json.dump(res, f, indent=1)
        return
    if a.serial:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        prev = json.load(open(os.path.join(root, "docs", "paper_experiments.json")))
        out = a.out if a.out.endswith("serial_accuracy.json") else os.path.join(root, "docs", "paper_serial_accuracy.json")
        for name, cfg in inputs.PAPER_EXPERIMENTS.items():
            if a.only and name != a.only:
                continue
            targets = {lab: v["max_rel_linf_error_k0..k5"][5] for lab, v in prev[name].items()
                       if isinstance(v, dict) and lab.startswith("asymptotic") and v["max_rel_linf_error_k0..k5"][5] == v["max_rel_linf_error_k0..k5"][5]}
            res[name] = serial_accuracy(name, cfg, {f"{k} (k=5)": t for k, t in targets.items()})
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
        return
    for name, cfg in inputs.PAPER_EXPERIMENTS.items():
        if a.only and name != a.only:
            continue
        res[name] = run(name, cfg)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
