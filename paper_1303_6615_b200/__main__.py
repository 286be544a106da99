"""Command-line runner of the asymptotic parareal solve on the GPU (SURVEY §5 config / flag system and
JSON report; flag names after SPEC's CLI).

  python -m paper_1303_6615_b200 --preset C1 [--epsilon 0.01] [--modes 64] [--slices 8] [--T 1.0]
         [--delta-t 1e-3] [--t0 0.05] [--mbar 32] [--mu 1e-4] [--F 1.0] [--tol 0] [--max-iter 4]
         [--fine etdrk4|strang|ifrk4] [--coarse rk4|midpoint|strang] [--schedule auto|bulk|pipelined]
         [--seed 0] [--output report.json] [--save-U U.npy] [--checkpoint ckpt.npz] [--resume ckpt.npz]

The preset (BASELINE.json configs, `inputs.C1..C5`) supplies every parameter and the initial-state
recipe; flags override single parameters.  The report echoes the configuration and carries the
per-iteration residuals, the status, the phase timings and the fine slice-steps/s.  Argument
marshalling only: the solve runs in librsw.so (no CPU fallback).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import sys

from . import inputs

FINE = {"etdrk4": 0, "strang": 1, "ifrk4": 2}
COARSE = {"rk4": 0, "midpoint": 1, "strang": 2}
SCHED = {"auto": 0, "bulk": 1, "pipelined": 2}


def parse_args(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1303_6615_b200", description=__doc__.split("\n\n")[0])
    ap.add_argument("--preset", default="C1", choices=[k for k in inputs.WORKLOADS if k != "C4"])
    ap.add_argument("--epsilon", type=float)
    ap.add_argument("--F", type=float)
    ap.add_argument("--mu", type=float)
    ap.add_argument("--modes", type=int, help="grid points n (power of two, 16..1024)")
    ap.add_argument("--T", type=float)
    ap.add_argument("--slices", type=int)
    ap.add_argument("--delta-t", type=float, dest="dt")
    ap.add_argument("--t0", type=float)
    ap.add_argument("--mbar", type=int, help="quadrature points M")
    ap.add_argument("--tol", type=float)
    ap.add_argument("--max-iter", type=int, dest="max_iters")
    ap.add_argument("--fine", choices=FINE, default="etdrk4")
    ap.add_argument("--coarse", choices=COARSE, default="rk4")
    ap.add_argument("--schedule", choices=SCHED, default="auto")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--output", help="JSON report path (default: stdout)")
    ap.add_argument("--save-U", dest="save_u", help="write the final iterate U (numpy .npy)")
    ap.add_argument("--checkpoint", help="write {U, G, k} after the run (numpy .npz) for --resume")
    ap.add_argument("--resume", help="continue from a --checkpoint file (bulk schedule)")
    return ap.parse_args(argv)


def workload_from_args(a) -> inputs.Workload:
    w = inputs.WORKLOADS[a.preset]
    over = {k: v for k, v in dict(eps=a.epsilon, F=a.F, mu=a.mu, n=a.modes, T=a.T, n_slices=a.slices, dt=a.dt,
                                  T0=a.t0, M=a.mbar, tol=a.tol, max_iters=a.max_iters).items() if v is not None}
    return dataclasses.replace(w, fine_scheme=FINE[a.fine], coarse_scheme=COARSE[a.coarse], **over)


def initial_state(w: inputs.Workload, seed: int):
    """The preset's initial-state recipe on this grid, projected onto the retained modes k <= n/3."""
    u0 = inputs.initial_state(w, seed=seed)
    u0[:, w.n // 3 + 1:, :] = 0.0
    u0[:, 0, 1] = 0.0
    return u0


def main(argv=None) -> int:
    import numpy as np
    import torch

    from . import RSW_NOT_CONVERGED, RSW_OK, Params, load, parareal_iterate, parareal_resume

    a = parse_args(argv)
    w = workload_from_args(a)
    load()
    p = Params(w.eps, w.F, w.mu, w.n)
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol,
              fine_scheme=w.fine_scheme, coarse_scheme=w.coarse_scheme)
    if a.resume:
        ck = np.load(a.resume)
        U = torch.from_numpy(np.ascontiguousarray(ck["U"])).cuda()
        G = torch.from_numpy(np.ascontiguousarray(ck["G"])).cuda()
        r = parareal_resume(p, U, G, int(ck["k"]), want_FG=bool(a.checkpoint), allow_diverged=True, **kw)
    else:
        u0 = torch.from_numpy(initial_state(w, a.seed)).cuda()
        r = parareal_iterate(p, u0, schedule=SCHED[a.schedule], want_FG=bool(a.checkpoint), allow_diverged=True, **kw)
    st = r["stats"]
    report = {
        "config": dict(dataclasses.asdict(w), dT=w.dT, m_fine=w.m_fine, dt_eff=w.dt_eff, seed=a.seed,
                       schedule=a.schedule, resumed_from=a.resume),
        "status": {RSW_OK: "ok", RSW_NOT_CONVERGED: "not converged"}.get(r["status"], "diverged"),
        "iterations": r["iters"], "residuals": r["resid"], "stats": st,
        "fine_slice_steps_per_s": (st["fine_slice_steps"] / (st["total_ms"] * 1e-3)) if st["total_ms"] else None,
    }
    text = json.dumps(report, indent=1)
    if a.output:
        with open(a.output, "w") as fh:
            fh.write(text)
    else:
        print(text)
    if a.save_u:
        np.save(a.save_u, r["U"].cpu().numpy())
    if a.checkpoint:
        np.savez(a.checkpoint, U=r["U"].cpu().numpy(), G=r["G"].cpu().numpy(), k=r["iters"])
    return 0 if r["status"] in (RSW_OK, RSW_NOT_CONVERGED) else 3


if __name__ == "__main__":
    sys.exit(main())
