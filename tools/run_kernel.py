"""Run one hot-path kernel of a workload a few times (for ncu / timing).  Not part of the product."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--what", default="fine", choices=["fine", "strang", "avg", "coarse", "parareal"])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--slices", type=int, default=0)
ap.add_argument("--iters", type=int, default=2, help="parareal: iterations (the bench runs the config's count)")
a = ap.parse_args()
w = inputs.WORKLOADS[a.config]
p = rsw.Params(w.eps, w.F, w.mu, w.n)
rsw.load()
if a.what in ("fine", "strang"):
    S = a.slices or w.n_slices
    u = torch.from_numpy(inputs.random_states(w.n, S, seed=0, kmax=64)).cuda()
    out = torch.empty_like(u)
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rsw.fine_propagate(p, u, w.dT, w.dt, 0 if a.what == "fine" else 1, out=out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        f = rsw.flops_per_unit(w.n, "etdrk4" if a.what == "fine" else "strang")
        print(f"{a.what} {w.name} S={S} m={w.m_fine}: {dt*1e3:.2f} ms  {S*w.m_fine/dt:.3e} slice-steps/s "
              f"{S*w.m_fine*f/dt/1e12:.2f} TF")
elif a.what == "avg":
    S = a.slices or 4096
    w4 = inputs.C4
    p = rsw.Params(w4.eps, w4.F, w4.mu, w4.n)
    u = torch.from_numpy(inputs.random_states(w4.n, S, seed=0)).cuda()
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rsw.averaged_rhs(p, u, w4.T0, w4.M)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        f = rsw.flops_per_unit(w4.n, "sample")
        print(f"avg C4 S={S}: {dt*1e3:.2f} ms  {S*(w4.M-1)/dt:.3e} sample-evals/s {S*(w4.M-1)*f/dt/1e12:.2f} TF")
elif a.what == "coarse":
    u = torch.from_numpy(inputs.initial_state(w)).cuda()[None].repeat(a.slices or 4, 1, 1, 1).contiguous()
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rsw.coarse_propagate(p, u, w.dT, w.T0, w.M)
        torch.cuda.synchronize()
        print(f"coarse {w.name} x{u.shape[0]}: {(time.perf_counter()-t)*1e3/u.shape[0]:.3f} ms per step")
else:
    u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
    for r in range(a.reps):
        res = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices,
                                   max_iters=min(w.max_iters, a.iters), tol=w.tol)
        print(res["stats"], res["resid"])
