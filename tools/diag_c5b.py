import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
w = inputs.C5
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
for S in (64, 512, 4096):
    r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=6, allow_diverged=True)
    print(S, r["status"], ["%.3e" % x for x in r["resid"]], r["stats"], flush=True)
    U = r["U"]
    print("   max|U| per 8 slices", [float(U[i].abs().max()) for i in range(0, S+1, max(1, S//8))])
w = inputs.C3
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=5, allow_diverged=True)
print("C3", r["status"], ["%.3e" % x for x in r["resid"]], r["stats"], flush=True)
w = inputs.C2
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=20, tol=w.tol, allow_diverged=True)
print("C2", r["status"], r["iters"], ["%.3e" % x for x in r["resid"]], r["stats"], flush=True)
