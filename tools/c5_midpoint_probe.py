"""Does the paper's midpoint slow solver (Alg.2) keep C5's parareal iterate bounded where BASELINE's
RK4 coarse step diverges?"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
w = inputs.C5
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
for S in (512, 4096):
    for coarse in (1, 0):
        r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=6,
                                 coarse_scheme=coarse, allow_diverged=True)
        print(S, "midpoint" if coarse else "rk4", ["%.3e" % x for x in r["resid"]], r["stats"]["total_ms"], flush=True)
