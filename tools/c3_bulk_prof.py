import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
w = inputs.WORKLOADS["C3"]
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
for rep in range(2):
    r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=0, allow_diverged=True, schedule=1)
    print(r["stats"]["total_ms"])
