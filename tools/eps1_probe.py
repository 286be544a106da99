import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
for n in (32, 64, 128):
    for coarse in (0, 1):
        for M in (10, 40):
            p = rsw.Params(1.0, 1.0, 1e-4, n)
            u0 = torch.from_numpy(inputs.paper_initial_state(n)).cuda()
            r = rsw.parareal_iterate(p, u0, dT=0.3, dt=1/200, T0=0.3, M=M, n_slices=60, max_iters=3, coarse_scheme=coarse, allow_diverged=True)
            U = r["U"].cpu().numpy()
            bad = np.where(~np.isfinite(U).all(axis=(1,2,3)))[0]
            print(n, "midpoint" if coarse else "rk4", M, r["resid"], "first nonfinite slice", bad[:1], flush=True)
