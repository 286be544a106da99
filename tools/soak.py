"""Long repeatability soak of the pipelined schedule (C2 tolerance stop, C3 fixed iterations): every run
must be bitwise identical to the first.  Usage: python tools/soak.py [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rsw.load()
for name in ("C2", "C3"):
    w = inputs.WORKLOADS[name]
    p = rsw.Params(w.eps, w.F, w.mu, w.n)
    u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol)
    ref = rsw.parareal_iterate(p, u0, **kw)
    bad = 0
    for _ in range(runs):
        r = rsw.parareal_iterate(p, u0, **kw)
        if not (r["iters"] == ref["iters"] and r["resid"] == ref["resid"] and torch.equal(r["U"], ref["U"])):
            bad += 1
    print(f"{name}: {runs} runs, iterations {ref['iters']}, mismatches {bad}", flush=True)
