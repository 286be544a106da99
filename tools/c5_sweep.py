"""C5 (n = 1024, 4096 slices) bulk coarse sweep alone (max_iters = 0) and one iteration: time per stage,
triad (default) vs per-sample quadrature (RSW_COARSE_TRIAD=0 in the environment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

w = inputs.C5
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
for k in (0, 1):
    for rep in range(2):
        r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=k,
                                 allow_diverged=True, schedule=rsw.SCHEDULE_BULK)
    s = r["stats"]
    print(f"C5 max_iters={k} triad={s['coarse_triad']}: total {s['total_ms']:.1f} ms sweep0 {s['sweep0_ms']:.1f} ms "
          f"({s['sweep0_ms'] * 1e3 / (4 * w.n_slices):.2f} us/stage) resid {r['resid']}", flush=True)
