"""Bulk-schedule coarse sweep time (k = 0 only) of a workload, median over repetitions: A/B of the die
placement (run with and without RSW_NO_DIE_AWARE=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
S = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = inputs.WORKLOADS[name]
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
ts = []
for _ in range(reps):
    r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S or w.n_slices, max_iters=0,
                             allow_diverged=True, schedule=rsw.SCHEDULE_BULK)
    ts.append(r["stats"]["sweep0_ms"])
print(f"{name} S={S or w.n_slices} bulk sweep {np.median(ts):.2f} ms ({np.median(ts) / (S or w.n_slices) / 4 * 1e3:.2f} us/stage RK4) "
      f"die_aware={r['stats']['die_aware']} NO_DIE_AWARE={os.environ.get('RSW_NO_DIE_AWARE', '0')}", flush=True)
