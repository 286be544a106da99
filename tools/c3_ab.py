"""C3 pipelined solve: median time-to-solution and phase split over a few repetitions (A/B of library
variants: run once per RSW_LIB).  Prints one line: total, sweep 0, lag, fine task (ms), bitwise hash."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
w = inputs.WORKLOADS[name]
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol,
          allow_diverged=True, schedule=rsw.SCHEDULE_PIPELINED)
rows = []
for _ in range(reps):
    r = rsw.parareal_iterate(p, u0, **kw)
    s = r["stats"]
    rows.append((s["total_ms"], s["sweep0_ms"], s["lag_ms"], s["fine_task_ms"]))
med = np.median(np.array(rows), axis=0)
h = hashlib.sha1(r["U"].cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{os.environ.get('RSW_LIB', 'default')}: total {med[0]:.2f} sweep0 {med[1]:.2f} lag {med[2]:.3f} "
      f"fine_task {med[3]:.3f} ms (min total {min(x[0] for x in rows):.2f}) U {h}", flush=True)
