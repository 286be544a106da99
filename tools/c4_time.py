"""C4 batched N-bar (4096 states, n = 512, M = 256): median CUDA-event time of rsw.averaged_rhs (no layout
check inside the timed calls), in the form the environment selects (RSW_COARSE_TRIAD)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

w = inputs.C4
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u = torch.from_numpy(inputs.random_states(w.n, 4096, seed=0)).cuda()
rsw.averaged_rhs(p, u, w.T0, w.M)
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rsw.averaged_rhs(p, u, w.T0, w.M, validate=False)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"C4 {os.environ.get('RSW_LIB', 'default')}: {ms:.3f} ms, {4096 * rsw.flops_per_unit(w.n, 'triad') / ms / 1e9:.2f} TF (triad flops)")
