"""Per-sweep coarse timing from parareal stats (device events inside the library)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
for name in sys.argv[1:] or ["C1", "C2", "C3"]:
    w = inputs.WORKLOADS[name]
    p = rsw.Params(w.eps, w.F, w.mu, w.n)
    u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
    S = w.n_slices if name != "C5" else 512
    for rep in range(2):
        r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=S, max_iters=1, allow_diverged=True)
    st = r["stats"]
    sweeps = 2
    print(f"{name}: S={S} coarse {st['coarse_ms']:.2f} ms for {sweeps} sweeps -> {st['coarse_ms']/sweeps/S*1e3:.2f} us/slice, "
          f"{st['coarse_ms']/sweeps/S/(4)*1e3:.2f} us/stage; fine {st['fine_ms']:.2f} ms", flush=True)
