"""Pipelined vs bulk parareal schedule: bitwise comparison and timing (GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs

names = sys.argv[1:] or ["C1", "C2", "C3"]
rsw.load()
for name in names:
    w = inputs.WORKLOADS[name]
    p = rsw.Params(w.eps, w.F, w.mu, w.n)
    u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol,
              allow_diverged=True)
    out = {}
    for sched in (rsw.SCHEDULE_BULK, rsw.SCHEDULE_PIPELINED):
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = rsw.parareal_iterate(p, u0, schedule=sched, **kw)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        out[sched] = r
        print(f"{name} schedule={sched}: iters {r['iters']} wall {dt*1e3:.2f} ms total_ms {r['stats']['total_ms']:.2f} "
              f"pipelined={r['stats'].get('pipelined')} resid {['%.3e' % x for x in r['resid']]}", flush=True)
    a, b = out[rsw.SCHEDULE_BULK], out[rsw.SCHEDULE_PIPELINED]
    same = torch.equal(a["U"], b["U"]) and a["resid"] == b["resid"] and a["iters"] == b["iters"]
    print(f"{name}: bitwise identical: {same}; max |dU| = {(a['U'] - b['U']).abs().max().item():.3e}", flush=True)
