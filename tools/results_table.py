"""BASELINE.md §4 rows on the GPU box: time-to-solution (pipelined and bulk), fine slice-steps/s, max
parity rel-L2 against the oracle (C1 run here, C2 / C3 from the committed oracle fixtures) and the
iteration counts.  Prints markdown rows.  Test/measurement tooling, not product."""
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402
from tests.helpers import rel_l2  # noqa: E402


def timed(p, u0, kw, sched, reps=5):
    rsw.parareal_iterate(p, u0, schedule=sched, **kw)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = rsw.parareal_iterate(p, u0, schedule=sched, **kw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return r, statistics.median(ts)


def main():
    rsw.load()
    oracle.build()
    for name in ("C1", "C2", "C3"):
        w = inputs.WORKLOADS[name]
        p = rsw.Params(w.eps, w.F, w.mu, w.n)
        u0h = inputs.initial_state(w)
        u0 = torch.from_numpy(u0h).cuda()
        kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol)
        rp, tp = timed(p, u0, kw, rsw.SCHEDULE_PIPELINED)
        rb, tb = timed(p, u0, kw, rsw.SCHEDULE_BULK, reps=3)
        assert torch.equal(rp["U"], rb["U"])
        U = rp["U"].cpu().numpy()
        if name == "C1":
            ref = oracle.parareal(u0h, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                                  n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol)
            err, it_ref, rref = rel_l2(U, ref["U"], w.n)[1:].max(), ref["iters"], np.array(ref["resid"])
        else:
            f = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz"))
            idx = f["idx"] if "idx" in f else np.arange(w.n_slices + 1)
            err, it_ref, rref = rel_l2(U[idx], f["U"], w.n)[1:].max(), int(f["iters"]), f["resid"]
        rerr = np.max(np.abs(np.array(rp["resid"]) - rref) / rref)
        steps = rp["iters"] * w.n_slices * w.m_fine
        print(f"| {name} | 1 | {steps / (tp * 1e-3):.3g} | — | — | {tp:.2f} ms pipelined ({tb:.2f} ms bulk) | "
              f"see cpu_baseline | U {err:.1e}, r_k {rerr:.1e} | {rp['iters']} / {it_ref} |", flush=True)


if __name__ == "__main__":
    main()
