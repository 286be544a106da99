"""Write the oracle fixtures used by the full-size GPU parity tests.  Calls ONLY oracle/ (and the
seeded input generators); no value here comes from the CUDA path.

  python tests/golden/make_oracle_fixtures.py [C2] [C3] [C5P]

C2  : the whole C2 solve with tol 1e-6 (iteration count, residual history, final U).
C3  : the whole C3 solve (5 iterations): residual history, final U at every 8th slice and the last.
C5P : the first 8 slices of C5 as a self-contained parareal problem (U^k_n for n <= 8 depends only
      on slices < n), k = 1, 2: the prefix of the full 4096-slice run.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def run(w, S=None, max_iters=None, tol=None):
    u0 = inputs.initial_state(w)
    return oracle.parareal(u0, w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                           n_slices=S or w.n_slices, max_iters=w.max_iters if max_iters is None else max_iters,
                           tol=w.tol if tol is None else tol)


def main(which):
    if "C2" in which:
        t = time.time()
        r = run(inputs.C2)
        np.savez_compressed(os.path.join(OUT, "oracle_C2.npz"), U=r["U"], resid=r["resid"], iters=r["iters"])
        print("C2", r["iters"], r["resid"], f"{time.time() - t:.0f}s", flush=True)
    if "C3" in which:
        t = time.time()
        r = run(inputs.C3)
        idx = np.unique(np.r_[np.arange(0, 513, 8), 512])
        np.savez_compressed(os.path.join(OUT, "oracle_C3.npz"), idx=idx, U=r["U"][idx], resid=r["resid"],
                            iters=r["iters"])
        print("C3", r["iters"], r["resid"], f"{time.time() - t:.0f}s", flush=True)
    if "C5P" in which:
        t = time.time()
        out = {}
        for k in (1, 2):
            r = run(inputs.C5, S=8, max_iters=k, tol=0.0)
            out[f"U{k}"] = r["U"]
        np.savez_compressed(os.path.join(OUT, "oracle_C5_prefix8.npz"), **out)
        print("C5P", f"{time.time() - t:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C5P"])
