"""Sweep-0 time of the C3 pipelined solve vs coarse layout and iteration count (is the pipelined stage
slow because of the fine tasks sharing the SMs, or because of the pipelined coarse code path?)."""
import os
import subprocess
import sys

code = r'''
import sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1303_6615_b200 as rsw
from paper_1303_6615_b200 import inputs
w = inputs.WORKLOADS["C3"]
p = rsw.Params(w.eps, w.F, w.mu, w.n)
u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
K = int(sys.argv[1])
rows = []
for rep in range(4):
    r = rsw.parareal_iterate(p, u0, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=K, tol=0.0,
                             allow_diverged=True, schedule=int(sys.argv[2]))
    s = r["stats"]
    rows.append((s["total_ms"], s.get("sweep0_ms", 0.0)))
m = np.median(np.array(rows), axis=0)
print("total %.2f sweep0 %.2f" % (m[0], m[1]))
'''
for K in (0, 1, 5):
    for sched, gc, ng in ((1, 0, 0), (2, 0, 0), (2, 64, 1), (2, 32, 1), (2, 24, 1)):
        if K == 5 and sched == 1:
            continue
        env = dict(os.environ)
        if gc:
            env.update(RSW_PIPE_GC=str(gc), RSW_PIPE_NG=str(ng if K == 0 else max(ng, 1)))
        r = subprocess.run([sys.executable, "-c", code, str(K), str(sched)], capture_output=True, text=True, env=env)
        print(f"K={K} schedule={'bulk' if sched == 1 else 'pipe'} GC={gc or 'auto'} NG={ng or 'auto'}:",
              r.stdout.strip() or r.stderr[-300:], flush=True)
