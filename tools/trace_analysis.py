"""Offline analysis of a pipelined solve's raw timeline (RSW_PIPE_TRACE=1 RSW_PIPE_TRACE_DUMP=file):
per sweep the slice rate over time, per iteration the fine tasks' queue wait (claim time minus the
time their input slices were finalized) and duration."""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
K, S, npairs, ntr0 = np.frombuffer(raw[:16], dtype=np.int32)
tr = np.frombuffer(raw[16:], dtype=np.uint64).astype(np.float64)
t0 = tr[0]
ms = lambda x: (x - t0) * 1e-6  # noqa: E731
sweep = tr[: 2 * (K + 1)].reshape(K + 1, 2)
sl = tr[2 * (K + 1): 2 * (K + 1) + (K + 1) * S].reshape(K + 1, S)
fine = tr[2 * (K + 1) + (K + 1) * S: 2 * (K + 1) + (K + 1) * S + 2 * max(K, 1) * npairs].reshape(max(K, 1), npairs, 2)
print(f"K={K} S={S} pairs={npairs}")
edges = np.arange(0, 40, 4.0)
print("slice rate (us/slice) of each sweep per 4 ms window:", " ".join(f"{e:.0f}" for e in edges))
for k in range(K + 1):
    t = ms(sl[k])
    row = []
    for a, b in zip(edges[:-1], edges[1:]):
        m = (t >= a) & (t < b)
        row.append(f"{(b - a) * 1e3 / m.sum():5.1f}" if m.sum() > 1 else "   - ")
    print(f"  sweep {k}: " + " ".join(row))
for k in range(K):
    ready = ms(sl[k][np.minimum(2 * np.arange(npairs) + 1, S - 1) - 1 + 1 - 1])  # slice 2p+1 finalized = U_{2p+2}?
    st, en = ms(fine[k, :, 0]), ms(fine[k, :, 1])
    # the task (k, p) is ready when slice 2p (U^k_{2p+1} written) is finalized: sl[k][2p]
    rdy = ms(sl[k][np.minimum(2 * np.arange(npairs), S - 1)])
    wait = st - rdy
    print(f"iteration {k}: queue wait mean {wait.mean():.3f} ms, max {wait.max():.3f}, p90 {np.percentile(wait, 90):.3f}; "
          f"duration mean {(en - st).mean():.3f} ms; first task start {st[0]:.3f} (ready {rdy[0]:.3f})")
