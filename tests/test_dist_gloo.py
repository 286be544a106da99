"""The N > 1 path's host logic on CPU with world size 2 (gloo): the slice sharding of the C-ABI
(`rsw_shard_range`), the in-place all-gather layout of the fine endpoints, and the replicated,
deterministic serial sweep.  The per-slice compute is the oracle's (CPU); the driver below mirrors
parareal_iterate_ex (csrc/rsw_capi.cu): fine sweep on this rank's block -> all-gather of F (rank r's
block lands at offset lo_r) -> every rank runs the same coarse sweep U_{n+1} = G(U_n) + F_n - G_n
-> residual, no collective for the stop decision.  Both ranks must end with bitwise identical U,
equal to the single-process oracle parareal."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_parareal(rank, world, w, max_iters):
    import oracle
    import paper_1303_6615_b200 as rsw
    from paper_1303_6615_b200 import inputs
    from paper_1303_6615_b200 import build
    build.build()
    S, L = w.n_slices, 3 * (w.n // 2 + 1) * 2
    lo, hi = rsw.shard_range(S, rank, world)
    u0 = inputs.initial_state(w)
    kw = dict(eps=w.eps, F=w.F, mu=w.mu, n=w.n)
    U = np.zeros((S + 1,) + u0.shape)
    G = np.zeros((S,) + u0.shape)
    U[0] = u0
    for s in range(S):  # k = 0 sweep, replicated
        G[s] = oracle.coarse_propagate(U[s], dT=w.dT, T0=w.T0, M=w.M, **kw)
        U[s + 1] = G[s]
    resid = []
    for _ in range(max_iters):
        Fl = oracle.fine_propagate(np.ascontiguousarray(U[lo:hi]), dT=w.dT, dt=w.dt, **kw)
        F = torch.zeros(S * L, dtype=torch.float64)
        F[lo * L:hi * L] = torch.from_numpy(Fl.reshape(-1))
        parts = list(F.chunk(world))
        dist.all_gather(parts, parts[rank].clone())
        F = torch.cat(parts).numpy().reshape((S,) + u0.shape)
        Uold = U.copy()
        for s in range(S):
            g = oracle.coarse_propagate(U[s], dT=w.dT, T0=w.T0, M=w.M, **kw)
            U[s + 1] = g + (F[s] - G[s])
            G[s] = g
        wk = np.full(w.n // 2 + 1, 2.0)
        wk[0] = wk[-1] = 1.0
        num = (((U[1:] - Uold[1:]) ** 2) * wk[:, None]).sum(axis=(1, 2, 3))
        den = ((U[1:] ** 2) * wk[:, None]).sum(axis=(1, 2, 3))
        resid.append(float(np.sqrt(num / den).max()))
    return U, resid


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1303_6615_b200 import inputs
    U, resid = _sharded_parareal(rank, world, inputs.C1, 2)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=U, resid=np.array(resid))
    dist.destroy_process_group()


def test_sharded_parareal_gloo_world2(tmp_path, orc):
    import sys
    sys.path.insert(0, ROOT)
    from paper_1303_6615_b200 import inputs
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    assert np.array_equal(r0["U"], r1["U"])            # replicated sweep: bitwise identical ranks
    assert np.array_equal(r0["resid"], r1["resid"])
    w = inputs.C1
    ref = orc.parareal(inputs.initial_state(w), w.eps, w.F, w.mu, w.n, dT=w.dT, dt=w.dt, T0=w.T0, M=w.M,
                       n_slices=w.n_slices, max_iters=2)
    assert np.array_equal(r0["U"], ref["U"])            # equals the single-process iteration
    assert np.allclose(r0["resid"], ref["resid"], rtol=1e-12, atol=0)


def test_shard_ranges_partition(lib_rsw=None):
    import paper_1303_6615_b200 as rsw
    from paper_1303_6615_b200 import build
    build.build()
    for S, world in [(8, 1), (8, 2), (8, 8), (512, 4), (4096, 8)]:
        cover = []
        for r in range(world):
            lo, hi = rsw.shard_range(S, r, world)
            assert hi - lo == S // world
            cover.extend(range(lo, hi))
        assert cover == list(range(S))
