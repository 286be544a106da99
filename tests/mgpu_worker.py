"""Worker of tests/test_multigpu.py (one rank per GPU, launched by torch.distributed.run).

Runs the C3 solve (BASELINE configs[2], 5 iterations) through the library with a real NCCL
communicator, under both schedules: bulk (each rank advances its shard of slices and its fine kernel
stores the endpoints into every peer's F — or, with RSW_ALLGATHER=1, an in-place ncclAllGather
exchanges them (a6) — and every rank runs the replicated coarse sweep) and the multi-GPU pipelined
one (replicated sweeps, each rank's fine tasks pushed into the peers' buffers).  Writes, per rank, a digest of U and the
residual history; rank 0 also writes the single-GPU (comm = None) bulk result and the sampled slices
the oracle fixture holds, for the test to compare."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1303_6615_b200 as rsw  # noqa: E402
from paper_1303_6615_b200 import inputs  # noqa: E402


def main(out_dir):
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    rsw.load()
    comm = rsw.Comm.from_torch_distributed()
    w = inputs.C3
    p = rsw.Params(w.eps, w.F, w.mu, w.n)
    u0 = torch.from_numpy(inputs.initial_state(w)).cuda()
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters)
    g = rsw.parareal_iterate(p, u0, comm=comm, schedule=rsw.SCHEDULE_BULK, **kw)
    U = g["U"].cpu().numpy()
    # the bulk schedule with the in-place NCCL all-gather instead of the fine kernel's peer stores
    os.environ["RSW_ALLGATHER"] = "1"
    ag = rsw.parareal_iterate(p, u0, comm=comm, schedule=rsw.SCHEDULE_BULK, **kw)
    del os.environ["RSW_ALLGATHER"]
    # the multi-GPU pipelined schedule: replicated sweeps, this rank's fine tasks, F pushed over NVLink
    q = rsw.parareal_iterate(p, u0, comm=comm, schedule=rsw.SCHEDULE_PIPELINED, **kw)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=U, resid=np.array(g["resid"]), iters=g["iters"],
             comm_ms=g["stats"]["comm_ms"], fine_steps=g["stats"]["fine_slice_steps"],
             Upipe=q["U"].cpu().numpy(), resid_pipe=np.array(q["resid"]), pipelined=q["stats"]["pipelined"],
             fine_steps_pipe=q["stats"]["fine_slice_steps"], Uag=ag["U"].cpu().numpy())
    if rank == 0:
        s = rsw.parareal_iterate(p, u0, schedule=rsw.SCHEDULE_BULK, **kw)
        np.savez(os.path.join(out_dir, "single.npz"), U=s["U"].cpu().numpy(), resid=np.array(s["resid"]))
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
