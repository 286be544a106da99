"""a6 / §8(e) on real GPUs: two ranks (torch.distributed.run, NCCL) run the C3 solve through
parareal_iterate with a library communicator.  U must be bitwise identical across ranks (replicated,
deterministic coarse sweep) and to the single-GPU bulk schedule, and match the oracle's full C3 run.
Skipped on fewer than 2 GPUs (the driver's round-end box has one; a multi-GPU node runs it)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1303_6615_b200 import inputs
from tests.helpers import rel_l2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_two_rank_nccl_c3_bitwise(rsw_gpu, tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}",
                        os.path.join(ROOT, "tests", "mgpu_worker.py"), str(tmp_path)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    r0, r1, single = (np.load(tmp_path / f) for f in ("rank0.npz", "rank1.npz", "single.npz"))
    assert np.array_equal(r0["U"], r1["U"]) and np.array_equal(r0["resid"], r1["resid"])
    assert np.array_equal(r0["U"], single["U"]) and np.array_equal(r0["resid"], single["resid"])
    assert np.array_equal(r0["Uag"], single["U"]) and np.array_equal(r1["Uag"], single["U"])  # all-gather path
    for r in (r0, r1):  # multi-GPU pipelined schedule: bitwise the single-GPU result on every rank
        assert bool(r["pipelined"])
        assert np.array_equal(r["Upipe"], single["U"]) and np.array_equal(r["resid_pipe"], single["resid"])
    w3 = inputs.C3
    assert int(r0["fine_steps_pipe"]) == w3.max_iters * (w3.n_slices // 2) * w3.m_fine
    w = inputs.C3
    assert int(r0["fine_steps"]) == w.max_iters * (w.n_slices // 2) * w.m_fine  # each rank ran its shard only
    ref = np.load(os.path.join(ROOT, "tests", "golden", "oracle_C3.npz"))
    assert int(r0["iters"]) == int(ref["iters"])
    assert np.allclose(r0["resid"], ref["resid"], rtol=1e-8, atol=0)
    assert rel_l2(r0["U"][ref["idx"]], ref["U"], w.n)[1:].max() < 1e-10
