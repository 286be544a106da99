"""bench.py's launch contract on CPU: `bench.py --gpus N` run as a plain process re-executes itself
under torch.distributed.run with N ranks (a driver-run `python bench.py --gpus 8` must
not silently run one rank)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_relaunch_cmd(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.relaunch_cmd(["--gpus", "1"], 1, 29500) is None
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "2"], 4, 29511)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29511" in cmd
    assert cmd[-5] == os.path.abspath(os.path.join(ROOT, "bench.py"))
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    monkeypatch.setenv("WORLD_SIZE", "4")  # already a torchrun rank: no second relaunch
    assert bench.relaunch_cmd(["--gpus", "4"], 4, 29500) is None


def test_gpus_2_relaunches_two_ranks_one_line():
    """End to end on CPU with the reference arm (the oracle): two torchrun ranks start, rank 0 alone
    prints ONE JSON line reporting n_gpus = 2, the other exits 0."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["OMP_NUM_THREADS"] = "2"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "C1", "--steps", "1", "--warmup", "0", "--cpu-sample-steps", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0


def test_runner_flags_override_the_preset():
    """`python -m paper_1303_6615_b200` (SURVEY §5 flags): a preset supplies every parameter, flags
    override single ones, and the initial state is projected onto the retained modes (CPU only)."""
    import numpy as np
    from paper_1303_6615_b200 import __main__ as cli
    from paper_1303_6615_b200 import inputs
    a = cli.parse_args(["--preset", "C3", "--modes", "64", "--slices", "16", "--T", "0.5", "--mbar", "16",
                        "--fine", "strang", "--coarse", "midpoint", "--max-iter", "2"])
    w = cli.workload_from_args(a)
    assert (w.n, w.n_slices, w.T, w.M, w.max_iters, w.fine_scheme, w.coarse_scheme) == (64, 16, 0.5, 16, 2, 1, 1)
    assert (w.eps, w.mu, w.T0) == (inputs.C3.eps, inputs.C3.mu, inputs.C3.T0)
    u0 = cli.initial_state(w, 0)
    assert u0.shape == (3, 33, 2) and not np.any(u0[:, 64 // 3 + 1:]) and not np.any(u0[:, 0, 1])
