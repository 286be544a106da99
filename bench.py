#!/usr/bin/env python
"""bench.py — fp64 RSW fine slice-steps/s and parareal time-to-solution on B200 (BASELINE.json).

One bench "step" = one complete asymptotic-parareal solve of the workload (the k = 0 coarse sweep,
then `max_iters` iterations of: fine sweep on this rank's slices -> NCCL all-gather of the slice
endpoints -> serial coarse sweep with the fused parareal update -> residual), i.e. one pass of every
SURVEY.md §8(a) row, with u0 resident in HBM.  value = fine slice-steps of the whole job / time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl rsw|reference]
  (N > 1: launched by torch.distributed.run, one rank per GPU, NCCL)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1303_6615_b200 import inputs  # noqa: E402

METRIC = "fp64 RSW fine slice-steps/s and parareal time-to-solution"
UNIT = "slice-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--impl", default="rsw", choices=["rsw", "reference"])
    ap.add_argument("--fine-scheme", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5-iteration", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=0, help="oracle sample: steps per slice")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()),
                                   default=None)}


# ---------------------------------------------------------------------------------------------
def cpu_baseline(w, steps_per_slice: int = 0, target_s: float = 15.0):
    """The CPU oracle, as it stands, timed on this host's cores on a bounded sample of the workload:
    its ETDRK4 fine sweep (OpenMP over slices) on `cores` slices x `steps` fine steps, the step count
    calibrated so the sample takes about `target_s` seconds."""
    import numpy as np
    import oracle
    oracle.build()
    cores = oracle.num_threads()
    u0 = inputs.initial_state(w)
    u = np.repeat(u0[None], cores, axis=0)
    fixed = bool(steps_per_slice)  # an explicit sample size is run as given
    if not steps_per_slice:  # per-step cost from a 1-step and a 3-step call (the difference drops the table setup)
        t = []
        for k in (1, 3):
            t0 = time.perf_counter()
            oracle.fine_propagate(u, w.eps, w.F, w.mu, w.n, k * w.dt_eff, min(w.dt_eff * (1 + 1e-12), k * w.dt_eff), 0)
            t.append(time.perf_counter() - t0)
        per_step = max((t[1] - t[0]) / 2.0, 1e-6)
        steps_per_slice = max(1, int((target_s - t[0]) / per_step))
    steps = steps_per_slice
    for attempt in range(3):  # re-scale the sample until it takes about target_s (setup costs distort the estimate)
        dT = steps * w.dt_eff
        t0 = time.perf_counter()
        oracle.fine_propagate(u, w.eps, w.F, w.mu, w.n, dT, min(w.dt_eff * (1 + 1e-12), dT), 0)
        dt = time.perf_counter() - t0
        if fixed or dt >= 0.5 * target_s or attempt == 2:
            break
        steps = max(steps + 1, int(steps * target_s / max(dt, 1e-3)))
    return {"value": cores * steps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"oracle ETDRK4 fine sweep, {cores} slices x {steps} steps of {w.name} "
                      f"(n={w.n}), {dt:.1f} s wall"}


def bench_config(w, args, world, iters=None, pipelined=True):
    """The workload description shared by both arms' JSON lines."""
    return {"workload": w.name, "n": w.n, "slices": w.n_slices, "fine_steps_per_slice": w.m_fine,
            "dt_eff": w.dt_eff, "iterations": w.max_iters if iters is None else iters, "M": w.M, "T0": w.T0,
            "eps": w.eps, "fine_scheme": "ETDRK4" if args.fine_scheme == 0 else "Strang",
            "parallelism": ("1 GPU, pipelined parareal megakernel" if world == 1 else
                            (f"dp{world}: fine tasks sharded by slice over {world} GPUs, endpoints pushed to every peer over "
                             "NVLink (IPC), replicated pipelined coarse sweeps" if pipelined else
                             f"dp{world}: slices sharded over {world} GPUs, NCCL all-gather, replicated coarse sweep (bulk)")),
            "l2": "flushed (256 MB write) before every timed step"}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = inputs.WORKLOADS[args.config]
    vals = []
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(w, args.cpu_sample_steps, target_s=20.0)
        if i >= args.warmup:
            vals.append(b["value"])
    v = statistics.median(vals)
    b["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(bench_config(w, args, 1), parallelism="CPU oracle, OpenMP over slices on the host cores",
                           l2="n/a", note="oracle fine sweep sample"),
            "cpu_baseline": b, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch_cmd(argv: list[str], gpus: int, port: int) -> list[str] | None:
    """`bench.py --gpus N` started as a plain process (no WORLD_SIZE in the environment) re-executes
    itself under torch.distributed.run with N ranks on this node (one per GPU, rendezvous on
    127.0.0.1); None when no relaunch is needed (N = 1, or already a torchrun rank)."""
    if gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    cmd = relaunch_cmd(sys.argv[1:], args.gpus, _free_port())
    if cmd is not None:
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1303_6615_b200 as rsw

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = rsw.Comm.from_torch_distributed()
    rsw.load()
    w = inputs.WORKLOADS[args.config]
    p = rsw.Params(w.eps, w.F, w.mu, w.n)
    u0_host = torch.from_numpy(inputs.initial_state(w)).pin_memory()
    u0 = u0_host.cuda()
    U = torch.empty((w.n_slices + 1,) + w.state_shape, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2
    kw = dict(dT=w.dT, dt=w.dt, T0=w.T0, M=w.M, n_slices=w.n_slices, max_iters=w.max_iters, tol=w.tol,
              fine_scheme=args.fine_scheme, comm=comm, U=U)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the first call also builds the per-configuration tables (eigenbasis, phi-functions, phases,
    # weights) and the workspace: reported separately as one-time setup
    t_first = time.perf_counter()
    fallback = None
    try:
        res = rsw.parareal_iterate(p, u0, **kw)
    except rsw.RSWError as e:  # multi-GPU pipelined schedule unavailable here: the bulk schedule
        if world == 1:
            raise
        fallback = str(e)
        kw["schedule"] = rsw.SCHEDULE_BULK
        res = rsw.parareal_iterate(p, u0, **kw)
    torch.cuda.synchronize()
    first_ms = (time.perf_counter() - t_first) * 1e3
    for _ in range(max(args.warmup - 1, 0)):
        res = rsw.parareal_iterate(p, u0, **kw)
    barrier()

    # ---- timed region: K whole solves, device events on the launching (current) stream
    stream = torch.cuda.current_stream()
    per = []
    stats = []
    launches = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = rsw.parareal_iterate(p, u0, **kw)
            e1.record(stream)
            e1.synchronize()
            per.append(e0.elapsed_time(e1))
            stats.append(res["stats"])
            launches += res["stats"]["kernel_launches"]
        barrier()
    ms = statistics.median(per)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    iters = res["iters"]
    total_slice_steps = iters * w.n_slices * w.m_fine  # all ranks together
    value = total_slice_steps / (ms_max * 1e-3)

    # roofline of the dominant kernel of the timed region.  Pipelined schedule (1 GPU): ONE launch of
    # k_parareal_pipe per solve (coarse sweeps + fine solves); its algorithmic flops = the fine
    # slice-steps x F_step + every sweep's N-bar sample evaluations x F_sample.
    # Bulk schedule (N > 1): the fine kernel k_fine, one launch per iteration.
    pipelined = bool(stats[-1].get("pipelined"))
    f_step = rsw.flops_per_unit(w.n, "etdrk4" if args.fine_scheme == 0 else "strang")
    f_sample = rsw.flops_per_unit(w.n, "sample")
    nominal_peak = 148 * 64 * 2 * 1965e6 / 1e12  # FP64 FMA units x clock
    measured_peak = rsw.fp64_peak_tflops()
    local_slices = w.n_slices // world
    fine_flops_iter = local_slices * w.m_fine * f_step
    # averaged RK4: 4 N-bar per coarse step, each M-1 samples — or, in triad form, one
    # contraction with the triad coefficients
    triad = bool(stats[-1].get("coarse_triad"))
    f_nbar = rsw.flops_per_unit(w.n, "triad") if triad else (w.M - 1) * f_sample
    coarse_flops_sweep = w.n_slices * 4 * f_nbar
    if pipelined:
        step_flops = iters * fine_flops_iter + (iters + 1) * coarse_flops_sweep
        kern_ms = ms_max
        roof = {"bound": "alu", "kernel": "k_parareal_pipe (pipelined sweeps + fine solves, 1 launch/step)",
                "achieved": step_flops / (kern_ms * 1e-3) / 1e12, "flops_per_launch": step_flops,
                "flops_fine": iters * fine_flops_iter, "flops_coarse": (iters + 1) * coarse_flops_sweep,
                "coarse_form": "triad (DESIGN §6d)" if triad else "M-sample quadrature",
                "share_of_step": 1.0}
    else:
        fine_ms = statistics.median(s["fine_ms"] for s in stats) / max(iters, 1)   # per launch
        roof = {"bound": "alu", "kernel": "k_fine (ETDRK4 fine sweep)", "achieved": fine_flops_iter / (fine_ms * 1e-3) / 1e12,
                "flops_per_launch": fine_flops_iter,
                "share_of_step": statistics.median(s["fine_ms"] for s in stats) / ms_max}
    traffic = {}
    try:  # DRAM bytes per launch from the committed ncu capture of this same workload (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh)
    except (OSError, ValueError):
        pass

    def traffic_of(key):
        t = traffic.get(key)
        return None if not t else t["read"] + t["write"]

    dpf = {}
    try:  # executed DP flops per unit from the committed ncu captures (profiles/dp_flops.json)
        with open(os.path.join(ROOT, "profiles", "dp_flops.json")) as fh:
            dpf = json.load(fh)
    except (OSError, ValueError):
        pass

    def measured_flops(key, achieved_canonical, peak):
        """executed DP flops (ncu) beside the canonical count; when they fall more than
        10% below it, the measured rate is the headline fraction."""
        e = dpf.get(key)
        if not e:
            return {}
        ratio = e["measured"] / e["canonical"]
        return {"dp_flops_per_unit_measured": e["measured"], "dp_flops_per_unit_canonical": e["canonical"],
                "achieved_measured_flops": achieved_canonical * ratio, "frac_measured_flops": achieved_canonical * ratio / peak,
                "headline_frac": achieved_canonical * (ratio if ratio < 0.9 else 1.0) / peak,
                "headline_rule": "measured flops" if ratio < 0.9 else "canonical flops (measured within 10%)"}

    roof_traffic = traffic_of("k_parareal_pipe C3 5 iterations") if (pipelined and w.name == "C3" and iters == 5) else None
    roof.update({"peak": nominal_peak, "unit": "TFLOP/s", "frac": roof["achieved"] / nominal_peak, "traffic": roof_traffic,
                 "peak_source": "148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz",
                 "peak_measured_dfma": measured_peak, "frac_of_measured": roof["achieved"] / measured_peak})
    if pipelined and w.name == "C3" and iters == 5 and args.fine_scheme == 0:
        # per launch (the whole solve), so the ratio applies to the launch's canonical flops
        e = dpf.get("k_parareal_pipe C3 5 iterations per launch" + ("" if triad else " (quadrature sweeps)"))
        if e:
            dpf["_pipe"] = {"measured": e["measured"], "canonical": step_flops}
            roof.update(measured_flops("_pipe", roof["achieved"], nominal_peak))
    coarse_ms = statistics.median(s["coarse_ms"] for s in stats)
    comm_ms = statistics.median(s["comm_ms"] for s in stats)

    # the fine kernel alone on this rank's slices of the workload (same launch configuration as the
    # bulk schedule's fine sweep): CUDA events around each launch, L2 flushed before each
    uf = torch.from_numpy(inputs.random_states(w.n, local_slices, seed=0, kmax=32)).cuda()
    of = torch.empty_like(uf)
    fk = []
    for r in range(4):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rsw.fine_propagate(p, uf, w.dT, w.dt, args.fine_scheme, out=of, validate=(r == 0))  # layout checked once, outside the timed launches
        e1.record(stream)
        e1.synchronize()
        if r:
            fk.append(e0.elapsed_time(e1))
    fine_ms = statistics.median(fk)
    fine_tf = fine_flops_iter / (fine_ms * 1e-3) / 1e12
    roof_fine = {"bound": "alu", "kernel": "k_fine (ETDRK4 fine sweep, standalone)", "achieved": fine_tf,
                 "peak": nominal_peak, "unit": "TFLOP/s", "frac": fine_tf / nominal_peak, "traffic": None,
                 "frac_of_measured": fine_tf / measured_peak, "ms_per_launch": fine_ms,
                 "flops_per_launch": fine_flops_iter, "slices": local_slices, "steps": w.m_fine}
    if w.name == "C3" and args.fine_scheme == 0:
        roof_fine.update(measured_flops("k_fine C3 ETDRK4 per slice-step", fine_tf, nominal_peak))

    # ---- the fine sweep of the large configuration (C5, BASELINE configs[4]: 4096 slices, n = 1024,
    # 391 ETDRK4 steps), sharded over the ranks: the throughput-bound kernel whose scaling the north
    # star targets (the C3 time-to-solution above is bounded by the serial coarse chain).  Max over
    # ranks of the per-launch CUDA-event time, L2 flushed before each launch.
    w5 = inputs.C5
    p5 = rsw.Params(w5.eps, w5.F, w5.mu, w5.n)
    s5 = w5.n_slices // world
    u5 = torch.from_numpy(inputs.random_states(w5.n, s5, seed=rank, kmax=64)).cuda()
    o5 = torch.empty_like(u5)
    def c5_sweep(scheme):
        f5 = []
        for r in range(4):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rsw.fine_propagate(p5, u5, w5.dT, w5.dt, scheme, out=o5, validate=(r == 0))
            e1.record(stream)
            e1.synchronize()
            if r:
                f5.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(f5)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c5_ms = float(t.item())
        c5_tf = w5.n_slices * w5.m_fine * rsw.flops_per_unit(w5.n, "etdrk4" if scheme == 0 else "strang") \
            / (c5_ms * 1e-3) / 1e12
        extra = measured_flops("k_fine C5 ETDRK4 per slice-step", c5_tf / world, nominal_peak) if scheme == 0 else {}
        return {**extra, "workload": f"C5 fine sweep ({'ETDRK4' if scheme == 0 else 'Strang'}, n=1024, 391 steps)",
                "slices_total": w5.n_slices, "slices_per_rank": s5, "ms_max_over_ranks": c5_ms,
                "slice_steps_per_s": w5.n_slices * w5.m_fine / (c5_ms * 1e-3), "achieved_tflops": c5_tf,
                "frac": c5_tf / (nominal_peak * world), "frac_of_measured": c5_tf / (measured_peak * world),
                "kernel": "k_fine<1024,16,192,2> (two pair-groups per CTA, twiddles in TMEM)",
                "traffic": traffic_of("k_fine C5 4096 slices ETDRK4") if (scheme == 0 and world == 1) else None}

    fine_c5 = c5_sweep(0)
    fine_c5["strang"] = c5_sweep(1)  # BASELINE configs[4]: "Strang-splitting variant also run"
    del u5, o5

    # ---- the standalone averaged-nonlinearity batch (C4, BASELINE configs[3]: 4096 states, n = 512,
    # M = 256) sharded over the ranks ("on 1 GPU and sharded across 8"), max over ranks
    w4 = inputs.C4
    p4 = rsw.Params(w4.eps, w4.F, w4.mu, w4.n)
    s4 = 4096 // world
    u4 = torch.from_numpy(inputs.random_states(w4.n, s4, seed=100 + rank)).cuda()
    def time_c4():
        a4 = []
        for r in range(4):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rsw.averaged_rhs(p4, u4, w4.T0, w4.M, validate=(r == 0))
            e1.record(stream)
            e1.synchronize()
            if r:
                a4.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(a4)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # default: N-bar in triad form (the same quadrature sum, 108 flops per (kappa, kappa1) row);
    # beside it the per-sample pseudo-spectral kernel (RSW_COARSE_TRIAD=0), canonical flops per sample
    c4_ms = time_c4()
    c4_tf = 4096 * rsw.flops_per_unit(w4.n, "triad") / (c4_ms * 1e-3) / 1e12
    os.environ["RSW_COARSE_TRIAD"] = "0"
    try:
        c4q_ms = time_c4()
    finally:
        del os.environ["RSW_COARSE_TRIAD"]
    c4q_tf = 4096 * (w4.M - 1) * rsw.flops_per_unit(w4.n, "sample") / (c4q_ms * 1e-3) / 1e12
    avg_c4 = {"workload": "C4 averaged-nonlinearity batch (4096 states, n=512, M=256)", "states_total": 4096,
              "states_per_rank": s4, "ms_max_over_ranks": c4_ms, "form": "triad (DESIGN §6d)",
              "states_per_s": 4096 / (c4_ms * 1e-3), "sample_evals_per_s": 4096 * (w4.M - 1) / (c4_ms * 1e-3),
              "achieved_tflops": c4_tf, "flops_per_state": rsw.flops_per_unit(w4.n, "triad"),
              "frac": c4_tf / (nominal_peak * world), "frac_of_measured": c4_tf / (measured_peak * world),
              "kernel": "k_avg_triad<512,4,256> (coefficients streamed from L2, 4 states per CTA)",
              **measured_flops("k_avg_triad C4 per state", c4_tf / world, nominal_peak),
              "speedup_vs_quadrature": c4q_ms / c4_ms,
              "quadrature": {"ms_max_over_ranks": c4q_ms, "achieved_tflops": c4q_tf,
                             "flops_per_state": (w4.M - 1) * rsw.flops_per_unit(w4.n, "sample"),
                             "frac": c4q_tf / (nominal_peak * world), "frac_of_measured": c4q_tf / (measured_peak * world),
                             "kernel": "k_avg_states<512,8,192> (state, accumulator and twiddles in TMEM)",
                             **measured_flops("k_avg_states C4 per sample-eval", c4q_tf / world, nominal_peak)}}
    del u4

    # ---- C5 (BASELINE configs[4]) time per parareal iteration at this rank count (bulk schedule: the
    # pipelined megakernel supports n <= 256): the k = 0 coarse sweep (16384 serial stages at n = 1024),
    # then one iteration = fine sweep of this rank's slices + all-gather + coarse sweep.  One iteration
    # only: the C5 iterate blows up at k = 2 (docs/c5_stability.json).
    c5_iteration = None
    if not args.no_c5_iteration:
        U5 = torch.empty((w5.n_slices + 1,) + w5.state_shape, dtype=torch.float64, device="cuda")
        u50 = torch.from_numpy(inputs.initial_state(w5)).cuda()
        # warm-up on a 2-slice prefix: the same kernels (module load on first launch), tables and workspace
        rsw.parareal_iterate(p5, u50, dT=w5.dT, dt=w5.dt, T0=w5.T0, M=w5.M, n_slices=2 * world, max_iters=1,
                             comm=comm, allow_diverged=True, schedule=rsw.SCHEDULE_BULK)
        barrier()
        r5 = rsw.parareal_iterate(p5, u50, dT=w5.dT, dt=w5.dt, T0=w5.T0, M=w5.M, n_slices=w5.n_slices, max_iters=1,
                                  comm=comm, U=U5, allow_diverged=True, schedule=rsw.SCHEDULE_BULK)
        s5 = r5["stats"]
        tt = torch.tensor([s5["total_ms"], s5["sweep0_ms"], s5["fine_ms"], s5["comm_ms"], s5["coarse_ms"] - s5["sweep0_ms"]],
                          dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tt = tt.tolist()
        c5_iteration = {"workload": "C5 parareal, k = 0 sweep + 1 iteration (bulk schedule)", "slices": w5.n_slices,
                        "total_ms": tt[0], "sweep0_ms": tt[1], "fine_sweep_ms": tt[2], "allgather_ms": tt[3],
                        "coarse_sweep_ms": tt[4], "coarse_stages_per_sweep": 4 * w5.n_slices,
                        "us_per_coarse_stage": tt[4] * 1e3 / (4 * w5.n_slices), "r_1": r5["resid"],
                        "status": r5["status"]}
        del U5

    # ---- e2e: same solve through the C-ABI from pinned host buffers, H2D + D2H inside the region
    U_host = torch.empty(U.shape, dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(max(1, args.steps)):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        u0d = u0_host.to("cuda", non_blocking=True)
        rsw.parareal_iterate(p, u0d, **kw)
        U_host.copy_(U, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1))
    t = torch.tensor([statistics.median(e2e)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(w, args, world, iters, pipelined),
            "schedule_fallback": fallback,
            "time_to_solution_ms": ms_max,
            "setup_ms": {"first_call_wall": first_ms, "steady_call": ms_max,
                         "one_time_setup_estimate": max(first_ms - ms_max, 0.0)},
            "schedule": "pipelined (one persistent launch per solve)" if pipelined else "bulk (fine sweep + coarse sweep per iteration)",
            "phases_ms": ({"pipelined_total": statistics.median(s["total_ms"] for s in stats),
                           "sweep0": statistics.median(s["sweep0_ms"] for s in stats),
                           "per_further_iteration": statistics.median(s["lag_ms"] for s in stats),
                           "fine_task_latency": statistics.median(s["fine_task_ms"] for s in stats),
                           "layout": {"coarse_groups": stats[-1]["coarse_groups"], "ctas_per_group": stats[-1]["group_ctas"],
                                      "die_aware": stats[-1]["die_aware"], "die_sms": rsw.device_topology()["die_sms"]},
                           "note": "k = 0 coarse sweep (2048 serial stages) + iterations x the lag each adds "
                                   "(one fine pair task + hand-off); in-kernel globaltimer stamps"} if pipelined else
                          {"fine": statistics.median(s["fine_ms"] for s in stats), "allgather": comm_ms,
                           "coarse": coarse_ms, "sweep0": statistics.median(s["sweep0_ms"] for s in stats),
                           "per_iteration": statistics.median(s["lag_ms"] for s in stats),
                           "total_library": statistics.median(s["total_ms"] for s in stats)}),
            "convergence": {"iterations": iters, "rule": "fixed count (BASELINE configs[2]: 5 iterations)",
                            "resid": res["resid"],
                            "converged": bool(res["resid"] and res["resid"][-1] < 1e-6),
                            "note": "time to 5 fixed iterations; the C3 iteration has not converged by k = 5"},
            "fine_kernel_slice_steps_per_s": local_slices * w.m_fine / (fine_ms * 1e-3) * world,
            "roofline": roof,
            "roofline_fine": roof_fine,
            "fine_c5": fine_c5,
            "avg_c4": avg_c4,
            "c5_iteration": c5_iteration,
            "clocks": clk.summary(),
            "e2e": {"value": total_slice_steps / (e2e_ms * 1e-3), "unit": UNIT, "ms": e2e_ms,
                    "h2d_bytes_per_step": u0_host.numel() * 8, "d2h_bytes_per_step": U_host.numel() * 8},
            "gpu_launches": launches,
            "resid": res["resid"],
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(w, args.cpu_sample_steps)
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
