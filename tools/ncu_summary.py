"""Summarise an ncu --set full report (one row per profiled kernel) into the numbers DESIGN.md and
profiles/README.md quote: duration, FP64 pipe, DP op mix, issue, occupancy, smem, stall reasons,
DRAM traffic.  Usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep [> profiles/rNN_x.txt]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("kernel", "Kernel Name"),
    ("grid", "launch__grid_size"), ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"), ("smem_dyn_KB", "launch__shared_mem_per_block_dynamic"),
    ("duration_ms", "gpu__time_duration.sum"),
    ("sm_clock_GHz", "smsp__cycles_elapsed.avg.per_second"),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("dadd_per_clk_smsp", "smsp__sass_thread_inst_executed_op_dadd_pred_on.avg.per_cycle_elapsed"),
    ("dfma_per_clk_smsp", "smsp__sass_thread_inst_executed_op_dfma_pred_on.avg.per_cycle_elapsed"),
    ("dmul_per_clk_smsp", "smsp__sass_thread_inst_executed_op_dmul_pred_on.avg.per_cycle_elapsed"),
    ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("inst_executed", "smsp__inst_executed.sum"),
    ("local_ld", "smsp__sass_inst_executed_op_local_ld.sum"),
    ("dram_read_MB", "dram__bytes_read.sum"), ("dram_write_MB", "dram__bytes_write.sum"),
]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "wait", "mio_throttle", "math_pipe_throttle",
          "not_selected", "branch_resolving", "dispatch_stall", "lg_throttle", "no_instruction"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    for v in data:
        d = dict(zip(head, v))
        u = dict(zip(head, units))
        print(f"## {d.get('Kernel Name', '?')[:100]}")
        for name, k in KEYS[1:]:
            if k in d:
                print(f"{name:22s} {d[k]} {u.get(k, '')}")
        print("stalls per issue:", ", ".join(
            f"{s} {float(d[k]):.2f}" for s in STALLS
            if (k := f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") in d and d[k]))
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
