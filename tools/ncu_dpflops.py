"""Executed fp64 work of each kernel in an ncu --set full report: DADD, DMUL, DFMA thread
instructions and DP flops (DADD + DMUL + 2 DFMA), from the per-cycle SASS counters times the elapsed
cycles.  Usage: python tools/ncu_dpflops.py rep.ncu-rep [units_per_launch]"""
import csv
import io
import json
import subprocess
import sys


def dp_counts(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    unit = dict(zip(head, units))
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}
    hz = {"hz": 1.0, "khz": 1e3, "mhz": 1e6, "ghz": 1e9, "cycle/second": 1.0, "cycle/nsecond": 1e9,
          "cycle/usecond": 1e6, "cycle/msecond": 1e3}
    out = []
    for v in data:
        d = dict(zip(head, v))
        f = lambda k: float(d[k].replace(",", ""))
        dur_s = f("gpu__time_duration.sum") * scale[unit["gpu__time_duration.sum"].lower()]
        clk = f("smsp__cycles_elapsed.avg.per_second") * hz[unit["smsp__cycles_elapsed.avg.per_second"].lower()]
        cycles = dur_s * clk
        c = {op: f(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cycles
             for op in ("dadd", "dmul", "dfma")}
        c["flops"] = c["dadd"] + c["dmul"] + 2 * c["dfma"]
        c["kernel"] = d["Kernel Name"][:80]
        c["duration_ms"] = dur_s * 1e3
        out.append(c)
    return out


if __name__ == "__main__":
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    for c in dp_counts(sys.argv[1]):
        c["flops_per_unit"] = c["flops"] / units
        print(json.dumps(c))
