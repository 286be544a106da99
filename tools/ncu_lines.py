"""Warp-stall samples of an ncu report aggregated by CUDA source line (needs -lineinfo and
--import-source).  Usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=45):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    cur, hdr, agg, tot = None, None, {}, 0.0
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5 or r[0] == "":
            continue
        key = (cur, int(r[0]), r[1].strip()[:80])
        s = f(r[4])
        agg[key] = agg.get(key, 0.0) + s
        tot += s
    print(f"total samples {tot:.0f}")
    byfile = {}
    for (fl, _, _), v in agg.items():
        byfile[fl] = byfile.get(fl, 0.0) + v
    print("by file:", ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(byfile.items(), key=lambda x: -x[1])))
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v / tot:6.2%} {k[0]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
