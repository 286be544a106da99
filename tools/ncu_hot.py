"""Top SASS instructions of an ncu report by warp-stall samples (needs -lineinfo + --import-source).
Usage: python tools/ncu_hot.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
    S = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[S] or 0) for d in data)
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    # aggregate by opcode
    byop = {}
    for d in data:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        op = op.split(".")[0]
        byop[op] = byop.get(op, 0) + float(d[S] or 0)
    print(f"total samples {tot:.0f}")
    print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(byop.items(), key=lambda x: -x[1])[:15]))
    data.sort(key=lambda d: -float(d[S] or 0))
    for d in data[:top]:
        st = sorted(((c[6:], float(d[c] or 0)) for c in stall_cols), key=lambda x: -x[1])[:3]
        print(f"{d['Address']:>6} {float(d[S] or 0) / tot:6.2%}  {d['Source'][:60]:60s} "
              + " ".join(f"{k}:{v:.0f}" for k, v in st if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
