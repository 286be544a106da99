"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: launches, total,
mean, share of the captured time.  Usage: python tools/launch_summary.py launches.csv [title]"""
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg = {}
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]])
    tot = sum(sum(v) for v in agg.values())
    print(title)
    print("kernel, launches, total_ms, mean_ms, share")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k}, {len(v)}, {sum(v):.3f}, {sum(v) / len(v):.4f}, {sum(v) / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
