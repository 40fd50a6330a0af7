"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum[,dram__bytes_*]) per kernel:
launches, average duration, share of GPU time, DRAM MB read/written per launch.
Usage: python scripts/launch_summary.py launches.csv > launches.txt"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = defaultdict(dict)
    for r in rows[1:]:
        per[(r[ii], r[ki])][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
             "Gbyte": 1e3}
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("rl::", "")[:60]
        a = agg[short]
        a[0] += 1
        t, u = m.get("gpu__time_duration.sum", (0.0, "ns"))
        a[1] += t * scale.get(u, 1.0)
        for j, key in ((2, "dram__bytes_read.sum"), (3, "dram__bytes_write.sum")):
            if key in m:
                a[j] += m[key][0] * scale.get(m[key][1], 1.0)
    total = sum(a[1] for a in agg.values())
    print(f"{'kernel':60s} launches    avg_us  share MB_rd/launch MB_wr/launch")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:60s} {a[0]:8d} {a[1] / a[0]:9.1f} {100 * a[1] / total:5.1f}% {a[2] / a[0]:12.1f} {a[3] / a[0]:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
