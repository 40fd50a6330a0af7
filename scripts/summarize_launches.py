"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in data:
    per.setdefault(r[0], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.OrderedDict()
for rec in per.values():
    name = rec["kernel"].split("(")[0].replace("void ", "")[:60]
    a = agg.setdefault(name, {"launches": 0, "time_ns": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    a["launches"] += 1
    a["time_ns"] += rec.get("gpu__time_duration.sum", 0)
    a["dram_read"] += rec.get("dram__bytes_read.sum", 0)
    a["dram_write"] += rec.get("dram__bytes_write.sum", 0)
tot = sum(a["time_ns"] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'avg_us':>9s} {'share':>6s} {'MB_rd/launch':>12s} {'MB_wr/launch':>12s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["time_ns"]):
    n = a["launches"]
    print(f"{k:60s} {n:8d} {a['time_ns']/n/1e3:9.1f} {a['time_ns']/tot:6.1%} {a['dram_read']/n/1e6:12.1f} {a['dram_write']/n/1e6:12.1f}")
