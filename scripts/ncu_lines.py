"""Per-CUDA-line totals (stall samples, instructions) from an ncu report's
source page (`ncu -i R --page source --csv --print-source cuda,sass`).
Usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
samples, instr, text = defaultdict(float), defaultdict(float), {}
cur = None
h = None
for r in rows:
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h) - 5:
        continue
    if r[0]:
        cur = int(r[0])
        text[cur] = r[1]
    if cur is None:
        continue
    try:
        samples[cur] += float(r[4] or 0)
        instr[cur] += float(r[7] or 0)
    except ValueError:
        pass
ts, ti = sum(samples.values()) or 1, sum(instr.values()) or 1
print(f"{'line':>5} {'samples':>8} {'instr':>7}  source")
for ln in sorted(samples, key=lambda k: -samples[k])[:top]:
    print(f"{ln:5d} {samples[ln] / ts:8.1%} {instr[ln] / ti:7.1%}  {text.get(ln, '').strip()[:90]}")
