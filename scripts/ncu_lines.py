"""Per-CUDA-line totals (stall samples, instructions, shared-memory bank-conflict
wavefronts) from an ncu report's source page (`ncu -i R --page source --csv
--print-source cuda,sass`), keyed by (file, line).
Usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
samples, instr, confl, text = defaultdict(float), defaultdict(float), defaultdict(float), {}
cur = None
h = None
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = os.path.basename(r[1])
        h = None
        continue
    if r and r[0] == "Line No":
        h = r
        ci = h.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in h else None
        continue
    if h is None or len(r) < len(h) - 5:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        text[cur] = r[1]
    if cur is None:
        continue
    try:
        samples[cur] += float(r[4] or 0)
        instr[cur] += float(r[7] or 0)
        if ci is not None and r[0]:
            confl[cur] += float(r[ci] or 0)
    except ValueError:
        pass
ts, ti = sum(samples.values()) or 1, sum(instr.values()) or 1
tc = sum(confl.values()) or 1
print(f"{'file:line':>22} {'samples':>8} {'instr':>7} {'smem_x':>7}  source")
for k in sorted(samples, key=lambda k: -samples[k])[:top]:
    print(f"{k[0][:15]:>16}:{k[1]:<5d} {samples[k] / ts:8.1%} {instr[k] / ti:7.1%} {confl[k] / tc:7.1%}  "
          f"{text.get(k, '').strip()[:80]}")
