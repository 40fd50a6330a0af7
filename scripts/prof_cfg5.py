"""cfg5 join -> ORDER BY pipeline at N rows per side (device resident), for launch lists."""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import SortSpec, pipeline, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
torch.cuda.set_device(0)
r, s = synth.cfg1_relations(n=a.n, domain=a.n)
dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
del r, s
spec = SortSpec(("payload",))
for i in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    j = pipeline.join(dr, ds, "key")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    o = pipeline.order_by(j, spec)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {i}: join {1e3*(t1-t0):.2f} ms ({j.row_count} rows), order_by {1e3*(t2-t1):.2f} ms", flush=True)
