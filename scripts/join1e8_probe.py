"""The 1e8 x 1e8 device join of bench.py's join_scaling (N=1): a few steps, for a launch list."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import pipeline, records as R, synth  # noqa: E402

n = 100_000_000
torch.cuda.set_device(0)
import os  # noqa: E402
if os.environ.get("L2FETCH"):  # experiment: L2 fetch granularity (bytes) for the random payload gathers
    from cuda.bindings import runtime as rt
    torch.zeros(1, device="cuda")  # primary context up
    lim = rt.cudaLimit.cudaLimitMaxL2FetchGranularity
    print("L2 fetch granularity before", rt.cudaDeviceGetLimit(lim), "set", rt.cudaDeviceSetLimit(lim, int(os.environ["L2FETCH"])),
          "after", rt.cudaDeviceGetLimit(lim))
cols_l = [torch.from_numpy(synth.uniform_keys(n, n, 0)).cuda(), torch.arange(n, dtype=torch.int64, device="cuda")]
cols_r = [torch.from_numpy(synth.uniform_keys(n, n, 1)).cuda(), torch.arange(n, dtype=torch.int64, device="cuda")]
schema = R.Schema((("key", R.Int64()), ("payload", R.Int64())))
dl, dr = pipeline.DeviceRelation(schema, cols_l), pipeline.DeviceRelation(schema, cols_r)
import statistics  # noqa: E402

ts = []
for r in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rows = pipeline.join(dl, dr, "key").row_count
    b.record()
    b.synchronize()
    if r >= 2:
        ts.append(a.elapsed_time(b))
print(f"rows={rows} join_ms={statistics.median(ts):.3f}")
