"""cfg3 (10M x 10M Zipf) exact pair count through the one-call join plan, device-resident keys."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import pipeline, synth  # noqa: E402
torch.cuda.set_device(0)
r, s = synth.cfg3_relations()
dl, dr = torch.from_numpy(r.column("key").copy()).cuda(), torch.from_numpy(s.column("key").copy()).cuda()
ts = []
for r in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    plan = pipeline.plan_join(dl, dr)
    b.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(a.elapsed_time(b))
print(f"cfg3 total={plan.total} count_ms={statistics.median(ts):.3f}")
