"""ncu driver: cfg3 streaming expansion (one 2^28-pair chunk) and the cfg1 expand."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, pipeline, synth  # noqa: E402
torch.cuda.set_device(0)
r3, s3 = synth.cfg3_relations()
p3 = pipeline.plan_join(torch.from_numpy(r3.column("key").copy()).cuda(), torch.from_numpy(s3.column("key").copy()).cuda())
lr = torch.empty(1 << 28, dtype=torch.int32, device="cuda"); rr = torch.empty_like(lr)
a0 = p3.total // 2
for _ in range(2):
    p3.expand(a0, a0 + (1 << 28), (), lr, rr)
r, s = synth.cfg1_relations()
dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
for _ in range(2):
    pipeline.join(dr, ds, "key")
torch.cuda.synchronize()
print("ok")
