"""distributed_join at world 1 vs the direct device join (pipeline.join), N rows per side."""
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import dist as D  # noqa: E402
from paper_2602_21237_b200 import pipeline, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29612")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
r, s = synth.cfg1_relations(n=n, domain=n)
dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)


def timed(fn, reps=5):
    ts = []
    for i in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


t_direct = timed(lambda: pipeline.join(dr, ds, "key"))
t_dist = timed(lambda: D.distributed_join(dr.columns, 0, 0, ds.columns, 0, 0))
res = D.distributed_join(dr.columns, 0, 0, ds.columns, 0, 0)
print(f"n={n} direct_join_ms={t_direct:.3f} distributed_join_ms(world 1)={t_dist:.3f} matches={res.total_matches}")
dist.destroy_process_group()
