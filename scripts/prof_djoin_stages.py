"""Stage timing of one dist.distributed_join step (one-rank NCCL group), N rows per side."""
import os
import statistics
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import dist as D  # noqa: E402
from paper_2602_21237_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29613")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
r, s = synth.cfg1_relations(n=n, domain=n, seed=0)
L = [torch.from_numpy(c.copy()).cuda() for c in r.columns]
R = [torch.from_numpy(c.copy()).cuda() for c in s.columns]
ops = D.GpuOps()
res = {}


def t(name, f):
    torch.cuda.synchronize()
    a = time.perf_counter()
    out = f()
    torch.cuda.synchronize()
    res.setdefault(name, []).append(1e3 * (time.perf_counter() - a))
    return out


for rep in range(8):
    rows_l, cnt_l = t("hash_partition_L", lambda: ops.hash_partition(L[0], 1, D.PARTITION_SEED))
    rows_r, cnt_r = t("hash_partition_R", lambda: ops.hash_partition(R[0], 1, D.PARTITION_SEED))
    (pl, pr) = t("push_both", lambda: ops.push_exchange_many([("join_left", L, rows_l, cnt_l, 0),
                                                              ("join_right", R, rows_r, cnt_r, 0)], None))
    out = t("local_join", lambda: ops.local_join(pl[0], 0, pr[0], 0, pl[1], pr[1]))
    tot = torch.tensor([out[1].numel()], dtype=torch.int64, device="cuda")
    t("allreduce_total", lambda: (dist.all_reduce(tot), int(tot.item())))
    full = t("distributed_join", lambda: D.distributed_join(L, 0, 0, R, 0, 0))
print(" ".join(f"{k}={statistics.median(v[2:]):.3f}ms" for k, v in res.items()))
dist.destroy_process_group()
