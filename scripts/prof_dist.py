"""Stage timing of one dist.distributed_sort step (one-rank NCCL group)."""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import dist as D  # noqa: E402
from paper_2602_21237_b200 import synth  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29611")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
rel = synth.cfg2_relation(10_000_000)
keys = torch.from_numpy(rel.column("key").copy()).cuda()
pay = torch.from_numpy(rel.column("payload").copy()).cuda()
ops = D.GpuOps()
stamps = {}


def mark(name):
    torch.cuda.synchronize()
    stamps[name] = time.perf_counter()


for rep in range(4):
    mark("start")
    sk, sg, bases = D.choose_splitters(keys, 0, False, with_bases=True)
    mark("splitters")
    rows, counts, moved = D._partition_take(ops, "range", keys, [keys, pay], gid_base=0, split_keys=sk,
                                            split_gids=sg, descending=False)
    mark("partition")
    recv, rc = D.exchange(moved + [rows], counts, None, with_counts=True)
    mark("exchange")
    g = D._global_ids(recv[-1], rc, bases)
    mark("gids")
    out = D._sort_take(ops, list(recv[:-1]) + [g], 0, False)
    mark("sort_take")
names = list(stamps)
print(" ".join(f"{b}={1e3 * (stamps[b] - stamps[a]):.3f}ms" for a, b in zip(names, names[1:])))
dist.destroy_process_group()
