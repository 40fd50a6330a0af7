"""Probe: one cfg5-shaped join -> ORDER BY at n rows per side (device
relations from torch.randint), for an ncu launch list; plus random 8-byte
gathers at n rows (TLB reach). Usage: python scripts/pipe_probe.py n [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import SortSpec, engine, pipeline
from paper_2602_21237_b200 import records as R


def main():
    n = int(float(sys.argv[1]))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(n)
    lk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
    rk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
    pay = torch.arange(n, device=dev, dtype=torch.int64)
    schema = R.Schema((("key", R.Int64()), ("payload", R.Int64())))
    dl = pipeline.DeviceRelation(schema, [lk, pay])
    dr = pipeline.DeviceRelation(schema, [rk, pay])
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = pipeline.join_then_order_by(dl, dr, "key", SortSpec(("payload",)))
        b.record()
        b.synchronize()
        print(f"join->ORDER BY {a.elapsed_time(b):.2f} ms rows={out.row_count}", flush=True)
        del out
    del dl, dr, lk, rk
    torch.cuda.empty_cache()
    # random gathers: 8-byte rows at a random permutation (TLB / sector behaviour)
    perm = torch.randperm(n, device=dev, generator=g).to(torch.int32)
    dst = torch.empty_like(pay)
    for _ in range(max(reps, 2)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.gather_rows(perm, [engine.OutColumn(pay, dst, 8, 0)])
        b.record()
        b.synchronize()
        print(f"random gather 8 B x {n:.0e}: {a.elapsed_time(b):.2f} ms", flush=True)
    seq = torch.arange(n, device=dev, dtype=torch.int32)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    engine.gather_rows(seq, [engine.OutColumn(pay, dst, 8, 0)])
    b.record()
    b.synchronize()
    print(f"sequential gather 8 B x {n:.0e}: {a.elapsed_time(b):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
