"""A/B: cfg2 sort with the payload gather fused into the sort kernel vs a separate gather launch."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, synth  # noqa: E402

rel = synth.cfg2_relation(10_000_000)
keys = torch.from_numpy(rel.column("key").copy()).cuda()
pay = torch.from_numpy(rel.column("payload").copy()).cuda()
n = keys.numel()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for fuse in (False, True, False, True):
    ts = []
    for r in range(13):
        flush.zero_()
        out = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
        sk = torch.empty(n, dtype=torch.int64, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        perm = engine.sort_permutation([engine.SortAxis(keys, False)], n, keys.device, sorted_keys_out=sk,
                                       gather=[engine.OutColumn(pay, out, 4, 0)], fuse_gather=fuse)
        b.record()
        b.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    p64 = perm.to(torch.int64) & 0xFFFFFFFF
    ok = bool((out == pay[p64]).all())
    print(f"fuse={fuse} median_ms={statistics.median(ts):.4f} ok={ok}")
