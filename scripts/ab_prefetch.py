"""A/B: cfg2 sort + separate payload gather, with and without L2 prefetch of the
payload rows issued by the sort's local phase (library built with
-DRL_GATHER_PREFETCH_ONLY: the fused-gather hook only prefetches)."""
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
for prefetch in (False, True, False, True):
    ts, tg = [], []
    for r in range(13):
        flush.zero_()
        out = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
        sk = torch.empty(n, dtype=torch.int64, device="cuda")
        a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        col = engine.OutColumn(pay, out, 4, 0)
        a.record()
        perm = engine.sort_permutation([engine.SortAxis(keys, False)], n, keys.device, sorted_keys_out=sk,
                                       gather=[col] if prefetch else (), fuse_gather=prefetch)
        m.record()
        engine.gather_rows(perm, [col])
        b.record()
        b.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
            tg.append(m.elapsed_time(b))
    p64 = perm.to(torch.int64) & 0xFFFFFFFF
    ok = bool((out == pay[p64]).all())
    print(f"prefetch={prefetch} total_ms={statistics.median(ts):.4f} gather_ms={statistics.median(tg):.4f} ok={ok}")
