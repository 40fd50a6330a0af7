"""Probe: index sorts, joins and join -> ORDER BY above the scatter hybrid's
167.8M-row cap (cfg5 shapes up to 1e9 rows per side), with a
torch.sort(stable=True) check of the index sort. Usage:
    python scripts/big_probe.py [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import SortSpec, engine, pipeline
from paper_2602_21237_b200 import records as R


def ev_time(fn, reps=3):
    ts = []
    res = None
    for _ in range(reps):
        res = None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return res, sorted(ts)[len(ts) // 2]


def main():
    sizes = [int(float(x)) for x in sys.argv[1:]] or [10**8, 2 * 10**8, 5 * 10**8, 10**9]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    for n in sizes:
        g.manual_seed(n)
        keys = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
        idx, ms = ev_time(lambda: engine.index_keys(keys))
        print(f"n={n:.0e} index_keys {ms:.2f} ms  ({n / ms / 1e3:.0f} Mrows/s)", flush=True)
        pos = idx.positions.to(torch.int64) & 0xFFFFFFFF
        ref = torch.sort(keys, stable=True)
        ok = bool((ref.indices == pos).all())
        print(f"  positions == torch.sort(stable) indices: {ok}", flush=True)
        del pos, ref, idx
        torch.cuda.empty_cache()
        pay = torch.arange(n, device=dev, dtype=torch.int64)
        rk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
        schema = R.Schema((("key", R.Int64()), ("payload", R.Int64())))
        dl = pipeline.DeviceRelation(schema, [keys, pay])
        dr = pipeline.DeviceRelation(schema, [rk, pay])
        try:
            out, ms = ev_time(lambda: pipeline.join(dl, dr, "key"), 2)
            print(f"  join {ms:.2f} ms rows_out={out.row_count} peak={torch.cuda.max_memory_allocated() / 2**30:.1f} GiB",
                  flush=True)
            del out
            torch.cuda.empty_cache()
            out, ms = ev_time(lambda: pipeline.join_then_order_by(dl, dr, "key", SortSpec(("payload",))), 2)
            print(f"  join->ORDER BY {ms:.2f} ms rows_out={out.row_count} "
                  f"peak={torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
            p = out.column("payload")
            print(f"  ORDER BY output sorted: {bool((p[1:] >= p[:-1]).all())}", flush=True)
            del out, p
        except Exception as e:
            print(f"  join failed: {e!r}"[:300], flush=True)
        del dl, dr, keys, rk, pay
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()


if __name__ == "__main__":
    main()
