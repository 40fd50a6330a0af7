"""Probe: where cfg2's step time goes besides the sort kernels — the payload
gather by the permutation, cold (L2 flushed) vs with the payload already in
L2, and the sort alone. Usage: python scripts/gather_probe.py [reps]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rel = synth.cfg2_relation(10_000_000)
    keys = torch.from_numpy(rel.column("key").copy()).cuda()
    pay = torch.from_numpy(rel.column("payload").copy()).cuda()
    n = keys.numel()
    out = torch.empty_like(pay)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sk = torch.empty_like(keys)
    perm = engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk)
    col = [engine.OutColumn(pay, out, 4, 0)]

    def t(fn, pre):
        ms = []
        for _ in range(reps):
            pre()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ms)

    cold = t(lambda: engine.gather_rows(perm, col), lambda: flush.zero_())
    warm_pay = t(lambda: engine.gather_rows(perm, col), lambda: (flush.zero_(), pay.sum()))
    sort_only = t(lambda: engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk),
                  lambda: flush.zero_())
    both = t(lambda: (engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk),
                      engine.gather_rows(perm, col)), lambda: flush.zero_())
    print(f"gather cold {cold:.1f} us, payload in L2 {warm_pay:.1f} us; sort {sort_only:.1f} us, sort + gather {both:.1f} us")


if __name__ == "__main__":
    main()
