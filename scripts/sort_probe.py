"""Probe: cfg2-shaped sorts (10M full-range keys, ~1% duplicates) through
rl_sort_axis, for ncu captures of one kernel. Usage: python scripts/sort_probe.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import engine, synth


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    rel = synth.cfg2_relation(10_000_000)
    keys = torch.from_numpy(rel.column("key").copy()).cuda()
    n = keys.numel()
    sk = torch.empty_like(keys)
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk)
        b.record()
        b.synchronize()
        print(f"sort {a.elapsed_time(b):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
