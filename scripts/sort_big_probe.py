"""Probe: one index sort (rl_sort_axis, positions + sorted keys) of n uniform
keys in [0, n) from torch.randint, for an ncu launch list.
Usage: python scripts/sort_big_probe.py n [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import engine


def main():
    n = int(float(sys.argv[1]))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    g = torch.Generator(device="cuda").manual_seed(n)
    dom = int(float(os.environ.get("PROBE_DOMAIN", n)))
    keys = torch.randint(0, dom, (n,), generator=g, device="cuda", dtype=torch.int64)
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        engine.index_keys(keys)
        b.record()
        b.synchronize()
        print(f"index_keys n={n:.0e}: {a.elapsed_time(b):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
