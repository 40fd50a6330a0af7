"""Short driver for ncu: cfg2-shaped sort (and optionally the cfg1 join) a few
times on cuda:0. Usage: python scripts/prof_sort.py [--n ROWS] [--reps R] [--join]"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2602_21237_b200 import engine, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--join", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    if a.join:
        r, s = synth.cfg1_relations()
        rk = torch.from_numpy(r.column("key").copy()).cuda()
        sk = torch.from_numpy(s.column("key").copy()).cuda()
        rp = torch.from_numpy(r.column("payload").copy()).cuda()
        sp = torch.from_numpy(s.column("payload").copy()).cuda()
        for _ in range(a.reps):
            li, ri = engine.index_keys(rk), engine.index_keys(sk)
            al = engine.align(li, ri)
            m, total = engine.fetch_scalars(al.m_total)
            cols = [engine.OutColumn(None, torch.empty(total, dtype=torch.int64, device="cuda"), 8, 2),
                    engine.OutColumn(rp, torch.empty(total, dtype=torch.int64, device="cuda"), 8, 0),
                    engine.OutColumn(sp, torch.empty(total, dtype=torch.int64, device="cuda"), 8, 1)]
            engine.expand(al, m, li, ri, 0, total, cols)
        torch.cuda.synchronize()
        print("join ok", total)
        return
    rel = synth.cfg2_relation(a.n)
    keys = torch.from_numpy(rel.column("key").copy()).cuda()
    pay = torch.from_numpy(np.ascontiguousarray(rel.column("payload"))).cuda()
    for _ in range(a.reps):
        sk = torch.empty(a.n, dtype=torch.int64, device="cuda")
        perm = engine.sort_permutation([engine.SortAxis(keys)], a.n, keys.device, sorted_keys_out=sk)
        out = torch.empty((a.n, 4), dtype=torch.uint8, device="cuda")
        engine.gather_rows(perm, [engine.OutColumn(pay, out, 4, 0)])
    torch.cuda.synchronize()
    assert bool((sk[1:] >= sk[:-1]).all())
    print("sort ok")


if __name__ == "__main__":
    main()
