"""Probe: cfg2's sort step with the 4-byte payload gathered after the sort vs
carried through the passes (idw words), same inputs: outputs compared, then
interleaved CUDA-event timings with an L2 flush between steps.
Usage: python scripts/idw_probe.py [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_21237_b200 import engine, synth


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rel = synth.cfg2_relation(n)
    dev = torch.device("cuda:0")
    keys = torch.from_numpy(rel.column("key").copy()).to(dev)
    pay = torch.from_numpy(np.ascontiguousarray(rel.column("payload")).view(np.int32).reshape(-1).copy()).to(dev)
    outs = {}
    graphs = {}
    for carry in (False, True):
        dst = torch.empty_like(pay)
        g = engine.SortGraph(keys, gather=[engine.OutColumn(pay, dst, 4, 0)], carry=carry)
        graphs[carry] = (g, dst)
        g.replay()
        torch.cuda.synchronize()
        outs[carry] = (g.sorted_keys.clone(), g.perm.clone(), dst.clone())
    same = all(torch.equal(a, b) for a, b in zip(outs[False], outs[True]))
    print(f"n={n} outputs equal: {same}", flush=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = {False: [], True: []}
    for r in range(reps + 3):
        for carry in (False, True):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graphs[carry][0].replay()
            b.record()
            b.synchronize()
            if r >= 3:
                times[carry].append(a.elapsed_time(b))
    for carry in (False, True):
        t = sorted(times[carry])
        print(f"{'carry' if carry else 'gather'}: p50 {t[len(t) // 2] * 1e3:.1f} us  min {t[0] * 1e3:.1f} us")


if __name__ == "__main__":
    main()
