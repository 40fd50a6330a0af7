"""Tail of the cfg1 e2e join latency (tensor_join(to_tensor(R), to_tensor(S))):
300 reps with Python's GC on, then off; prints percentiles and the slow reps."""
import gc
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import synth, tensor_join, to_tensor  # noqa: E402

torch.cuda.set_device(0)
r, s = synth.cfg1_relations()
for _ in range(5):
    tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))


def pct(xs, q):
    xs = sorted(xs)
    return xs[max(math.ceil(q / 100 * len(xs)), 1) - 1]


for label, gc_on in (("gc on", True), ("gc off", False)):
    (gc.enable if gc_on else gc.disable)()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        out, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
        ts.append(1e3 * (time.perf_counter() - t0))
        del out
    slow = [(i, round(t, 2)) for i, t in enumerate(ts) if t > 1.6 * pct(ts, 50)]
    print(f"{label}: p50 {pct(ts, 50):.3f} p99 {pct(ts, 99):.3f} p99.9 {pct(ts, 99.9):.3f} max {max(ts):.3f} ms; "
          f"slow reps {slow[:12]}")
gc.enable()
