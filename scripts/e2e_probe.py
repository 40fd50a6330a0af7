"""Per-step e2e timings of the drop-in sort/join (host numpy in/out)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import SortSpec, synth, tensor_join, tensor_sort, to_tensor
torch.cuda.set_device(0)
rel = synth.cfg2_relation()
spec = SortSpec(("key",))
ts = []
for i in range(15):
    t0 = time.perf_counter()
    out, _ = tensor_sort(rel, spec)
    ts.append(1e3 * (time.perf_counter() - t0))
print("sort e2e ms", [round(x, 2) for x in ts])
r, s = synth.cfg1_relations()
ts = []
for i in range(30):
    t0 = time.perf_counter()
    o, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
    ts.append(1e3 * (time.perf_counter() - t0))
print("join e2e ms", [round(x, 2) for x in ts])
# phase breakdown of one sort
import paper_2602_21237_b200.tensor_path as tp
t0 = time.perf_counter(); up = tp._Uploads(rel.columns, torch.device("cuda")); k = up.get(0); p = up.get(1); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"upload 120MB: {1e3*(t1-t0):.2f} ms")
h = torch.empty((10_000_000,), dtype=torch.int64, pin_memory=True)
t0 = time.perf_counter(); h.copy_(k, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"D2H 80MB pinned: {1e3*(t1-t0):.2f} ms")
t0 = time.perf_counter(); h2 = torch.empty((10_000_000,), dtype=torch.int64, pin_memory=True); t1 = time.perf_counter()
print(f"pinned alloc 80MB: {1e3*(t1-t0):.2f} ms")
