"""Per-step sort times over many steps, with and without clock sampling (outlier hunt)."""
import ctypes, subprocess, sys, threading, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import _capi, engine, synth  # noqa
torch.cuda.set_device(0)
lib = _capi.load()
rel = synth.cfg2_relation()
keys = torch.from_numpy(rel.column("key").copy()).cuda()
n = keys.numel()
ws = engine.workspace(lib.rl_sort_workspace_bytes(n), keys.device)
sk = torch.empty(n, dtype=torch.int64, device="cuda"); perm = torch.empty(n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(steps):
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.rl_sort_axis(ctypes.c_void_p(keys.data_ptr()), 0, 8, 0, 0, None, n, ctypes.c_void_p(sk.data_ptr()),
                         ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(), engine.stream_handle())
        b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return ts
run(5)
stop = threading.Event()
def smi():
    while not stop.is_set():
        subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True)
        stop.wait(0.2)
for label, sampler in (("no sampler", False), ("nvidia-smi sampler", True), ("no sampler again", False)):
    th = None
    if sampler:
        stop.clear(); th = threading.Thread(target=smi, daemon=True); th.start()
    ts = run(60)
    if th: stop.set(); th.join()
    ts_sorted = sorted(ts)
    print(f"{label}: median {ts_sorted[30]:.3f} ms max {ts_sorted[-1]:.3f} ms >1.2ms: {sum(t > 1.2 for t in ts)}")
