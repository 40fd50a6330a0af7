"""cfg2 sort step (histogram + cooperative sort + payload gather) eager vs CUDA-graph replay."""
import ctypes
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import _capi, engine, synth  # noqa: E402

torch.cuda.set_device(0)
lib = _capi.load()
rel = synth.cfg2_relation(10_000_000)
keys = torch.from_numpy(rel.column("key").copy()).cuda()
pay = torch.from_numpy(rel.column("payload").copy()).cuda()
n = keys.numel()
ws = engine.workspace(lib.rl_sort_workspace_bytes(n), keys.device)
sk = torch.empty(n, dtype=torch.int64, device="cuda")
perm = torch.empty(n, dtype=torch.int32, device="cuda")
out = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    s = engine.stream_handle()
    _capi.check(lib.rl_sort_axis(ctypes.c_void_p(keys.data_ptr()), 0, 8, 0, 0, None, n, ctypes.c_void_p(sk.data_ptr()),
                                 ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(), s), "sort")
    engine.gather_rows(perm, [engine.OutColumn(pay, out, 4, 0)])


def timed(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


print(f"eager median {timed(step):.4f} ms")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
try:
    with torch.cuda.graph(g):
        step()
    ok_before = sk.clone()
    print(f"graph median {timed(g.replay):.4f} ms")
    p64 = perm.to(torch.int64) & 0xFFFFFFFF
    print("graph result ok", bool((keys[p64] == sk).all()) and bool((sk[1:] >= sk[:-1]).all()) and bool((pay[p64] == out).all()))
except Exception as e:  # noqa: BLE001
    print("capture failed:", repr(e)[:300])
