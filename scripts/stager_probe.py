"""Stager throughput for different (threads, chunk, slots) on the GPU box."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import _capi as C, engine  # noqa: E402

torch.cuda.set_device(0)
lib = C.load()
n = 120 << 20
src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for threads, chunk_mb, slots in [(8, 8, 4), (8, 4, 6), (8, 16, 3), (12, 8, 4), (16, 8, 4), (4, 8, 4), (8, 2, 8),
                                 (16, 4, 8)]:
    h = lib.rl_stager_create(threads, chunk_mb << 20, slots)
    ts = []
    for r in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        C.check(lib.rl_stager_h2d(h, ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.ctypes.data), n,
                                  engine.stream_handle(), None), "h2d")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    lib.rl_stager_destroy(h)
    best = min(ts[1:])
    print(f"threads={threads:2d} chunk={chunk_mb:2d}MB slots={slots}: {n/best/1e9:5.1f} GB/s ({best*1e3:.2f} ms)")
assert (dst.cpu().numpy() == src).all()
