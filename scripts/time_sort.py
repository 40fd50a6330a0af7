"""Event-timed cfg2-shaped sort (10M int64 keys) for kernel A/B work.
Usage: RELAB_B200_LIB=path python scripts/time_sort.py [--n N] [--reps R]"""
import argparse
import ctypes
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import _capi, engine, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--uniform-bits", type=int, default=0, help="keys uniform in [0, 2^bits) instead of cfg2")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _capi.load()
    if a.uniform_bits:
        keys_h = np.random.default_rng(0).integers(0, 2**a.uniform_bits, a.n, dtype=np.int64)
    else:
        keys_h = synth.cfg2_relation(a.n).column("key")
    keys = torch.from_numpy(keys_h.copy()).cuda()
    n = a.n
    ws = engine.workspace(lib.rl_sort_workspace_bytes(n), keys.device)
    sk = torch.empty(n, dtype=torch.int64, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = engine.stream_handle()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(_capi.RL_SORT_EVENTS)]
    for e in evs:
        e.record()
    arr = (ctypes.c_void_p * len(evs))(*[ctypes.c_void_p(e.cuda_event) for e in evs])
    stamps = torch.zeros(_capi.RL_SORT_STAMPS, dtype=torch.int64, device="cuda")
    tot, passes, hist, local, full, scan, span, tail = [], [], [], [], [], [], [], []
    e_end = torch.cuda.Event(enable_timing=True)
    for r in range(a.reps + 3):
        flush.zero_()
        stamps.zero_()
        _capi.check(lib.rl_sort_axis_profiled(ctypes.c_void_p(keys.data_ptr()), 0, 8, 0, 0, None, n,
                                              ctypes.c_void_p(sk.data_ptr()), ctypes.c_void_p(perm.data_ptr()),
                                              None, 0, ctypes.c_void_p(ws.data_ptr()), ws.numel(), s, arr,
                                              ctypes.c_void_p(stamps.data_ptr())), "sort")
        e_end.record()
        torch.cuda.synchronize()
        if r >= 3:
            tot.append(evs[0].elapsed_time(evs[2]))
            st = stamps.cpu().tolist()
            if st[11] == 3:  # scatter hybrid: K1 st[0], K2 st[2], K3 st[3], local phase st[1]..st[10]
                hist.append((st[2] - st[0]) / 1e6)
                span.append((st[10] - st[0]) / 1e6)
                tail.append([(st[8] - st[10]) / 1e3, (st[9] - st[8]) / 1e3, (st[9] - st[0]) / 1e3])
                passes.append([(st[3] - st[2]) / 1e6, (st[1] - st[3]) / 1e6] + [0.0] * 6)
                scan.append(0.0)
                local.append((st[10] - st[1]) / 1e6)
                full.append(evs[0].elapsed_time(e_end))
                continue
            hist.append((st[1] - st[0]) / 1e6)
            hybrid = st[11] == 1
            prev, pp = st[1], []
            for p in range(8):
                if st[2 + p] and not (hybrid and p == 0):
                    pp.append((st[2 + p] - prev) / 1e6)
                    prev = st[2 + p]
                else:
                    pp.append(0.0)
            passes.append(pp)
            if hybrid:
                scan.append((st[2] - st[9]) / 1e6)
                local.append((st[10] - st[2]) / 1e6)
            else:
                local.append((st[10] - prev) / 1e6)
            full.append(evs[0].elapsed_time(e_end))
    ok = bool((sk[1:] >= sk[:-1]).all()) and bool((keys[perm.long() & 0xFFFFFFFF] == sk).all())
    pm = np.median(np.array(passes), axis=0)
    act = pm[pm > 0.01]
    print(f"lib={os.environ.get('RELAB_B200_LIB','default')} path={int(st[11])} n={n} ok={ok} total_ms={statistics.median(tot):.4f} "
          f"with_fallback_ms={statistics.median(full):.4f} scan_us={1e3*statistics.median(scan) if scan else 0:.1f} local_us={1e3*statistics.median(local):.1f} "
          f"hist_us={1e3*statistics.median(hist):.1f} pass_us={[round(1e3*x,1) for x in pm]} "
          f"pass_GBps={24*n/(np.mean(act)/1e3)/1e9:.0f}"
          + (f" outside_kernels_us={1e3*(statistics.median(tot)-statistics.median(span)):.1f}"
             f" [local_last_end-cta0_end, coop_start-local_last_end, k1_start->coop_start] us={np.median(np.array(tail), axis=0).round(1).tolist()}" if span else ""))


if __name__ == "__main__":
    main()
