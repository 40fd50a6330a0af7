"""Probe: the cfg2 sort's globaltimer stamps (us after the first kernel start),
averaged over reps. Usage: python scripts/stamp_probe.py [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import _capi, engine, synth


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    lib = _capi.load()
    dev = torch.device("cuda:0")
    rel = synth.cfg2_relation(10_000_000)
    keys = torch.from_numpy(rel.column("key").copy()).to(dev)
    n = keys.numel()
    ws = engine.workspace(lib.rl_sort_workspace_bytes(n), dev)
    sk = torch.empty(n, dtype=torch.int64, device=dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.zeros(_capi.RL_SORT_STAMPS, dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for e in ev:  # (creates the CUDA events)
        e.record()
    arr = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(e.cuda_event) for e in ev])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    acc = None
    for r in range(reps + 2):
        flush.zero_()
        st.zero_()
        _capi.check(lib.rl_sort_axis_profiled(ctypes.c_void_p(keys.data_ptr()), 0, 8, 0, 0, None, n,
                                              ctypes.c_void_p(sk.data_ptr()), ctypes.c_void_p(perm.data_ptr()), None,
                                              0, ctypes.c_void_p(ws.data_ptr()), ws.numel(), engine.stream_handle(),
                                              arr, ctypes.c_void_p(st.data_ptr())), "sort")
        torch.cuda.synchronize()
        s = st.cpu().tolist()
        rel_us = [(x - s[0]) / 1e3 if x > 0 else float("nan") for x in s]
        if r >= 2:
            acc = rel_us if acc is None else [a + b for a, b in zip(acc, rel_us)]
    print(" ".join(f"[{i}]={a / reps:.1f}" for i, a in enumerate(acc)))


if __name__ == "__main__":
    main()
