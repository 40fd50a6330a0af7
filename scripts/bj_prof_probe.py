"""Probe (RL_BJ_PROFILE builds): per-phase SM clock totals of the bucket join's
emit kernel (cfg5-shaped join, device inputs). Usage: RELAB_B200_LIB=<variant.so>
python scripts/bj_prof_probe.py [n] [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import _capi, pipeline
from paper_2602_21237_b200 import records as R


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    lib = _capi.load()
    prof = lib.rl_debug_bj_prof
    prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(n)
    lk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
    rk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
    pay = torch.arange(n, device=dev, dtype=torch.int64)
    schema = R.Schema((("key", R.Int64()), ("payload", R.Int64())))
    dl, dr = pipeline.DeviceRelation(schema, [lk, pay]), pipeline.DeviceRelation(schema, [rk, pay])
    buf = (ctypes.c_ulonglong * 16)()
    out = pipeline.join(dl, dr, "key")
    del out
    prof(buf, 1)
    for _ in range(reps):
        out = pipeline.join(dl, dr, "key")
        del out
    prof(buf, 1)
    v = list(buf)
    runs = v[8] or 1
    names = {7: "group setup", 0: "row loads", 1: "left sort", 2: "right sort", 3: "match+prefix", 4: "output map",
             5: "write outputs"}
    tot = sum(v[i] for i in names) or 1
    print(f"emit: {runs // reps} runs/join, cycles per run: " + ", ".join(
        f"{names[i]} {v[i] / runs:.0f} ({v[i] / tot:.0%})" for i in (7, 0, 1, 2, 3, 4, 5)))


if __name__ == "__main__":
    main()
