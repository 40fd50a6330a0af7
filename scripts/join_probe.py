"""Probe: the cfg5-shaped join alone (device relations from torch.randint),
bucket plan vs sort plan, for timing and an ncu launch list.
Usage: python scripts/join_probe.py n [reps] [bucket|sort|both]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import pipeline
from paper_2602_21237_b200 import records as R


def main():
    n = int(float(sys.argv[1]))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    which = sys.argv[3] if len(sys.argv) > 3 else "both"
    shape = os.environ.get("PROBE_SHAPE", "cfg5")
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(n)
    if shape == "cfg4":  # (a << 32) | b, a, b < 2^16; 16-byte payload
        mk = lambda: (torch.randint(0, 1 << 16, (n,), generator=g, device=dev) << 32) | torch.randint(  # noqa: E731
            0, 1 << 16, (n,), generator=g, device=dev)
        lk, rk = mk(), mk()
        pay = torch.randint(0, 256, (n, 16), generator=g, device=dev, dtype=torch.uint8)
        schema = R.Schema((("key", R.Int64()), ("payload", R.Bytes(16))))
    else:
        lk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
        rk = torch.randint(0, n, (n,), generator=g, device=dev, dtype=torch.int64)
        pay = torch.arange(n, device=dev, dtype=torch.int64)
        schema = R.Schema((("key", R.Int64()), ("payload", R.Int64())))
    dl = pipeline.DeviceRelation(schema, [lk, pay])
    dr = pipeline.DeviceRelation(schema, [rk, pay])
    modes = ["bucket", "sort"] if which == "both" else [which]
    for mode in modes:
        os.environ["RL_NO_BJOIN"] = "1" if mode == "sort" else "0"
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = pipeline.join(dl, dr, "key")
            b.record()
            b.synchronize()
            print(f"{mode} join n={n:.0e}: {a.elapsed_time(b):.3f} ms rows={out.row_count}", flush=True)
            del out


if __name__ == "__main__":
    main()
