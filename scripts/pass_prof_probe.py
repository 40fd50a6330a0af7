"""Probe (RL_PASS_PROFILE builds): per-phase SM clock totals of the counting
passes over cfg2-shaped sorts: tile atomics (incl. the wait for the tile's
loads), digit scan, staging, write-out. Usage: RELAB_B200_LIB=<variant.so>
python scripts/pass_prof_probe.py [n] [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_21237_b200 import _capi, engine, synth


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    lib = _capi.load()
    prof = lib.rl_debug_pass_prof
    prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
    rel = synth.cfg2_relation(n)
    keys = torch.from_numpy(rel.column("key").copy()).cuda()
    sk = torch.empty_like(keys)
    buf = (ctypes.c_ulonglong * 32)()
    engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk)
    prof(buf, 1)
    for _ in range(reps):
        engine.sort_permutation([engine.SortAxis(keys)], n, keys.device, sorted_keys_out=sk)
    prof(buf, 1)
    v = list(buf)
    for name, o in (("digit-7 pass", 0), ("digit-6 pass", 8)):
        tiles = v[o + 4] or 1
        idx = [0, 1, 2, 5, 3]
        tot = sum(v[o + i] for i in idx) or 1
        print(f"{name}: {tiles // reps} tiles/sort, cycles per tile: " + ", ".join(
            f"{k} {v[o + i] / tiles:.0f} ({v[o + i] / tot:.0%})"
            for i, k in zip(idx, ["atomics+load wait", "scan", "staging", "next loads", "write-out"])))

    runs = v[24] or 1
    names = ["prefetch: TMA issue (warp 0)", "zero+data+barrier", "count", "scan", "scatter", "rank+emit", "prefetch: groups (warp 0)", "big bins"]
    tot = sum(v[16 + i] for i in (0, 1, 2, 3, 4, 5, 6, 7)) or 1
    print(f"local phase: {runs // reps} runs/sort, cycles per run: " + ", ".join(
        f"{names[i]} {v[16 + i] / runs:.0f} ({v[16 + i] / tot:.0%})" for i in (6, 0, 1, 2, 3, 4, 5, 7)))


if __name__ == "__main__":
    main()
