"""Debug probe: a sequence of sorts in one process, e.g. `E0 E1` (extremes asc
then desc), `U0` (uniform, no fallback), `N0` (narrow keys: K1 wrap / pre-check)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2602_21237_b200 import engine
I64_MIN, I64_MAX = -(2**63), 2**63 - 1
n = 600_000


def make(kind):
    rng = np.random.default_rng(10)
    keys = rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64, endpoint=True)
    if kind == "E":
        keys[::97] = I64_MIN; keys[::89] = I64_MAX; keys[::83] = -1; keys[::79] = 0
    elif kind == "N":
        keys = rng.integers(0, 1 << 40, n, dtype=np.int64)
    return keys


for step in sys.argv[1:]:
    keys = make(step[0])
    kd = torch.from_numpy(keys).cuda()
    sk = torch.empty(n, dtype=torch.int64, device="cuda")
    perm = engine.sort_permutation([engine.SortAxis(kd, step[1] == "1")], n, kd.device, sorted_keys_out=sk)
    torch.cuda.synchronize()
    print("ok", step, flush=True)
