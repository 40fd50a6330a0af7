import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine
torch.cuda.set_device(0)
fails = []
for n in list(range(2, 700)) + [3071, 3072, 3073, 7000]:
    for mode in ("neg", "wide", "small"):
        rng = np.random.default_rng(n)
        keys = {"neg": rng.integers(-8, 8, n), "wide": rng.integers(-(2**62), 2**62, n), "small": rng.integers(0, 4, n)}[mode]
        kd = torch.from_numpy(keys.astype(np.int64)).cuda()
        sk = torch.empty(n, dtype=torch.int64, device="cuda")
        perm = engine.sort_permutation([engine.SortAxis(kd)], n, kd.device, sorted_keys_out=sk)
        got = perm.cpu().numpy().view(np.uint32).astype(np.int64)
        want = np.argsort(keys, kind="stable")
        if not (got == want).all():
            fails.append((n, mode))
print("fails", len(fails), fails[:60])
