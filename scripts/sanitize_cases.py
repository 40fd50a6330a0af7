"""Small cases for compute-sanitizer: hybrid sort (+ post-pass fallback), LSD
sort, multi-key sort, join plan + expansion, each checked against numpy."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import tensorpath_oracle as O  # noqa: E402
from paper_2602_21237_b200 import engine, synth, tensor_join, to_tensor  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(1)


def sort_check(keys, desc=False):
    kd = torch.from_numpy(keys).cuda()
    perm = engine.sort_permutation([engine.SortAxis(kd, desc)], len(keys), kd.device)
    assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == O.stable_axis_order(keys, desc)).all()


full = lambda n: rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64, endpoint=True)  # noqa: E731
sort_check(full(300_000))                      # hybrid
sort_check(full(300_000), True)
k = full(300_000)
k[rng.choice(300_000, 3000, replace=False)] = (np.int64(0x1234) << 48) | rng.integers(0, 1 << 40, 3000)
sort_check(k)                                  # hybrid -> post-pass LSD fallback
sort_check(rng.integers(0, 1 << 20, 200_000).astype(np.int64))  # LSD
a = rng.integers(-3, 3, 50_000).astype(np.int64)
w = rng.integers(0, 3, (50_000, 11), dtype=np.uint8)
perm = engine.sort_permutation([engine.SortAxis(torch.from_numpy(a).cuda(), True),
                                engine.SortAxis(torch.from_numpy(w).cuda(), False)], 50_000, "cuda")
assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == O.sort_permutation([a, w], [True, False])).all()
r, s = synth.cfg1_relations(n=200_000, domain=150_000, seed=2)
out, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
want = O.join_columns(list(r.columns), 0, list(s.columns), 0)
assert all((x == y).all() for x, y in zip(out.columns, want))
torch.cuda.synchronize()
print("sanitize cases ok")
