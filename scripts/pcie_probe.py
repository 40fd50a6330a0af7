"""PCIe and e2e timeline probe for the cfg2 sort: raw pinned H2D / D2H bandwidth,
H2D and D2H concurrently (full duplex?), and tensor_sort's wall time."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import synth, tensor_sort, SortSpec  # noqa: E402

torch.cuda.set_device(0)
MB = 1 << 20
def bw(fn, nbytes, reps=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9

n = 80 * MB
hs = torch.empty(n, dtype=torch.uint8, pin_memory=True); hd = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("h2d GB/s", round(bw(lambda: d1.copy_(hs, non_blocking=True), n), 1))
print("d2h GB/s", round(bw(lambda: hd.copy_(d2, non_blocking=True), n), 1))
def both():
    with torch.cuda.stream(s1):
        d1.copy_(hs, non_blocking=True)
    with torch.cuda.stream(s2):
        hd.copy_(d2, non_blocking=True)
print("h2d+d2h concurrent GB/s (sum)", round(bw(both, 2 * n), 1))
# pageable numpy -> registered
a = np.random.default_rng(0).integers(0, 1 << 60, n // 8, dtype=np.int64)
rel = synth.cfg2_relation()
spec = SortSpec(("key",))
for _ in range(3):
    tensor_sort(rel, spec)
ts = []
for _ in range(20):
    t = time.perf_counter(); out, _ = tensor_sort(rel, spec); ts.append(time.perf_counter() - t)
print("tensor_sort cfg2 ms p50", round(1e3 * sorted(ts)[10], 3), "min", round(1e3 * min(ts), 3))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    tensor_sort(rel, spec)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# ---- timeline of one tensor_sort (same steps as tensor_path.tensor_sort, with events)
from paper_2602_21237_b200 import tensor_path as TP, engine  # noqa: E402
import paper_2602_21237_b200._capi as C  # noqa: E402
def timeline():
    dev = torch.device("cuda:0")
    cur = torch.cuda.current_stream()
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("t0", "keys_up", "sorted", "sorted_again", "pay_up", "gathered", "keys_down", "pay_down")}
    ev["t0"].record()
    up = TP._Uploads(rel.columns, dev)
    kd = up.get(0)
    ev["keys_up"].record()  # (the current stream waits on the stager's copy)
    sk = torch.empty(rel.row_count, dtype=torch.int64, device=dev)
    perm = engine.sort_permutation([engine.SortAxis(kd, False)], rel.row_count, dev, sorted_keys_out=sk)
    ev["sorted"].record()
    if AGAIN:
        engine.sort_permutation([engine.SortAxis(kd, False)], rel.row_count, dev, sorted_keys_out=torch.empty_like(sk))
    ev["sorted_again"].record()
    down = TP._d2h_stream(dev)
    hk = TP._host_out_on(sk, down)
    with torch.cuda.stream(down):
        ev["keys_down"].record()
    col = TP._out_column(up.get(1), rel.schema.attributes[1][1], rel.row_count, dev, C.RL_SIDE_LEFT)
    ev["pay_up"].record()
    engine.gather_rows(perm, [col])
    ev["gathered"].record()
    hp = TP._host_out_on(col.dst, down)
    with torch.cuda.stream(down):
        ev["pay_down"].record()
    down.synchronize(); torch.cuda.synchronize()
    return {k: round(ev["t0"].elapsed_time(e), 3) for k, e in ev.items() if k != "t0"}
AGAIN = False
for _ in range(3):
    timeline()
AGAIN = False
for _ in range(3):
    print("timeline ms (from t0):", timeline())
AGAIN = True
for _ in range(2):
    print("timeline + 2nd sort ms:", timeline())
