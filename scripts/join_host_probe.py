"""Host-side stage times of the cfg1 e2e join (to_tensor x2 + tensor_join), cProfile top entries."""
import cProfile, pstats, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import synth, tensor_join, to_tensor  # noqa: E402
torch.cuda.set_device(0)
r, s = synth.cfg1_relations()
for _ in range(10):
    tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
t = {"to_tensor_R": 0.0, "to_tensor_S": 0.0, "tensor_join": 0.0}
N = 100
for _ in range(N):
    t0 = time.perf_counter(); a = to_tensor(r, "key"); t1 = time.perf_counter(); b = to_tensor(s, "key")
    t2 = time.perf_counter(); tensor_join(a, b); t3 = time.perf_counter()
    t["to_tensor_R"] += t1 - t0; t["to_tensor_S"] += t2 - t1; t["tensor_join"] += t3 - t2
print({k: round(1e3 * v / N, 3) for k, v in t.items()})
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
