"""cfg3 exact count (plan_join on the 10M x 10M Zipf keys) and streaming, event-timed."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, pipeline, synth  # noqa: E402
torch.cuda.set_device(0)
r, s = synth.cfg3_relations()
lk = torch.from_numpy(r.column("key").copy()).cuda(); sk = torch.from_numpy(s.column("key").copy()).cuda()
def ev(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
t_idx = ev(lambda: engine.index_keys(lk))
t_plan = ev(lambda: pipeline.plan_join(lk, sk))
p3 = pipeline.plan_join(lk, sk)
lr = torch.empty(1 << 30, dtype=torch.int32, device="cuda"); rr = torch.empty_like(lr)
a0 = p3.total // 2
t_str = ev(lambda: p3.expand(a0, a0 + (1 << 30), (), lr, rr), 3)
print(f"index={t_idx:.3f}ms plan={t_plan:.3f}ms total={p3.total} stream={(1<<30)/(t_str/1e3)/1e9:.0f} Gpairs/s")
