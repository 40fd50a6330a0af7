"""cfg1 join plan pieces: one index, both indexes (plan without the alignment is not separable, so
the plan is timed whole), with and without the concurrent sides (RL_PLAN_SERIAL)."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, pipeline, synth  # noqa: E402
torch.cuda.set_device(0)
r, s = synth.cfg1_relations()
lk = torch.from_numpy(r.column("key").copy()).cuda(); rk = torch.from_numpy(s.column("key").copy()).cuda()
def ev(fn, reps=30):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
li = engine.index_keys(lk); ri = engine.index_keys(rk)
print(f"index1={1e3*ev(lambda: engine.index_keys(lk)):.1f}us "
      f"index2_serial={1e3*ev(lambda: (engine.index_keys(lk), engine.index_keys(rk))):.1f}us "
      f"align={1e3*ev(lambda: engine.align(li, ri)):.1f}us "
      f"plan={1e3*ev(lambda: pipeline.plan_join(lk, rk)):.1f}us")
