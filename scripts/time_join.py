"""Event-timed device join pieces (cfg1 shape) + cfg3 streaming, for kernel A/B work."""
import os, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import engine, pipeline, synth  # noqa: E402
torch.cuda.set_device(0)
r, s = synth.cfg1_relations()
dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
def ev(fn, reps=20):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
plan = pipeline.plan_join(dr.columns[0], ds.columns[0])
cols = pipeline.join_out_columns(dr.columns, 0, ds.columns, 0, plan.total)
t_exp = ev(lambda: plan.expand(0, plan.total, cols))
t_idx = ev(lambda: engine.index_keys(dr.columns[0]))
t_al = ev(lambda: pipeline.plan_join(dr.columns[0], ds.columns[0]))
t_join = ev(lambda: pipeline.join(dr, ds, "key"))
r3, s3 = synth.cfg3_relations()
p3 = pipeline.plan_join(torch.from_numpy(r3.column("key").copy()).cuda(), torch.from_numpy(s3.column("key").copy()).cuda())
lr = torch.empty(1 << 30, dtype=torch.int32, device="cuda"); rr = torch.empty_like(lr)
a0 = p3.total // 2
t_str = ev(lambda: p3.expand(a0, a0 + (1 << 30), (), lr, rr), 5)
acc = torch.zeros(1, dtype=torch.int64, device="cuda")
t_ck = ev(lambda: p3.pair_checksum(a0, a0 + (1 << 32), acc), 3)
out_bytes = plan.total * 24
print(f"lib={os.environ.get('RELAB_B200_LIB','default')} expand_cfg1={t_exp*1e3:.1f}us ({out_bytes/(t_exp/1e3)/1e9:.0f} GB/s out) "
      f"index={t_idx*1e3:.1f}us plan={t_al*1e3:.1f}us join={t_join*1e3:.1f}us "
      f"cfg3_stream={(1<<30)/(t_str/1e3)/1e9:.1f} Gpairs/s ({(1<<30)*8/(t_str/1e3)/1e9:.0f} GB/s) "
      f"cfg3_checksum={(1<<32)/(t_ck/1e3)/1e9:.1f} Gpairs/s")
