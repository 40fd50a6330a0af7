"""RELCOL01 ingest throughput: a 1e8-row (key int64, payload int64) relation file -> HBM
(page-cache-resident file), vs numpy read_relation-style reading + upload."""
import os, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_21237_b200 import pipeline, relfile, synth  # noqa: E402
torch.cuda.set_device(0)
n = 100_000_000
r, _ = synth.cfg1_relations(n=n, domain=n)
path = Path(os.environ.get("TMPDIR", "/tmp")) / "cfg5_r.relcol"
dr = pipeline.DeviceRelation.from_host(r)
t0 = time.perf_counter(); dr.to_file(path); torch.cuda.synchronize(); tw = time.perf_counter() - t0
nbytes = path.stat().st_size
for _ in range(2):
    t0 = time.perf_counter(); d2 = pipeline.DeviceRelation.from_file(path); torch.cuda.synchronize(); tr = time.perf_counter() - t0
t0 = time.perf_counter(); rel = relfile.read_pinned(path); tp = time.perf_counter() - t0
t0 = time.perf_counter()
with open(path, "rb") as f:
    f.seek(len(relfile.header_bytes(r.schema, n)))
    cols = [np.frombuffer(f.read(n * 8), dtype="<i8").astype(np.int64) for _ in range(2)]
d3 = [torch.from_numpy(c).cuda() for c in cols]; torch.cuda.synchronize(); tn = time.perf_counter() - t0
ok = all(bool(torch.equal(a, b)) for a, b in zip(d2.columns, dr.columns))
print(f"file {nbytes/1e9:.2f} GB ok={ok}: to_file {nbytes/tw/1e9:.1f} GB/s, from_file {nbytes/tr/1e9:.1f} GB/s, "
      f"read_pinned {nbytes/tp/1e9:.1f} GB/s, numpy read + upload {nbytes/tn/1e9:.1f} GB/s")
path.unlink()
