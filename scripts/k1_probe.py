import ctypes, statistics, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2602_21237_b200 import _capi, engine, synth
lib = _capi.load(); torch.cuda.set_device(0)
keys = torch.from_numpy(synth.cfg2_relation(10_000_000).column("key").copy()).cuda()
n = keys.numel()
ws = engine.workspace(lib.rl_sort_workspace_bytes(n), keys.device)
sk = torch.empty(n, dtype=torch.int64, device="cuda"); perm = torch.empty(n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for e in evs: e.record()
arr = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(e.cuda_event) for e in evs])
st = torch.zeros(12, dtype=torch.int64, device="cuda")
res = []
for r in range(23):
    flush.zero_(); st.zero_()
    _capi.check(lib.rl_sort_axis_profiled(ctypes.c_void_p(keys.data_ptr()), 0, 8, 0, 0, None, n, ctypes.c_void_p(sk.data_ptr()), ctypes.c_void_p(perm.data_ptr()), None, 0, ctypes.c_void_p(ws.data_ptr()), ws.numel(), engine.stream_handle(), arr, ctypes.c_void_p(st.data_ptr())), "sort")
    torch.cuda.synchronize()
    t = st.cpu().tolist()
    if r >= 3: res.append([(t[4]-t[0])/1e3, (t[5]-t[4])/1e3, (t[6]-t[5])/1e3, (t[7]-t[0])/1e3, (t[8]-t[0])/1e3, (t[2]-t[0])/1e3])
m = np.median(np.array(res), axis=0)
print("CTA0: zero %.1f us, count loop %.1f us, copy-out %.1f us; from K1 start: last count loop end %.1f us, last CTA end %.1f us, pass A start %.1f us" % tuple(m))
