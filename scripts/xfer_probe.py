"""Probe host<->device copy paths on the GPU box (for the e2e design)."""
import os, time, threading
import numpy as np
import torch
torch.cuda.set_device(0)
n = 120 * 2**20
src = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts)
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin_np = pin.numpy()
x = t(lambda: dev.copy_(torch.from_numpy(src)))
print(f"pageable H2D: {n/x/1e9:.1f} GB/s")
x = t(lambda: dev.copy_(pin, non_blocking=True))
print(f"pinned H2D: {n/x/1e9:.1f} GB/s")
x = t(lambda: pin.copy_(dev, non_blocking=True))
print(f"pinned D2H: {n/x/1e9:.1f} GB/s")
x = t(lambda: np.copyto(pin_np, src))
print(f"memcpy 1 thread: {n/x/1e9:.1f} GB/s")
for nt in (2, 4, 8, 16):
    def mt():
        ch = n // nt
        th = [threading.Thread(target=np.copyto, args=(pin_np[i*ch:(i+1)*ch], src[i*ch:(i+1)*ch])) for i in range(nt)]
        [a.start() for a in th]; [a.join() for a in th]
    x = t(mt)
    print(f"memcpy {nt} threads: {n/x/1e9:.1f} GB/s")
x = t(lambda: torch.from_numpy(src).to("cuda"))
print(f"torch.from_numpy().to(cuda): {n/x/1e9:.1f} GB/s")
# fresh numpy output allocation + D2H pageable
x = t(lambda: dev.cpu())
print(f"pageable D2H .cpu(): {n/x/1e9:.1f} GB/s")
# cudaHostRegister cost
cudart = torch.cuda.cudart()
buf = np.empty(n, dtype=np.uint8); buf[:] = 1
t0 = time.perf_counter()
r = cudart.cudaHostRegister(buf.ctypes.data, n, 0)
t1 = time.perf_counter()
print("cudaHostRegister", r, f"{(t1-t0)*1e3:.1f} ms for {n/2**20:.0f} MiB")
cudart.cudaHostUnregister(buf.ctypes.data)
