import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as sm

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29613")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
print("backend", sm.get_backend(torch.device("cuda", 0)) if hasattr(sm, "get_backend") else "?")
t = sm.empty(1 << 20, dtype=torch.uint8, device="cuda")
h = sm.rendezvous(t, dist.group.WORLD.group_name)
print("world", h.world_size, "rank", h.rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "size", h.buffer_size)
h.barrier()
t.fill_(7)
torch.cuda.synchronize()
print("ok", int(t[0]), "multicast", h.has_multicast_support())
dist.destroy_process_group()
