"""Does torch symmetric memory (NVLink peer buffers) work here at world 1?"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = symm.empty(1024, dtype=torch.float32, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD)
print("backend", symm.get_backend("cuda") if hasattr(symm, "get_backend") else "?")
print("world", h.world_size, "rank", h.rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "local", hex(t.data_ptr()))
print("signal pads", [hex(p) for p in h.signal_pad_ptrs], "pad size", h.signal_pad_size)
peer = h.get_buffer(0, (1024,), torch.float32)
peer.fill_(3.0)
torch.cuda.synchronize()
print("write via peer view visible locally:", float(t[5]))
dist.destroy_process_group()
