"""Pinned H2D rate vs transfer size on the box (is an 11.5 MB frame copy
latency- or bandwidth-bound?)."""
import torch

dev = torch.device("cuda", 0)
for mb in (1, 4, 11.5, 23, 46, 92, 184, 369):
    n = int(mb * 2**20) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{mb:7.1f} MB  {ms:7.3f} ms  {n * 4 / ms / 1e6:6.1f} GB/s")

# one 11.5 MB frame copied in chunks
n = int(11.5 * 2**20) // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device=dev)
for ch_mb in (0.5, 1, 2, 4, 8):
    c = int(ch_mb * 2**20) // 4

    def go():
        for o in range(0, n, c):
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        go()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"11.5 MB in {ch_mb} MB chunks: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
# a second, separately allocated 11.5 MB buffer (placement effects?)
for k in range(3):
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        d.copy_(h2, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    print(f"fresh 11.5 MB pinned buffer {k}: {s.elapsed_time(e) / 20:.3f} ms")
