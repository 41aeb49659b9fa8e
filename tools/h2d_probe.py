"""H2D bandwidth from pinned memory: one stream vs two / four concurrent streams."""
import json, time
import torch
n = 369098752 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True).normal_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
out = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = [(i * n // ns, (i + 1) * n // ns) for i in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for k in range(5):
            for s, (a, b) in zip(streams, parts):
                with torch.cuda.stream(s):
                    d[a:b].copy_(h[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    out[f"h2d_GBps_{ns}streams"] = round(5 * n * 4 / dt / 1e9, 2)
# h2d and d2h concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n // 8, dtype=torch.float32, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter()
for k in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d[: n // 8], non_blocking=True)
torch.cuda.synchronize()
out["h2d_with_d2h_GBps"] = round(5 * n * 4 / (time.perf_counter() - t) / 1e9, 2)
print(json.dumps(out))
