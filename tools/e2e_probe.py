"""Probe host<->device bandwidth and the e2e pipeline chunking on the box."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as ME

ctx, grid, n_s = ME.config_geometry("cfg2")
B = 32
eng = bm.BmodeEngine(ctx, grid)
rf_h, disp_h = eng.pinned(B, n_s)
rf_h.normal_()
dev = torch.empty_like(rf_h, device="cuda")
out = {}
for _ in range(2):
    dev.copy_(rf_h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    dev.copy_(rf_h, non_blocking=True)
torch.cuda.synchronize()
out["h2d_GBps"] = 5 * rf_h.numel() * 4 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(5):
    rf_h.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
out["d2h_GBps"] = 5 * rf_h.numel() * 4 / (time.perf_counter() - t) / 1e9
for chunk in (1, 2, 4, 8):
    eng.reconstruct_host_stream([(rf_h, disp_h)] * 2, chunk=chunk)
    t = time.perf_counter(); eng.reconstruct_host_stream([(rf_h, disp_h)] * 10, chunk=chunk)
    out[f"stream_fps_chunk{chunk}"] = 10 * B / (time.perf_counter() - t)
    for _ in range(2):
        eng.reconstruct_host(rf_h, disp_h, chunk=chunk)
    t = time.perf_counter()
    for _ in range(5):
        eng.reconstruct_host(rf_h, disp_h, chunk=chunk)
    out[f"e2e_fps_chunk{chunk}"] = 5 * B / (time.perf_counter() - t)
print(json.dumps(out))
