"""experiment: cost of cudaHostRegister/Unregister of one 11.5 MB numpy frame"""
import statistics
import time

import numpy as np
import torch

n = 11 * 128 * 2048
a = np.random.default_rng(0).standard_normal(n).astype(np.float32)
dev = torch.empty(n, device="cuda")
rt = torch.cuda.cudart()
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    dev.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1, t3 - t2))
print("register / copy / unregister ms", [round(statistics.median(v) * 1e3, 4) for v in zip(*ts)], r)
