"""Can the TMA DAS kernel read RF straight from pinned (mapped) host memory?
(one cfg2 frame; bitwise vs the device-resident launch, and timing)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm  # noqa: E402
from bench import synth_frames  # noqa: E402
from paper_1811_01566_b200 import _native as N  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = synth_frames(ctx, n_s, 1, 0)
plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
dev_rf = torch.from_numpy(host).cuda()
ref = plan.beamform_batch(dev_rf)
pin = torch.from_numpy(host).pin_memory()
out = torch.empty_like(ref)
g = plan.geometry(n_s, "linear", True)
stride = ctx.n_tx * ctx.n_elements * n_s
try:
    N.call("bm_das_beamform", ctypes.byref(g), pin.data_ptr(), stride, out.data_ptr(),
           grid.n_z * grid.n_x, 1, N.stream_ptr())
    torch.cuda.synchronize()
    print("zero-copy TMA ran; bitwise equal:", torch.equal(out, ref))
except Exception as exc:
    print("zero-copy failed:", exc)
    sys.exit(0)


def t(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def zc():
    N.call("bm_das_beamform", ctypes.byref(g), pin.data_ptr(), stride, out.data_ptr(),
           grid.n_z * grid.n_x, 1, N.stream_ptr())


print("device-resident DAS ms", t(lambda: plan.beamform_batch(dev_rf, out=out[None])))
print("zero-copy DAS ms", t(zc))
print("H2D pinned + DAS ms", t(lambda: plan.beamform_batch(pin.to("cuda", non_blocking=True), out=out[None])))
