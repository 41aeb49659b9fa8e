"""One-frame cfg2 / sta-paper DAS time per apodisation (the drop-in path with
non-uniform receive weights)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402

for name in ("cfg2", "sta-paper"):
    ctx, grid, n_s = bm.environment.config_geometry(name)
    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    rf = torch.randn((1, ctx.n_tx, n_rx, n_s), device="cuda")
    for apod in (("rectangular", 0.0), ("hann", 0.0), ("hann", 1.5), ("rectangular", 1.5)):
        plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(*apod), np.float32, n_rx)
        out = plan.beamform_batch(rf)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            plan.beamform_batch(rf, out=out)
        b.record()
        torch.cuda.synchronize()
        print(name, apod, round(a.elapsed_time(b) / 20, 4), "ms", plan.launch_shape(n_s, 1))
