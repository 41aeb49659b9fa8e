"""f64 pwi-paper one-frame DAS (192 elements: the generic kernel): time per
launch, and with the generic kernel's tile-row override."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402
from paper_1811_01566_b200 import _native as N  # noqa: E402

for name in ("pwi-paper", "sta-paper"):
    ctx, grid, n_s = bm.environment.config_geometry(name)
    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    for interp in ("nearest", "linear"):
        plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float64, n_rx)
        rf = torch.randn((1, ctx.n_tx, n_rx, n_s), device="cuda", dtype=torch.float64)
        for tz in (0, 1, 2, 4):
            with N.debug_overrides(das_generic_tz=tz):
                out = plan.beamform_batch(rf, interp)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10):
                    plan.beamform_batch(rf, interp, out=out)
                b.record()
                torch.cuda.synchronize()
                print(name, interp, plan.kernel_for(n_s, interp), "tz", tz,
                      round(a.elapsed_time(b) / 10, 4), "ms")
