"""One cfg2 one-frame DAS launch with Hann apodisation (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
rf = torch.randn((1, ctx.n_tx, ctx.n_elements, n_s), device="cuda")
plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec("hann", 0.0), np.float32, ctx.n_elements)
for _ in range(4):
    out = plan.beamform_batch(rf)
torch.cuda.synchronize()
print("table", plan.delay_table(build=False) is not None)
