"""One-frame cfg2 DAS time vs tile count (rows of the grid cropped): how much
the partial last wave costs (2 CTAs/SM x 148 SMs = 296 slots)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
rf = torch.randn((1, ctx.n_tx, ctx.n_elements, n_s), device="cuda")
for rows in (128, 144, 288, 296, 432, 448, 512):
    g = bm.ImageGrid(grid.x_positions.copy(), grid.z_positions[:rows].copy())
    plan = bm.DasPlan(ctx, g, bm.ApodizationSpec(), np.float32, ctx.n_elements)
    out = plan.beamform_batch(rf)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30):
        plan.beamform_batch(rf, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 30
    tiles = ((rows + 15) // 16) * 32
    print(f"rows {rows} tiles {tiles} waves {tiles / 296:.2f} ms {ms:.4f} ms/tile-wave-equiv "
          f"{ms / (tiles / 296):.4f}")
