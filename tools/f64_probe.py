"""f64 frames (the reference's oracle precision) through DasPlan: which kernel, how fast."""
import sys, numpy as np, torch
sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm
for cfg in ("cfg2", "cfg1"):
    ctx, grid, n_s = bm.environment.config_geometry(cfg)
    plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float64, ctx.n_elements)
    rf = torch.randn(8, len(ctx.tx_scheme), ctx.n_elements, n_s, device="cuda", dtype=torch.float64)
    for _ in range(2): plan.beamform_batch(rf)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): plan.beamform_batch(rf)
    e.record(); torch.cuda.synchronize()
    print(cfg, "f64 kernel", plan.kernel_for(n_s), "ms/frame", round(s.elapsed_time(e) / 24, 3))
