"""f64 DAS (the reference's oracle precision, the paper's Titan X runs):
one-frame and 8-frame launches per config, generic kernel."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402

res = {}
for name in sys.argv[1:] or ["cfg2", "cfg1", "sta-paper", "pwi-paper"]:
    ctx, grid, n_s = bm.environment.config_geometry(name)
    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float64, n_rx)
    g = torch.Generator(device="cuda").manual_seed(1)
    for F in (1, 8):
        rf = torch.randn((F, ctx.n_tx, n_rx, n_s), generator=g, device="cuda", dtype=torch.float64)
        out = torch.empty((F,) + plan.shape, device="cuda", dtype=torch.float64)
        for _ in range(2):
            plan.beamform_batch(rf, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            plan.beamform_batch(rf, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3 / F
        res[f"{name}_F{F}"] = {"ms_per_frame": round(ms, 4), "kernel": plan.kernel_for(n_s)}
        print(name, F, res[f"{name}_F{F}"], flush=True)
json.dump(res, open("gpurun_out/f64_probe.json", "w"), indent=1)
