"""One-frame DAS (the drop-in path: every das_beamform / plugin call is one
frame): kernel time per config with CUDA events, the FP32-roof fraction at 9
lane-ops per contribution, and the drop-in chain rate."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1811_01566_b200 as bm  # noqa: E402

from paper_1811_01566_b200 import _native as N  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
write_json = "no_json=1" not in sys.argv  # the run under ncu must not overwrite it
for kv in (a for a in sys.argv[1:] if "=" in a and a != "no_json=1"):  # tuning hooks, e.g. das_tjc=64
    k, v = kv.split("=")
    N.load().bm_debug_set(N.DEBUG_KEYS[k], int(v))
only = args or ["cfg2", "cfg1", "cfg3", "cfg5", "sta-paper", "pwi-paper"]
res = {}
for name in only:
    ctx, grid, n_s = bm.environment.config_geometry(name)
    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, n_rx)
    g = torch.Generator(device="cuda").manual_seed(1)
    rf = torch.randn((1, ctx.n_tx, n_rx, n_s), generator=g, device="cuda")
    out = torch.empty((1,) + plan.shape, device="cuda")
    reps = 5 if name in ("cfg3", "cfg5") else 30
    for _ in range(3):
        plan.beamform_batch(rf, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.beamform_batch(rf, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    contrib = ctx.n_tx * n_rx * grid.n_z * grid.n_x
    t_fp32 = contrib * 9 / (148 * 128 * 1.965e9) * 1e3
    res[name] = {"das_ms": round(ms, 4), "fp32_roof_ms": round(t_fp32, 4),
                 "frac": round(t_fp32 / ms, 3), "shape": plan.launch_shape(n_s, 1)}
    print(name, json.dumps(res[name]), flush=True)
ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = bench.synth_frames(ctx, n_s, 8, 0)
res["dropin_fps_cfg2"] = round(bench.dropin_fps(ctx, grid, host, "linear"), 1)
print("dropin", res["dropin_fps_cfg2"])
if write_json:
    json.dump(res, open("gpurun_out/das1_probe.json", "w"), indent=1)
