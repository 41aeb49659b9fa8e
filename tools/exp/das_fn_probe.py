"""das_beamform (function API) on numpy cfg2 frames: calls per second."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1811_01566_b200 as bm  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = bench.synth_frames(ctx, n_s, 4, 0)
frames = [bm.RfFrame(h) for h in host]
plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
for i in range(8):
    bm.das_beamform(frames[i % 4], ctx, grid, plan=plan)
t0 = time.perf_counter()
for i in range(100):
    img = bm.das_beamform(frames[i % 4], ctx, grid, plan=plan)
print("das_beamform numpy cfg2 calls/s", round(100 / (time.perf_counter() - t0), 1))
