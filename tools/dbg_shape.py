import os, sys, numpy as np, torch
sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm
os.environ["BM_DAS_FPC"] = "8"
for nz, nx in ((90, 70), (240, 100), (300, 140), (400, 140)):
  for scheme in (bm.StaScheme(tuple(range(0, 48, 5))), bm.PwScheme(tuple(np.deg2rad([-7.0, 0.0, 9.0])))):
    ctx = bm.AcquisitionContext(1540.0, 40e6, 48, 2e-4, scheme)
    ex = ctx.element_positions()
    grid = bm.ImageGrid(np.linspace(ex[0], ex[-1], nx), np.linspace(2e-3, 25e-3, nz))
    plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, 48)
    print(nz, nx, type(scheme).__name__, "W", plan._geom.window_hint_g4, plan.launch_shape(1024, 11, "linear"), flush=True)
