"""cProfile of the one-frame drop-in chain (cfg2): where the host time goes."""
import cProfile, pstats, sys
import numpy as np
import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm
from bench import synth_frames

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = synth_frames(ctx, n_s, 2, 0)
frames = [bm.RfFrame(host[i]) for i in range(2)]
g = bm.build_graph(bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                                        "z_positions": grid.z_positions.tolist()}))
for i in range(5):
    bm.execute(g, (frames[i % 2], ctx))[0]["dynamic_adjustment"].numpy()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(100):
    bm.execute(g, (frames[i % 2], ctx))[0]["dynamic_adjustment"].numpy()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
