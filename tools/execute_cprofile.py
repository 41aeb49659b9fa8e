"""cProfile of execute() per frame: where the host time of one
reference-style call goes.  ``pwi-paper`` / ``sta-paper``: device-resident
RF; ``cfg2-host``: the drop-in case (numpy RF in, numpy display out)."""
import cProfile
import pstats
import sys

import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm  # noqa: E402
from paper_1811_01566_b200 import cli  # noqa: E402
from paper_1811_01566_b200.pipeline import _to_device_obs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "pwi-paper"
sort = sys.argv[2] if len(sys.argv) > 2 else "tottime"
if name == "cfg2-host":
    from bench import synth_frames

    ctx, grid, n_s = bm.environment.config_geometry("cfg2")
    host = synth_frames(ctx, n_s, 4, 0)
    g = bm.build_graph(bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                                            "z_positions": grid.z_positions.tolist()}))
    obs = [(bm.RfFrame(h), ctx) for h in host]
else:
    env = cli.preset_environment(name)
    g = bm.build_graph(cli.preset_pipeline(name))
    obs = [_to_device_obs(env.next_observation()) for _ in range(4)]
for i in range(10):
    bm.execute(g, obs[i % 4])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    bm.execute(g, obs[i % 4])
pr.disable()
pstats.Stats(pr).sort_stats(sort).print_stats(30)
