"""cProfile of execute() per frame for a paper preset (device-resident RF):
where the host time of one reference-style call goes."""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm  # noqa: E402
from paper_1811_01566_b200 import cli  # noqa: E402
from paper_1811_01566_b200.pipeline import _to_device_obs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "pwi-paper"
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
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
