"""Host-side cost of each piece of the one-frame drop-in chain (cfg2):
wall time of each call with the GPU idle before it (synchronised), so the
numbers are what the host spends issuing the work plus any blocking."""
import sys
import time

import numpy as np
import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm  # noqa: E402
from bench import synth_frames  # noqa: E402
from paper_1811_01566_b200 import _device as D  # noqa: E402
from paper_1811_01566_b200 import pipeline as P  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = synth_frames(ctx, n_s, 2, 0)
frame = bm.RfFrame(host[0])
dev = torch.device("cuda", 0)
spec = bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                            "z_positions": grid.z_positions.tolist()})
g = bm.build_graph(spec)
for _ in range(5):
    bm.execute(g, (frame, ctx))[0]["dynamic_adjustment"].numpy()
torch.cuda.synchronize()


def host_ms(fn, n=50):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return round(sorted(ts)[n // 2] * 1e3, 4)


nodes = g.nodes
rf_dev = D.to_device(frame.data, dev)
img = nodes["beamform"].fn((frame, ctx))
an = nodes["analytic_signal"].fn(img)
env = nodes["envelope"].fn(an)
torch.cuda.synchronize()
print("to_device (staged) host ms", host_ms(lambda: D.to_device(frame.data, dev)))
print("beamform op (incl. H2D) host ms", host_ms(lambda: nodes["beamform"].fn((frame, ctx))))
plan = nodes["beamform"].fn._plan
print("beamform_batch launch host ms", host_ms(lambda: plan.beamform_batch(rf_dev)))
print("analytic op host ms", host_ms(lambda: nodes["analytic_signal"].fn(img)))
print("envelope op host ms", host_ms(lambda: nodes["envelope"].fn(an)))
print("dyn op host ms (incl. status sync)", host_ms(lambda: nodes["dynamic_adjustment"].fn(env)))
d = nodes["dynamic_adjustment"].fn(env)
print(".numpy() host ms", host_ms(lambda: d.numpy()))
print("execute host ms", host_ms(lambda: bm.execute(g, (frame, ctx))))
print("execute+numpy host ms", host_ms(lambda: bm.execute(g, (frame, ctx))[0]["dynamic_adjustment"].numpy()))
