"""Where the time of the one-frame drop-in call goes (cfg2): pageable H2D,
the single-frame DAS, the rest of the chain, the D2H of the display."""
import sys, time
import numpy as np
import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm
from bench import synth_frames

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = synth_frames(ctx, n_s, 4, 0)
frames = [bm.RfFrame(host[i]) for i in range(4)]
dev = torch.device("cuda", 0)


def t(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("h2d pageable torch.from_numpy().to(dev) ms", t(lambda: torch.from_numpy(host[0]).to(dev)))
pin = torch.empty(host[0].shape, dtype=torch.float32).pin_memory()
print("np->pinned memcpy ms", t(lambda: pin.copy_(torch.from_numpy(host[0]))))
print("h2d pinned ms", t(lambda: pin.to(dev, non_blocking=True)))
plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
rf1 = torch.from_numpy(host[0]).to(dev)
print("das 1 frame ms", t(lambda: plan.beamform_batch(rf1, "linear")))
print("shape 1 frame", plan.launch_shape(n_s, 1))
spec = bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                            "z_positions": grid.z_positions.tolist()})
g = bm.build_graph(spec)
i = [0]


def ex():
    outs, tm = bm.execute(g, (frames[i[0] % 4], ctx))
    i[0] += 1
    return outs


print("execute (no readback) ms", t(ex))
print("execute + numpy ms", t(lambda: ex()["dynamic_adjustment"].numpy()))
outs, tm = bm.execute(g, (frames[0], ctx))
print("stages", tm.stages, "total", tm.total_ms)

from paper_1811_01566_b200 import _device as D  # noqa: E402

print("staged to_device ms", t(lambda: D.to_device(host[0], dev)))
for step_div in (1, 2, 4, 8):
    def staged(div=step_div):
        src = torch.from_numpy(host[0]).reshape(-1)
        n = src.numel()
        step = -(-n // div)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        for o in range(0, n, step):
            pin[:].view(-1)[o:o + step].copy_(src[o:o + step])
            out[o:o + step].copy_(pin.view(-1)[o:o + step], non_blocking=True)
        return out
    print("manual staged chunks", step_div, "ms", t(staged))
img_h = np.empty(grid.shape, np.float32)
dd = torch.empty(grid.shape, device=dev)
print("d2h 1 MB .cpu() ms", t(lambda: dd.cpu()))
r1 = bm.RfFrame(host[0])
print("das_beamform drop-in (numpy in, numpy out) ms", t(lambda: bm.das_beamform(r1, ctx, grid, plan=plan)))
