"""GPU timeline of one drop-in execute (cfg2, numpy in -> numpy out): the
per-node CUDA-event times, the gaps between them, and the host wall time, so
the part of the frame the GPU is idle shows up."""
import statistics
import sys
import time

import torch

sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm  # noqa: E402
from bench import synth_frames  # noqa: E402
from paper_1811_01566_b200 import _native as N  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = synth_frames(ctx, n_s, 2, 0)
frame = bm.RfFrame(host[0])
spec = bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                            "z_positions": grid.z_positions.tolist()})
g = bm.build_graph(spec)
for _ in range(10):
    bm.execute(g, (frame, ctx))
torch.cuda.synchronize()
rows = []
for _ in range(50):
    outs, t = bm.execute(g, (frame, ctx))
    rows.append(t)
for name, _ in rows[0].stages:
    print(f"{name:22s} gpu ms {statistics.median(r.stage_ms(name) for r in rows):.4f}")
print("sum of stages", round(statistics.median(sum(ms for _, ms in r.stages) for r in rows), 4))
print("execute total (host) ms", round(statistics.median(r.total_ms for r in rows), 4))
# raw pieces on an idle GPU
dev = torch.device("cuda", 0)
x = torch.from_numpy(frame.data)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
from paper_1811_01566_b200 import _device as D  # noqa: E402
for what, fn in (("staged H2D", lambda: D.to_device(frame.data, dev)),
                 ("pinned->dev", None)):
    if fn is None:
        pin = x.pin_memory()
        fn = lambda: pin.to(dev, non_blocking=True)  # noqa: E731
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(((time.perf_counter() - t0) * 1e3, a.elapsed_time(b)))
    print(what, "wall ms %.4f  gpu ms %.4f" % tuple(statistics.median(v) for v in zip(*ts)))
d = torch.empty((512, 512), device=dev)
for what, fn in (("d2h pinned 1MB", lambda: torch.empty(d.shape, pin_memory=True).copy_(d, non_blocking=True)),):
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(((time.perf_counter() - t0) * 1e3, a.elapsed_time(b)))
    print(what, "wall ms %.4f  gpu ms %.4f" % tuple(statistics.median(v) for v in zip(*ts)))
