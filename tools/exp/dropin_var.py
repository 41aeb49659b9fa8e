"""Drop-in rate variance: per-round rates of bench.dropin_fps on one box."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1811_01566_b200 as bm  # noqa: E402

ctx, grid, n_s = bm.environment.config_geometry("cfg2")
host = bench.synth_frames(ctx, n_s, 8, 0)
for _ in range(3):
    t0 = time.perf_counter()
    r = bench.dropin_fps(ctx, grid, host, "linear")
    print("median of 3 rounds", round(r, 1), "in", round(time.perf_counter() - t0, 2), "s")
r1 = bench.dropin_fps(ctx, grid, host[:1], "linear")
print("one cached frame", round(r1, 1))
