# drop-in rate for each host chunk count (DasPlan.HOST_CHUNKS)
for k in 1 2 3 4 6; do
  python -c "
import sys; sys.path[:0]=['.']
import bench, paper_1811_01566_b200 as bm
bm.DasPlan.HOST_CHUNKS = $k
ctx, grid, n_s = bm.environment.config_geometry('cfg2')
host = bench.synth_frames(ctx, n_s, 8, 0)
print('chunks', $k, 'dropin fps', round(bench.dropin_fps(ctx, grid, host, 'linear', n_frames=96), 1))
"
done
