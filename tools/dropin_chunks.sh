# drop-in rate for each host-frame piece count (DasPlan.HOST_PIECES: transmit
# groups the upload lands one by one while the DAS launch reads them)
for k in 1 2 3 4 6 11; do
  python -c "
import sys; sys.path[:0]=['.']
import bench, paper_1811_01566_b200 as bm
bm.DasPlan.HOST_PIECES = $k
ctx, grid, n_s = bm.environment.config_geometry('cfg2')
host = bench.synth_frames(ctx, n_s, 8, 0)
print('pieces', $k, 'dropin fps', round(bench.dropin_fps(ctx, grid, host, 'linear'), 1))
"
done
