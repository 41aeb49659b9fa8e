set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_das.py -q -x -k "contiguous" > gpurun_out/pt_tile.log 2>&1; tail -2 gpurun_out/pt_tile.log; grep -E "^E   " gpurun_out/pt_tile.log | head -6
run() { timeout 300 env BM_DAS_VERBOSE=1 $1 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $2 > gpurun_out/bv.log 2>&1
  echo "[$1 $2] $(grep -m1 das_tma gpurun_out/bv.log | cut -c1-60) $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], d.get('stages_ms_per_frame')['das'], r['binding']['frac'])")"; }
for cfg in sta-paper "sta-paper --interp nearest" pwi-paper cfg1 cfg2 "cfg3 --frames 8"; do
  for t in 3 2 1 4; do
    run "BM_DAS_TILE=$t" "--config $cfg"
  done
done
