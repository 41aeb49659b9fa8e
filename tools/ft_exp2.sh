set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_das.py -q -x -k "two_frames or cine_batch" > gpurun_out/pt_das.log 2>&1; tail -3 gpurun_out/pt_das.log
run() { timeout 300 env BM_DAS_VERBOSE=1 $1 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e $2 > gpurun_out/bv.log 2>&1
  echo "[$1 $2] $(grep -m1 das_tma gpurun_out/bv.log) $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], r.get('kernel_ms_per_launch'), d.get('stages_ms_per_frame'))")"; }
for cfg in cfg2 cfg1 "cfg3 --frames 8" "cfg1 --interp nearest"; do
  for v in "BM_DAS_FP=2 BM_DAS_FT=2" "BM_DAS_FP=1 BM_DAS_FT=2"; do
    run "$v" "--config $cfg"
  done
done
