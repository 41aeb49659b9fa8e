run() { env $1 timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e $2 > gpurun_out/bv.log 2>&1
  echo "[$1 $2] $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['binding']['frac'])")"; }
run "" ""
run "BM_DAS_FP=1" ""
run "BM_DAS_TJC=32" ""
timeout 600 python -m pytest tests/test_gpu_das.py -q -x 2>&1 | tail -2
