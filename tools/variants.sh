run() { env $1 timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e $2 > gpurun_out/bv.log 2>&1
  echo "[$1 $2] $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['binding']['frac'])")"; }
run "" ""
run "BM_DAS_TJC=32" ""
