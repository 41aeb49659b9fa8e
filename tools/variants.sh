timeout 600 python -m pytest tests/test_gpu_sigproc.py tests/test_gpu_pipeline.py -q -x > gpurun_out/pt_sig.log 2>&1; tail -3 gpurun_out/pt_sig.log
for v in "" "BM_FFT_KERNEL=smem"; do
  env $v timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.log 2>&1
  echo "[$v] $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms_per_launch'], d['stages_ms_per_frame'])")"
done
for c in cfg1 cfg3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bc_$c.log 2>&1
  echo "[$c] $(tail -1 gpurun_out/bc_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms_per_frame'])")"
done
