for c in cfg1 cfg2 cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bc_$c.log 2>&1
  echo "[$c] $(tail -1 gpurun_out/bc_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], d['unit'], r.get('kernel'), r.get('kernel_ms_per_launch'), r.get('binding',{}).get('frac'), d.get('stages_ms_per_frame'), d.get('ms_per_step'))")"
done
for c in cfg1 cfg3; do
  BM_DAS_FP=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bx_$c.log 2>&1
  echo "[FP1 $c] $(tail -1 gpurun_out/bx_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], r.get('kernel_ms_per_launch'), r.get('binding',{}).get('frac'))")"
done
