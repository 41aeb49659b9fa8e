run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $1 > gpurun_out/bv.log 2>&1
  echo "[$1] $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], d['ms_per_step'], r.get('kernel_ms_per_launch'), d.get('stages_ms_per_frame'), d['config'].get('workload'))")"; }
run "--interp nearest"
run "--config cfg1 --interp nearest"
run "--frames 256 --steps 4"
