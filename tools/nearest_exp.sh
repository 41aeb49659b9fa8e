for cfg in cfg2 cfg1 sta-paper; do
for v in "" "--debug das_fp=2 --debug das_ft=2" "--debug das_fp=1 --debug das_ft=4" "--debug das_tjc=32" "--debug das_fp=2 --debug das_ft=2 --debug das_tjc=32"; do
  python bench.py --steps 20 --no-cpu --no-stai --no-e2e --config $cfg --interp nearest $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$v', d['value'], d['stages_ms_per_frame']['das'], r['frac'], r['launch_shape'])"
done; done
