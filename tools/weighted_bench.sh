# weighted-apodisation and wide-pitch DAS configs (bench lines, 32 frames)
for a in "--window hann" "--window hann --f-number 1.5" "--window rectangular --f-number 1.5" "--config pwi-paper" "--config sta-paper --window hann --f-number 1.5"; do
  python bench.py --steps 20 --no-cpu --no-e2e --no-stai $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$a', d['value'], d['stages_ms_per_frame'], r['bound'], r['frac'], r['launch_shape'])"
done
