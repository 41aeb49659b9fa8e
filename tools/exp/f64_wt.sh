one() {
  l=$1; shift
  timeout 300 python bench.py --steps 5 --frames 8 --no-cpu --no-stai --no-e2e --dtype f64 "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], d['stages_ms_per_frame'])" ||
    echo "$l FAILED"
}
one "f64 cfg2" --config cfg2
one "f64 cfg2 hann" --config cfg2 --window hann
one "f64 cfg2 hann F1.5" --config cfg2 --window hann --f-number 1.5
one "f64 sta hann F1.5" --config sta-paper --window hann --f-number 1.5
