one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e --config cfg2 --window hann --f-number 1.5 "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one "fp=1 tjc=16" --debug das_fp=1 --debug das_tjc=16
one "rect F1.5" --window rectangular
one "hann F1.0" --f-number 1.0
one "hann F3" --f-number 3.0
