one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one "cfg1 hann" --config cfg1 --window hann
one "cfg1 hann F1.5" --config cfg1 --window hann --f-number 1.5
one "pwi hann" --config pwi-paper --window hann
one "pwi hann F1.5" --config pwi-paper --window hann --f-number 1.5
one "cfg3 hann F1.5" --config cfg3 --window hann --f-number 1.5 --frames 8
