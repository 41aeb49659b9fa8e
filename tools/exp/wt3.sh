one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'])" ||
    echo "$l FAILED"
}
one "cfg2 hann" --config cfg2 --window hann
one "cfg2 hann F1.5" --config cfg2 --window hann --f-number 1.5
one "cfg2 rect F1.5" --config cfg2 --f-number 1.5
one "sta hann F1.5" --config sta-paper --window hann --f-number 1.5
one "cfg2 uniform" --config cfg2
