one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one "cfg1 nearest" --config cfg1 --interp nearest
one "cfg2 nearest" --config cfg2 --interp nearest
one "sta nearest" --config sta-paper --interp nearest
one "pwi nearest" --config pwi-paper --interp nearest
one "cfg3 nearest" --config cfg3 --interp nearest --frames 8
one "cfg1 linear" --config cfg1
