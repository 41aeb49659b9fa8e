one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one "cfg1" --config cfg1
one "cfg1 nearest" --config cfg1 --interp nearest
one "cfg1 ft2" --config cfg1 --debug das_ft=2
one "cfg1 fpc8" --config cfg1 --debug das_fpc=8
one "cfg1 tile4" --config cfg1 --debug das_tile=4
