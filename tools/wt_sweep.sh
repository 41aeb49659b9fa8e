# Weighted (Hann, F = 1.5) cfg2 DAS: launch-shape sweep (frames per thread,
# warp groups, stage width), binding-roof fraction of each.
one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e --config cfg2 --window hann --f-number 1.5 "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one default
one "ft=2" --debug das_ft=2
one "ft=2 fp=1" --debug das_ft=2 --debug das_fp=1
one "fp=1" --debug das_fp=1
one "ft=1" --debug das_ft=1
one "ft=2 tjc=32" --debug das_ft=2 --debug das_tjc=32
one "fpc=8" --debug das_fpc=8
one "fpc=32" --debug das_fpc=32
