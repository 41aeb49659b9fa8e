# pwi-paper with four warp groups per delay table (FP = 4) -- run against the
# experimental FP = 4 build (since reverted: no gain)
one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
one "pwi default" --config pwi-paper
one "pwi fp4" --config pwi-paper --debug das_fp=4
one "pwi nearest default" --config pwi-paper --interp nearest
one "pwi nearest fp4" --config pwi-paper --interp nearest --debug das_fp=4
