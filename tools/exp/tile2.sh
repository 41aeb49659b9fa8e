one() {
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
for t in 2 3 4; do
  one "cfg1 tile=$t" --config cfg1 --debug das_tile=$t
  one "cfg2 tile=$t" --config cfg2 --debug das_tile=$t
  one "cfg2_nearest tile=$t" --config cfg2 --interp nearest --debug das_tile=$t
  one "sta_paper tile=$t" --config sta-paper --debug das_tile=$t
  one "sta_paper_nearest tile=$t" --config sta-paper --interp nearest --debug das_tile=$t
  one "cfg3 tile=$t" --config cfg3 --frames 8 --debug das_tile=$t
done
one "cfg1_nearest default" --config cfg1 --interp nearest
