# DAS tile shape (das_tile: lane blocks 1 = 16x2, 2 = 8x4, 3 = 4x8, 4 = 2x16
# pixels) and stage width per weighted / wide-pitch config: binding-roof
# fraction of each, one line per run.
one() {  # $1 = label, rest = bench args
  l=$1; shift
  timeout 300 python bench.py --steps 10 --no-cpu --no-stai --no-e2e "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['value'], r['bound'], r['frac'], r.get('launch_shape'))" ||
    echo "$l FAILED"
}
for t in 1 2 3 4; do
  one "hann_f15 tile=$t" --config cfg2 --window hann --f-number 1.5 --debug das_tile=$t
  one "pwi_paper tile=$t" --config pwi-paper --debug das_tile=$t
  one "cfg1_nearest tile=$t" --config cfg1 --interp nearest --debug das_tile=$t
done
for j in 32 64; do
  one "hann_f15 tjc=$j" --config cfg2 --window hann --f-number 1.5 --debug das_tjc=$j
  one "pwi_paper tjc=$j" --config pwi-paper --debug das_tjc=$j
done
