# Per-config bench lines (BASELINE configs, paper presets, weighted and
# nearest variants) into gpurun_out/configs/, one JSON line each.
mkdir -p gpurun_out/configs
run() {  # $1 = name, rest = bench args
  n=$1; shift
  timeout 600 python bench.py --steps 20 --no-cpu --no-stai "$@" > gpurun_out/configs/$n.log 2>&1
  tail -1 gpurun_out/configs/$n.log > gpurun_out/configs/$n.jsonl
  python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/configs/{n}.jsonl").read())
    r = d.get("roofline") or {}
    print(n, d["value"], d.get("stages_ms_per_frame"), r.get("bound"), r.get("frac"),
          (d.get("e2e") or {}).get("value"))
except Exception as exc:
    print(n, "FAILED", exc)
PY
}
run cfg2 --config cfg2
run cfg2_nearest --config cfg2 --interp nearest
run cfg1 --config cfg1
run cfg1_nearest --config cfg1 --interp nearest
run cfg3 --config cfg3 --frames 8
run cfg4_256 --config cfg2 --frames 256 --steps 5 --no-e2e
run sta_paper --config sta-paper
run sta_paper_nearest --config sta-paper --interp nearest
run pwi_paper --config pwi-paper
run pwi_paper_nearest --config pwi-paper --interp nearest
run cfg2_hann --config cfg2 --window hann
run cfg2_hann_f15 --config cfg2 --window hann --f-number 1.5
run cfg5_cols --config cfg5 --steps 5
run cfg5_rows --config cfg5 --steps 5 --split rows
run cfg1_fp2ft2 --config cfg1 --no-e2e --debug das_fp=2 --debug das_ft=2
run cfg1_fpc8 --config cfg1 --no-e2e --debug das_fpc=8
