set -u
mkdir -p gpurun_out
cat > /tmp/h.py <<'PY'
import sys, hashlib, numpy as np, torch
sys.path[:0] = ["."]
import paper_1811_01566_b200 as bm
cfg, nf = sys.argv[1], int(sys.argv[2])
ctx, grid, n_s = bm.environment.config_geometry(cfg)
plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
g = torch.Generator(device="cuda").manual_seed(5)
rf = torch.randn((nf, len(ctx.tx_scheme), ctx.n_elements, n_s), generator=g, device="cuda")
out = plan.beamform_batch(rf, "linear")
torch.cuda.synchronize()
print("H", cfg, nf, hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16])
PY
for c in "cfg2 32" "cfg2 13" "cfg1 16"; do
  for v in "1 1" "2 4" "1 4"; do
    set -- $v
    echo "FP=$1 FT=$2 $(BM_DAS_VERBOSE=1 BM_DAS_FP=$1 BM_DAS_FT=$2 BM_DAS_FPC=8 timeout 300 python /tmp/h.py $c 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
run() { timeout 300 env BM_DAS_VERBOSE=1 $1 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e $2 > gpurun_out/bv.log 2>&1
  echo "[$1 $2] $(grep -m1 das_tma gpurun_out/bv.log) $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], r.get('kernel_ms_per_launch'), d.get('stages_ms_per_frame'))")"; }
for cfg in cfg2 cfg1 "cfg3 --frames 8"; do
  for v in "BM_DAS_FP=2 BM_DAS_FT=2" "BM_DAS_FP=2 BM_DAS_FT=4" "BM_DAS_FP=1 BM_DAS_FT=4"; do
    run "$v" "--config $cfg"
  done
done
