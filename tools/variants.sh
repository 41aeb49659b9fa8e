python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as E
for c in ("cfg1","cfg2","cfg3","cfg5"):
    ctx, grid, n_s = E.config_geometry(c)
    plan = bm.DasPlan(ctx, grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
    print(c, "W", plan.fast_window, "W_g4", plan.tma_window)
PY
for c in cfg1 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bc_$c.log 2>&1
  echo "[$c] $(tail -1 gpurun_out/bc_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['unit'], r.get('kernel'), r.get('kernel_ms_per_launch'), r.get('binding',{}).get('frac'), d.get('stages_ms_per_frame'))")"
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
