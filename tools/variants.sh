timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.log 2>&1
echo "[default] $(tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['binding']['frac'])")"
python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as E
ctx, grid, n_s = E.config_geometry("cfg2")
rf = torch.randn(8, ctx.n_tx, ctx.n_elements, n_s, device="cuda")
for apod in (bm.ApodizationSpec(), bm.ApodizationSpec("hann", 1.5), bm.ApodizationSpec("rectangular", 1.5), bm.ApodizationSpec("hann", 0.0)):
    plan = bm.DasPlan(ctx, grid, apod, np.float32, ctx.n_elements)
    out = plan.beamform_batch(rf); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): plan.beamform_batch(rf, out=out)
    e1.record(); torch.cuda.synchronize()
    print(apod, plan.kernel_for(n_s), "ms/frame", round(e0.elapsed_time(e1) / 24, 4))
PY
