"""K2/K3 timing probe: the fused envelope->display kernel against envelope +
display as two launches, per BASELINE image shape (CUDA events, 32-frame
batches from the engine's own DAS output)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_01566_b200 as bm  # noqa: E402
from paper_1811_01566_b200 import _native as N  # noqa: E402
from paper_1811_01566_b200 import sigproc as S  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
wss = {}
for name, F in (("cfg2", 32), ("cfg1", 32), ("cfg3", 8), ("sta-paper", 8)):
    ctx, grid, n_s = bm.environment.config_geometry(name)
    n_z, n_x = grid.n_z, grid.n_x
    g = torch.Generator(device="cuda").manual_seed(0)
    if name == "cfg2":  # the bench's own data: DAS of the wire-phantom cine
        import bench

        eng = bm.BmodeEngine(ctx, grid)
        rf = torch.from_numpy(bench.synth_frames(ctx, n_s, F, 0)).cuda()
        x = eng.plan.beamform_batch(rf)
        del rf
    else:
        x = torch.randn((F, n_z, n_x), generator=g, device="cuda")
    disp = torch.empty_like(x)
    peak = torch.empty(F, dtype=torch.int32, device="cuda")
    st = torch.empty(F, dtype=torch.int32, device="cuda")
    lib = N.load()

    def fused():
        nb = int(lib.bm_sigproc_ws_bytes(N.SIG_ENVELOPE_DISPLAY, 0, F, n_z, n_x))
        key = (name, nb)
        if key not in wss:
            wss[key] = N.workspace(nb, x.device)
        N.call("bm_envelope_display", 0, x.data_ptr(), disp.data_ptr(), peak.data_ptr(),
               st.data_ptr(), F, n_z, n_x, 30.0, wss[key].data_ptr(), nb, N.stream_ptr())

    def envpk():
        S.envelope_peak_device(x, F, n_z, n_x)

    out = {"fused_us_per_frame": 1000 * timeit(fused) / F,
           "envelope_peak_us_per_frame": 1000 * timeit(envpk) / F}
    ref = disp.clone()
    with N.debug_overrides(no_fused_display=1):
        out["two_launch_us_per_frame"] = 1000 * timeit(fused) / F
        fused()
        torch.cuda.synchronize()
        out["bitwise_equal_two_launch"] = bool(torch.equal(ref, disp))
    for path in (1, 2, 3):
        with N.debug_overrides(fft_path=path, no_fused_display=1 if path > 1 else 0):
            out[f"path{path}_us_per_frame"] = 1000 * timeit(fused, 5) / F
    out["hbm_floor_us_per_frame"] = n_z * n_x * 8 / 6.45e12 * 1e6
    res[name] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}
    print(name, json.dumps(res[name]), flush=True)
json.dump(res, open("gpurun_out/k2_probe.json", "w"), indent=1)
