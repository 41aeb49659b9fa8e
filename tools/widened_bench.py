"""Measurement of the widened rows on one B200:
device time of each kernel on cfg2-sized inputs (CUDA events on the launching
stream, after warm-up, median of the timed launches), its roof, and the CPU
restatement of the reference on the same input for context.  One JSON line
per kernel on stdout.

  * bm_fir_filter       cfg2 frame [11, 128, 2048] f32 -> f64, 64 taps
                        (sigproc.py:36-45); FP64 pipe: 2 DP ops per tap
  * bm_sliding_moments  512 x 512 f32 envelope, 16 x 16 windows, stride 1
                        (qus.py:122-158); FP64 pipe: x^2, x^3 and three
                        Kahan-compensated sums (4 DP ops each) = 14 per
                        element and placement
  * bm_quantize_u8      32 cfg2 display frames f32 -> u8 (formats.py:189-200);
                        HBM: 4 B read + 1 B written per pixel
  * bm_simulate_rf      cfg2 wire frame [11, 128, 2048] f32 (environment.py:
                        91-129); timed against the host simulator

FP64 peak: 148 SMs x 64 DP FMA/clk x 2 at the NVML SM clock (nominal, not in
MEASURED_PEAKS.json); HBM peak: MEASURED_PEAKS.json.  Both FP64 kernels issue
one DP instruction per counted op (rounded products and sums kept separate,
no FMA), so their instruction roof is half the nominal FLOP peak:
dp_issue_frac = achieved ops/s / (148 x 64 x f)."""

import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_01566_b200 as bm  # noqa: E402
from paper_1811_01566_b200 import _native as N  # noqa: E402
from paper_1811_01566_b200 import environment as ME  # noqa: E402
from oracle import oracle as O  # noqa: E402  (CPU context only)


def sm_mhz():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    except Exception:
        return 1965.0


def time_launch(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def cpu_time(fn, budget=5.0):
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        el = time.perf_counter() - t0
        if el > budget or n >= 20:
            return el / n * 1e3, n


def main():
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = sm_mhz()
    fp64_peak = n_sm * 64 * 2 * mhz * 1e6 / 1e12  # TFLOP/s
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm_peak = peaks["hbm_gbs"]
    s = N.stream_ptr()
    lines = []

    ctx, grid, n_s = ME.config_geometry("cfg2")
    frame = ME.simulate_rf(ME.wire_phantom(), ctx, n_s, dtype=np.float32)
    x_h = np.ascontiguousarray(frame.data)

    # ---- FIR -----------------------------------------------------------------
    taps = np.hanning(66)[1:-1] * np.cos(2 * np.pi * 5e6 / 40e6 * (np.arange(64) - 31.5))
    taps = taps / np.abs(taps).sum()
    x = torch.from_numpy(x_h).to(dev)
    y = torch.empty(x.shape, dtype=torch.float64, device=dev)
    h = torch.from_numpy(taps).to(dev)
    outer, n, inner = x.numel() // n_s, n_s, 1
    ms = time_launch(lambda: N.call("bm_fir_filter", N.BM_F32, x.data_ptr(), N.BM_F64,
                                    y.data_ptr(), outer, n, inner, h.data_ptr(), 64, s))
    flops = 2.0 * 64 * x.numel()
    byts = x.numel() * (4 + 8)
    ref = O.fir_filter(x_h, taps, axis=-1)
    err = float(np.abs(y.cpu().numpy() - ref).max() / max(np.abs(ref).max(), 1e-300))
    cms, cn = cpu_time(lambda: O.fir_filter(x_h, taps, axis=-1))
    lines.append({"kernel": "bm_fir_filter", "workload": "cfg2 frame 11x128x2048 f32 -> f64, 64 taps",
                  "ms": round(ms, 4), "bound": "fp64",
                  "achieved_tflops": round(flops / ms / 1e9, 3), "peak_tflops": round(fp64_peak, 2),
                  "frac": round(flops / ms / 1e9 / fp64_peak, 3),
                  "dp_issue_frac": round(2 * flops / ms / 1e9 / fp64_peak, 3),
                  "hbm_gbs": round(byts / ms / 1e6, 1), "hbm_frac": round(byts / ms / 1e6 / hbm_peak, 3),
                  "max_rel_err_vs_oracle": err,
                  "cpu_ms": round(cms, 3), "cpu_kind": "port (scipy lfilter)", "cpu_runs": cn})

    # ---- sliding moments -----------------------------------------------------
    rng = np.random.default_rng(0)
    img_h = rng.rayleigh(size=(512, 512)).astype(np.float32)
    img = torch.from_numpy(img_h).to(dev)
    wh = ww = 16
    orr, oc = 512 - wh + 1, 512 - ww + 1
    m = torch.empty((3, orr, oc), dtype=torch.float64, device=dev)
    ms = time_launch(lambda: N.call("bm_sliding_moments", N.BM_F32, img.data_ptr(), 512, 512, wh, ww,
                                    1, 1, m[0].data_ptr(), m[1].data_ptr(), m[2].data_ptr(), s))
    flops = 14.0 * wh * ww * orr * oc
    ref = O.sliding_moments(img_h, (wh, ww), (1, 1))
    mm = m.cpu().numpy()
    err = max(float(np.abs(mm[i] - np.asarray(r)).max() / np.abs(np.asarray(r)).max())
              for i, r in enumerate(ref[:3]))
    cms, cn = cpu_time(lambda: O.sliding_moments(img_h, (wh, ww), (1, 1)))
    lines.append({"kernel": "bm_sliding_moments", "workload": "512x512 f32, 16x16 windows, stride 1",
                  "ms": round(ms, 4), "bound": "fp64",
                  "achieved_tflops": round(flops / ms / 1e9, 3), "peak_tflops": round(fp64_peak, 2),
                  "frac": round(flops / ms / 1e9 / fp64_peak, 3),
                  "dp_issue_frac": round(2 * flops / ms / 1e9 / fp64_peak, 3),
                  "max_rel_err_vs_oracle": err,
                  "cpu_ms": round(cms, 3), "cpu_kind": "port (numpy)", "cpu_runs": cn})

    # ---- quantize ------------------------------------------------------------
    disp_h = rng.random((32, 512, 512), dtype=np.float32)
    disp = torch.from_numpy(disp_h).to(dev)
    q = torch.empty(disp.shape, dtype=torch.uint8, device=dev)
    ms = time_launch(lambda: N.call("bm_quantize_u8", N.BM_F32, disp.data_ptr(), q.data_ptr(),
                                    disp.numel(), s))
    byts = disp.numel() * 5
    ref = np.floor(disp_h * np.float32(255) + np.float32(0.5)).astype(np.uint8)  # f32 ops
    same = bool(np.array_equal(q.cpu().numpy(), ref))
    cms, cn = cpu_time(lambda: np.floor(disp_h * 255 + 0.5).astype(np.uint8))
    lines.append({"kernel": "bm_quantize_u8", "workload": "32 cfg2 displays 512x512 f32 -> u8",
                  "ms": round(ms, 4), "bound": "hbm",
                  "achieved_gbs": round(byts / ms / 1e6, 1), "peak_gbs": hbm_peak,
                  "frac": round(byts / ms / 1e6 / hbm_peak, 3), "bitwise_equal_numpy_f32": same,
                  "cpu_ms": round(cms, 3), "cpu_kind": "numpy", "cpu_runs": cn})

    # ---- simulator -----------------------------------------------------------
    ph = ME.wire_phantom()
    ms = time_launch(lambda: ME.simulate_rf_device(ph, ctx, n_s, dtype=np.float32), reps=10)
    d = ME.simulate_rf_device(ph, ctx, n_s, dtype=np.float32).cpu().numpy()
    same = bool(np.array_equal(d, x_h))
    cms, cn = cpu_time(lambda: ME.simulate_rf(ph, ctx, n_s, dtype=np.float32), budget=3.0)
    lines.append({"kernel": "bm_simulate_rf", "workload": "cfg2 wire frame 11x128x2048 f32",
                  "ms": round(ms, 4), "bound": "launch/geometry upload (3 scatterers)",
                  "bitwise_equal_host": same,
                  "cpu_ms": round(cms, 3), "cpu_kind": "host restatement (numpy)", "cpu_runs": cn})

    for ln in lines:
        ln["sm_mhz"] = mhz
        print(json.dumps(ln))


if __name__ == "__main__":
    main()
