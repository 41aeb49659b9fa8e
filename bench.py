#!/usr/bin/env python
"""B-mode frames/sec on B200 -- BASELINE.json metric, config 2 at N = 1.

Workload (one "step" per GPU): B PWI frames of BASELINE config 2
(128 elements, 11 plane-wave angles, 2048 samples, 512 x 512 image, f32,
linear interpolation, rectangular apodisation, 30 dB) reconstructed by the
full chain  DAS -> analytic signal -> envelope -> dB clip.  Frames are
partitioned across ranks with no data-path collective (config 4's cine
stream split over GPUs; at N = 8 and B = 32 a step is the whole 256-frame
cine of config 4), so scaling is "weak".

`value`: device-resident throughput (RF already in HBM; B x 11.5 MB per
GPU > 126 MB L2, so no L2 flush is needed between steps).
`e2e`:   the same metric through the public engine API from pinned HOST
buffers, H2D of the RF and D2H of the display inside the timed region.

--impl reference: the CPU restatement of the reference (oracle/: C DAS
kernel + scipy.fft analytic signal + numpy dB) on all host cores, rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "cfg1": "cfg1 STAI 64el x 64tx x 2048 samples -> 256x256, DAS+envelope+dB30, linear",
    "cfg2": "cfg2 PWI 128el x 11 angles x 2048 samples -> 512x512, DAS+envelope+dB30, linear",
    "cfg3": "cfg3 STAI 128el x 128tx x 4096 samples -> 1024x512, DAS+envelope+dB30, linear",
    "sta-paper": "sta-paper STAI 128el x 128tx x 64 rx (centred map) x 2048 samples -> 2048x128, "
                 "DAS+envelope+dB30, linear",
    "pwi-paper": "pwi-paper PWI 192el x 11 angles x 2048 samples -> 512x128, DAS+envelope+dB30, "
                 "linear",
}
WORKLOAD = WORKLOADS["cfg2"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--frames", type=int, default=32, help="frames per GPU per step")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--interp", default="linear")
    ap.add_argument("--split", default="cols", choices=["cols", "rows"],
                    help="cfg5: split one frame by image columns (rank-local FFT, gather of "
                         "display tiles) or by depth rows (gather of RF rows, K2 on rank 0)")
    ap.add_argument("--window", default="rectangular", choices=["rectangular", "hann"],
                    help="receive apodisation window (ApodizationSpec)")
    ap.add_argument("--f-number", type=float, default=0.0,
                    help="dynamic-aperture f-number (0: all elements)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def synth_frames(ctx, n_s, n_frames, seed0):
    """Wire phantom (presets.py:41-51) + N(0, 0.01) noise per frame, f32."""
    import paper_1811_01566_b200 as bm

    clean = bm.simulate_rf(bm.wire_phantom(), ctx, n_s, dtype=np.float64).data
    out = np.empty((n_frames,) + clean.shape, np.float32)
    for i in range(n_frames):
        rng = np.random.default_rng(seed0 + i)
        out[i] = (clean + rng.normal(0.0, 0.01, clean.shape)).astype(np.float32)
    return out


def dropin_fps(ctx, grid, host, interp, n_frames=48, warmup=4):
    """Frames/s a reference user sees calling the drop-in operator chain one
    frame at a time: ``execute(build_graph(bmode_chain(...)), (RfFrame, ctx))``
    with numpy RF in and the numpy display read back (pageable H2D/D2H and a
    synchronisation per frame).  RfFrame construction (the reference's host
    finiteness scan) happens before the clock, as in echopipe's own
    benchmark()."""
    import paper_1811_01566_b200 as bm

    spec = bm.bmode_chain(interpolation=interp,
                          grid={"x_positions": grid.x_positions.tolist(),
                                "z_positions": grid.z_positions.tolist()})
    graph = bm.build_graph(spec)
    frames = [bm.RfFrame(host[i]) for i in range(min(len(host), 8))]
    for i in range(warmup):
        outs, _ = bm.execute(graph, (frames[i % len(frames)], ctx))
        outs["dynamic_adjustment"].numpy()
    t0 = time.perf_counter()
    for i in range(n_frames):
        outs, _ = bm.execute(graph, (frames[i % len(frames)], ctx))
        outs["dynamic_adjustment"].numpy()
    return n_frames / (time.perf_counter() - t0)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms by a
    background nvidia-smi loop (the recipe's clocks line) while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._p = None
        self._t = None
        self._mark = 0

    def _read(self):
        for line in self._p.stdout:
            parts = [c.strip() for c in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def start(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None

    def mark(self):
        """Only samples taken after this call count."""
        self._mark = len(self.rows)

    def stop(self):
        if self._p is not None:
            time.sleep(0.25)  # let the sample covering the end of the region land
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            if self._t:
                self._t.join(timeout=5)
        rows = self.rows[self._mark:] or self.rows[-1:]
        num = lambda x: x.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[0]) for r in rows if num(r[0])]
        mx = [float(r[1]) for r in rows if num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_reference(ctx, grid, frames, seconds, interp, max_frames=None):
    """Reference algorithm on the host (oracle/ port): frames/s, threads."""
    from oracle import oracle as O

    plan = O.Plan(ctx, grid, "rectangular", 0.0, np.float32, frames.shape[2])
    O.bmode_chain(frames[0], ctx, grid, interp=interp, plan=plan)  # warm (thread spin-up)
    t0 = time.perf_counter()
    n = 0
    while True:
        O.bmode_chain(frames[n % len(frames)], ctx, grid, interp=interp, plan=plan)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_frames and n >= max_frames):
            break
    return n / el, O.max_threads(), n, el


def run_cfg5(args, ctx, grid, n_s, rank, world, local, dev):
    """BASELINE config 5: one 2048 x 2048 STAI frame per step, image columns
    split across ranks (parallel.LateralSplit), one all-reduce(MAX) of the
    peak and one all-gather of display slabs per frame (strong scaling)."""
    import torch

    import paper_1811_01566_b200 as bm
    from paper_1811_01566_b200 import parallel as P

    rows = args.split == "rows"
    split = (P.RowSplit if rows else P.LateralSplit)(grid, world, rank)
    eng = bm.BmodeEngine(ctx, split.sub_grid)
    frame = torch.from_numpy(synth_frames(ctx, n_s, 1, 0)).to(dev)  # replicated RF
    _, rf_img, env, peak, status = eng._buffers(1)

    def step():
        if rows:
            # DAS of this rank's depth band, RF bands gathered, K2 on rank 0
            eng.plan.beamform_batch(frame, eng.interp, out=rf_img[:1])
            full = split.gather(rf_img[0]) if world > 1 else rf_img[0]
            return P.envelope_display(full, eng.range_db)[0] if full is not None else None
        eng.reconstruct(frame)  # DAS + envelope + local peak of this slab
        if world > 1:
            return split.display(env[0], eng.range_db)
        return P.map_display(env[0], float(env[0].max()), eng.range_db)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    if rank == 0:
        print(json.dumps({
            "metric": "B-mode frames/sec", "value": round(args.steps / (ms / 1000.0), 3),
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic wire phantom + N(0,0.01)",
            "config": {"workload": "cfg5 STAI 128el x 128tx x 4096 samples -> 2048x2048, " + (
                "depth-row split, all-gather of RF rows, envelope + display on rank 0" if rows else
                "lateral column split, all-reduce(max) + all-gather of display slabs"),
                       ("rows_per_rank" if rows else "columns_per_rank"): split.hi - split.lo},
            "e2e": None, "gpu_launches": 3 * args.steps}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import paper_1811_01566_b200 as bm
    from paper_1811_01566_b200 import environment as ME

    ctx, grid, n_s = ME.config_geometry(args.config)
    global WORKLOAD
    WORKLOAD = WORKLOADS.get(args.config, WORKLOAD).replace("linear", args.interp)
    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    frame_bytes = ctx.n_tx * n_rx * n_s * 4
    img_bytes = grid.n_z * grid.n_x * 4

    if args.impl == "reference":
        if rank != 0:
            return
        frames = synth_frames(ctx, n_s, 2, 0)
        times = []
        for i in range(args.warmup + args.steps):
            fps, cores, n, el = cpu_reference(ctx, grid, frames, 0.0, args.interp, max_frames=1)
            if i >= args.warmup:
                times.append(el / n)
        ms = statistics.median(times) * 1000.0
        val = 1000.0 / ms
        print(json.dumps({
            "impl": "reference", "metric": "B-mode frames/sec", "value": round(val, 4),
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic wire phantom + N(0,0.01)",
            "config": {"workload": WORKLOAD, "frames_per_step": 1},
            "cpu_baseline": {"value": round(val, 4), "unit": "frames/s", "cores": cores,
                             "kind": "port",
                             "sample": f"1 {args.config} frame per step: oracle/ C DAS (pthreads, all "
                                       "cores) + scipy.fft analytic + numpy dB"},
            "e2e": {"value": round(val, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    if args.config == "cfg5":
        return run_cfg5(args, ctx, grid, n_s, rank, world, local, dev)

    B = args.frames
    host = synth_frames(ctx, n_s, B, seed0=rank * B)
    apod = bm.ApodizationSpec(args.window, args.f_number)
    eng = bm.engine.BmodeEngine(ctx, grid, apod=apod, interp=args.interp, dtype=np.float32)
    if not eng.plan.uniform:
        WORKLOAD = WORKLOAD + f", {args.window} F={args.f_number:g}"
    rf = torch.from_numpy(host).to(dev)
    out = torch.empty((B, grid.n_z, grid.n_x), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region --------------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        eng.reconstruct(rf, out=out)
    torch.cuda.synchronize()
    eng.check()
    das_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    clocks.mark()  # keep only samples taken from here on
    launches0 = eng.launches
    barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record()
    for k in range(args.steps):
        # the DAS launch is bracketed by events on its own stream, for the roofline
        eng.reconstruct(rf, out=out, stream=stream, das_events=das_ev[k])
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = eng.launches - launches0
    ms_total = max_over_ranks(t_start.elapsed_time(t_end))
    ms_step = ms_total / args.steps
    das_ms = statistics.mean(a.elapsed_time(b) for a, b in das_ev)
    value = world * B * args.steps / (ms_total / 1000.0)

    # ---- end-to-end through the public API from pinned host memory ----------
    e2e = None
    if not args.no_e2e:
        rf_h, disp_h = eng.pinned(B, n_s)
        rf_h.copy_(torch.from_numpy(host))
        eng.reconstruct_host_stream([(rf_h, disp_h)] * max(1, args.warmup))
        e2e_steps = max(3, args.steps // 2)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # every step: H2D of its 32 RF frames from pinned host memory, the
        # chain, D2H of its 32 displays; steps are pipelined back to back and
        # the clock stops when the last display is on the host
        eng.reconstruct_host_stream([(rf_h, disp_h)] * e2e_steps)
        el = max_over_ranks(time.perf_counter() - t0)
        eng.check()
        e2e = {"value": round(world * B * e2e_steps / el, 2), "unit": "frames/s",
               "h2d_bytes_per_step": B * frame_bytes, "d2h_bytes_per_step": B * img_bytes,
               "ms_per_step": round(el / e2e_steps * 1000.0, 3)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    if e2e is not None and world == 1:
        e2e["dropin_per_frame_fps"] = round(dropin_fps(ctx, grid, host, args.interp), 1)
        e2e["dropin_note"] = ("one frame per call through the reference-facing operator chain "
                              "(numpy in, numpy display out, pageable copies); value above is "
                              "the batched engine from pinned memory")

    # ---- roofline of the dominant kernel (DAS) ------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    das_bytes = B * (frame_bytes + img_bytes)  # algorithmic HBM bytes per launch
    achieved = das_bytes / (das_ms / 1000.0) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "das_traffic.json")))
        if prof.get("workload") == WORKLOAD and prof.get("interp") == args.interp:
            traffic = prof["dram_bytes_per_frame"] * B
    except Exception:
        pass
    contrib = B * ctx.n_tx * n_rx * grid.n_z * grid.n_x
    span = eng.plan._bufs.get("span")
    if span is not None and eng.plan._geom.rx_identity:
        # F-number gate: terms outside a pixel's active span have weight 0 and
        # are exact zeros the kernel may skip, so the algorithmic work is the
        # active contributions (identity / contiguous maps: the span clipped
        # to the elements each transmit records)
        sp = span.view(-1, 2).to(torch.int64)
        lo, hi = sp[:, 0].clamp(min=0), sp[:, 1].clamp(max=ctx.n_elements - 1)
        contrib = int(B * ctx.n_tx * (hi - lo + 1).clamp(min=0).sum().item())
    sm_mhz = clk["sm_mhz"] or 1965.0
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # Rooflines of DAS, both measured on this B200
    # (profiles/r01_microbench.json):
    #  * FP32 pipe: the exact (bitwise) linear formulation is 9 FP32 lane-ops
    #    per contribution (t, floor, k0, a, 1-a, 2 rounded products, 2 adds;
    #    nearest: 4); FADD2/FFMA2 retire 2 warp-instr/clk/SM = 128 lane-ops.
    #  * shared-memory gathers: 2 x 4 B per linear contribution (1 nearest);
    #    LDS.32 retires 1 warp-instr/clk/SM = 128 B/clk/SM.
    # The binding roof is the slower of the two; HBM is ~100x away.
    #  * a thread that accumulates ft frames (bm_das_launch_shape) computes the
    #    frame-independent part once per (pixel, channel): linear 5 lane-ops
    #    (t, floor, k0, a, 1-a) + 4 per frame, nearest 3 (t, +0.5, floor) + 1.
    shape = eng.plan.launch_shape(n_s, B, args.interp) or {"ft": 1}
    ft = shape["ft"]
    #    Non-uniform apodisation adds w*(1-a), w*a per (pixel, channel)
    #    (linear) or one w*x per frame (nearest).
    if eng.plan.uniform:
        ops = (5.0 / ft + 4.0) if args.interp == "linear" else (3.0 / ft + 1.0)
    else:
        ops = (7.0 / ft + 4.0) if args.interp == "linear" else (3.0 / ft + 2.0)
    gb = 8 if args.interp == "linear" else 4
    t_fp32 = contrib * ops / (n_sm * 128 * sm_mhz * 1e6)
    t_lds = contrib * gb / (n_sm * 128 * sm_mhz * 1e6)
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
        "kernel": f"bm_das_beamform ({eng.plan.kernel_for(n_s, args.interp)})",
        "kernel_ms_per_launch": round(das_ms, 4),
        "algorithmic_bytes_per_launch": das_bytes,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
        "note": "DAS is bound on chip (SMEM gathers / FP32 pipe), not by HBM: see binding",
        "binding": {
            "resource": ("max of: SMEM gather roof (%d B per contribution, 128 B/clk/SM) and "
                         "FP32 pipe (%.4g lane-ops per contribution at %d frame(s) per thread, "
                         "128 lane-ops/clk/SM)" % (gb, ops, ft)),
            "bound_by": "smem_gather" if t_lds >= t_fp32 else "fp32",
            "launch_shape": shape,
            "contributions_per_launch": contrib,
            "achieved_gcontrib_s": round(contrib / (das_ms / 1000.0) / 1e9, 1),
            "achieved_tflops_fp32_lane_ops": round(contrib * ops / (das_ms / 1000.0) / 1e12, 2),
            "peak_tflops_fp32_lane_ops": round(n_sm * 128 * sm_mhz * 1e6 / 1e12, 2),
            "t_fp32_roof_ms": round(t_fp32 * 1000, 4),
            "t_smem_gather_roof_ms": round(t_lds * 1000, 4),
            "frac": round(max(t_fp32, t_lds) / (das_ms / 1000.0), 4),
            "sm_mhz": sm_mhz, "n_sm": n_sm},
    }

    cpu = None
    if not args.no_cpu and args.cpu_seconds > 0 and world == 1:  # rank 0 at N=1 only
        fps, cores, n, el = cpu_reference(ctx, grid, host[:4], args.cpu_seconds, args.interp)
        cpu = {"value": round(fps, 4), "unit": "frames/s", "cores": cores, "kind": "port",
               "sample": f"{n} {args.config} frames in {el:.1f}s: oracle/ C DAS (pthreads) + scipy.fft "
                         f"+ numpy dB, plan prebuilt"}

    line = {
        "metric": "B-mode frames/sec", "value": round(value, 2), "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic wire phantom + N(0,0.01)",
        "config": {"workload": WORKLOAD, "frames_per_gpu_per_step": B,
                   "global_frames_per_step": B * world, "parallelism": f"frames over {world} GPU",
                   "l2": f"inputs {B * frame_bytes / 1e6:.0f} MB per GPU > 126 MB L2, no flush"},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roofline,
        "cpu_baseline": cpu,
        "stages_ms_per_frame": {"das": round(das_ms / B, 5),
                                "envelope+dB": round((ms_step - das_ms) / B, 5)},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
