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

`roofline`: the DAS kernel against the roof that binds it -- shared-memory
gathers (8 B per linear contribution at 128 B/clk/SM) or, with one frame per
thread, the FP32 pipe -- at the SM clock sampled during the run; its HBM
traffic sits under roofline.hbm.  `stai`: the STAI pipelines (cfg1, cfg3)
measured in the same run the same way.

--impl reference: the reference itself -- echopipe's own
pipeline.benchmark (numba DAS on all host cores + scipy.fft + numpy) from
baseline/_ref, on its own simulator source -- on rank 0, with the C port of
the same algorithm (oracle/) timed beside it.
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
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="cfg5 column split: envelope kernel writes tiles into the destination's "
                         "NVLink peer buffer (peer), or one NCCL gather (nccl)")
    ap.add_argument("--window", default="rectangular", choices=["rectangular", "hann"],
                    help="receive apodisation window (ApodizationSpec)")
    ap.add_argument("--f-number", type=float, default=0.0,
                    help="dynamic-aperture f-number (0: all elements)")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                    help="frame dtype (f64: the reference's oracle precision, the f64 TMA kernel)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stai", action="store_true",
                    help="skip the STAI blocks (cfg1 / cfg3) of the default cfg2 run")
    ap.add_argument("--debug", action="append", default=[],
                    help="library tuning hook KEY=VALUE (_native.DEBUG_KEYS), e.g. das_ft=2")
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


def dropin_fps(ctx, grid, host, interp, n_frames=100, warmup=8, rounds=3):
    """Frames/s a reference user sees calling the drop-in operator chain one
    frame at a time: ``execute(build_graph(bmode_chain(...)), (RfFrame, ctx))``
    with numpy RF in and the numpy display read back (pageable H2D/D2H and a
    synchronisation per frame).  RfFrame construction (the reference's host
    finiteness scan) happens before the clock, as in echopipe's own
    benchmark().  The median of ``rounds`` timed runs of ``n_frames`` calls
    (host-side noise moves single runs by ~10 %)."""
    import paper_1811_01566_b200 as bm

    spec = bm.bmode_chain(interpolation=interp,
                          grid={"x_positions": grid.x_positions.tolist(),
                                "z_positions": grid.z_positions.tolist()})
    graph = bm.build_graph(spec)
    frames = [bm.RfFrame(host[i]) for i in range(min(len(host), 8))]
    for i in range(warmup):
        outs, _ = bm.execute(graph, (frames[i % len(frames)], ctx))
        outs["dynamic_adjustment"].numpy()
    rates = []
    for _ in range(rounds):
        t0 = time.perf_counter()
        for i in range(n_frames):
            outs, _ = bm.execute(graph, (frames[i % len(frames)], ctx))
            outs["dynamic_adjustment"].numpy()
        rates.append(n_frames / (time.perf_counter() - t0))
    return statistics.median(rates)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms by a
    background nvidia-smi loop (the recipe's clocks line) while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,temperature.gpu")

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
        temp = [float(r[7]) for r in rows if len(r) > 7 and num(r[7])]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "temp_c": max(temp) if temp else None, "samples": len(rows)}


def cpu_reference(ctx, grid, frames, seconds, interp, max_frames=None):
    """Reference algorithm on the host (oracle/ port): frames/s, threads."""
    from oracle import oracle as O

    plan = O.Plan(ctx, grid, "rectangular", 0.0, frames.dtype, frames.shape[2])
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
    """BASELINE config 5: one 2048 x 2048 STAI frame per step (strong
    scaling).  Columns: each rank beamforms its column slab, writes
    [envelope | peak] into its tile, ONE gather to rank 0, rank 0 maps the
    frame (parallel.LateralSplit).  Rows: each rank beamforms a depth band,
    ONE gather of the bands, rank 0 runs envelope + display (RowSplit)."""
    import torch

    import paper_1811_01566_b200 as bm
    from paper_1811_01566_b200 import parallel as P

    rows = args.split == "rows"
    split = (P.RowSplit if rows else P.LateralSplit)(grid, world, rank)
    plan = bm.DasPlan(ctx, split.sub_grid, bm.ApodizationSpec(), np.float32, ctx.n_elements)
    frame = torch.from_numpy(synth_frames(ctx, n_s, 1, 0)).to(dev)  # replicated RF
    f32 = torch.float32
    launches = [0]
    if rows and args.transport == "peer":
        # the DAS kernel stores this rank's rows into rank 0's frame buffer
        # over NVLink; device-side flags, no collective kernel
        bands = P.PeerBands(split, dev)

        def step():
            launches[0] += 3 + (2 + world if rank == 0 else 0)
            return bands.step(plan, frame, 30.0)
    elif rows:
        send = split.send_band(f32, dev)
        recv = split.recv_bands(f32, dev) if rank == 0 else None
        mine = send[None, : split.hi - split.lo]

        def step():
            plan.beamform_batch(frame, out=mine)
            full = split.gather(send, recv) if world > 1 else send
            launches[0] += 1
            if full is not None:
                launches[0] += 1
                return P.envelope_display(full, 30.0)
    elif args.transport == "peer":
        # the envelope kernel writes each tile into rank 0's symmetric buffer
        # over NVLink; device-side epoch flags, no collective kernel
        peer = P.PeerTiles(split, dev)
        slab = torch.empty((1,) + plan.shape, dtype=f32, device=dev)

        def step():
            plan.beamform_batch(frame, out=slab)
            launches[0] += 4 + (1 + world if rank == 0 else 0)
            return peer.step(slab[0], 30.0)
    else:
        tile = split.send_tile(f32, dev)
        recv = split.recv_tiles(f32, dev) if rank == 0 else None
        slab = torch.empty((1,) + plan.shape, dtype=f32, device=dev)

        def step():
            plan.beamform_batch(frame, out=slab)
            split.envelope_into_tile(slab[0], tile)
            got = split.gather(tile, recv) if world > 1 else tile[None]
            launches[0] += 2
            if got is not None:
                launches[0] += 1
                return split.display(got, 30.0)

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    if res is not None and int(res[1].item()) != 0:
        raise bm.AllZeroInput("dynamic adjustment needs a strictly positive element")
    if world > 1:
        torch.distributed.barrier()
    launches[0] = 0
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
                ("depth-row split, the DAS kernel stores its rows into rank 0's NVLink peer "
                 "frame buffer, device-side flags, envelope + display on rank 0"
                 if args.transport == "peer" else
                 "depth-row split, one NCCL gather of RF bands, envelope + display on rank 0")
                if rows
                else ("lateral column split, envelope kernel writes [envelope | peak] tiles into "
                      "rank 0's NVLink peer buffer, device-side flags, display on rank 0"
                      if args.transport == "peer" else
                      "lateral column split, one NCCL gather of [envelope | peak] tiles, display "
                      "on rank 0")),
                       ("rows_per_rank" if rows else "columns_per_rank"): split.hi - split.lo},
            "e2e": None, "gpu_launches": launches[0]}), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def das_roofline(eng, ctx, grid, n_s, B, das_ms, interp, clk, n_sm, peaks, workload):
    """Roofline of one DAS launch of B frames, measured
    peaks from profiles/r01_microbench.json at the SM clock sampled in the run:
      * shared-memory gathers: 8 B per linear contribution (4 nearest); LDS.32
        retires one warp instruction (128 B) per clk per SM;
      * FP32 pipe: 5/FT + 4 lane-ops per linear contribution (3/FT + 1
        nearest; +2 per (pixel, channel) and +... with weights) at 128
        lane-ops/clk/SM, FT = frames per thread of the launch shape.
    The binding one is the larger time; HBM (RF + image bytes) is ~50x away
    and reported under "hbm" with the ncu DRAM traffic."""
    import torch

    n_rx = ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements
    contrib = B * ctx.n_tx * n_rx * grid.n_z * grid.n_x
    span = eng.plan._bufs.get("span")
    if span is not None and eng.plan._geom.rx_contig:
        # F-number gate: terms outside a pixel's active span have weight 0 and
        # are exact zeros the kernel skips -- the algorithmic work is the
        # active contributions: per transmit, the span clipped to the run of
        # elements that transmit records (identity or centred maps)
        sp = span.view(-1, 2).to(torch.int64)
        rmap = ctx.channel_elements(n_rx)
        active = 0
        for e in range(ctx.n_tx):
            first = int(rmap[e][0])
            lo = sp[:, 0].clamp(min=first)
            hi = sp[:, 1].clamp(max=first + n_rx - 1)
            active += int((hi - lo + 1).clamp(min=0).sum().item())
        contrib = B * active
    sm_mhz = clk.get("sm_mhz") or 1965.0
    shape = eng.plan.launch_shape(n_s, B, interp) or {"ft": 1, "fp": 1}
    ft = shape["ft"]
    if eng.plan.uniform:
        ops = (5.0 / ft + 4.0) if interp == "linear" else (3.0 / ft + 1.0)
    else:
        ops = (7.0 / ft + 4.0) if interp == "linear" else (3.0 / ft + 2.0)
    f64 = np.dtype(eng.plan.dtype) == np.float64
    esz = 8 if f64 else 4
    gb = 2 * esz if interp == "linear" else esz
    # FP32: 128 lane-ops/clk/SM (FADD2/FFMA2); FP64: 64 (DADD/DMUL at 2
    # warp-instr/clk/SM, profiles/r02_microbench.json)
    lane_rate = 64 if f64 else 128
    clk_hz = sm_mhz * 1e6
    t_fp32 = contrib * ops / (n_sm * lane_rate * clk_hz)
    t_lds = contrib * gb / (n_sm * 128 * clk_hz)
    t = das_ms / 1000.0
    frame_bytes = ctx.n_tx * n_rx * n_s * esz
    img_bytes = grid.n_z * grid.n_x * esz
    hbm_bytes = B * (frame_bytes + img_bytes)
    hbm_peak = peaks.get("hbm_gbs", 6450.0)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "das_traffic.json")))
        if prof.get("workload") == workload and prof.get("interp") == interp:
            traffic = round(prof["dram_bytes_per_frame"] * B, 0)
    except Exception:
        pass
    if t_lds >= t_fp32:
        bound, achieved = "smem_gather", contrib * gb / t / 1e9
        peak, unit = n_sm * 128 * clk_hz / 1e9, "GB/s"
        per = f"{gb} B gathered per contribution"
    else:
        pipe = "fp64" if f64 else "fp32"
        bound, achieved = pipe, contrib * ops / t / 1e12
        peak, unit = n_sm * lane_rate * clk_hz / 1e12, "TFLOP/s"
        per = f"{ops:.4g} {pipe.upper()} lane-ops per contribution"
    return {
        "bound": bound, "achieved": round(achieved, 1 if unit == "GB/s" else 3),
        "peak": round(peak, 1 if unit == "GB/s" else 3), "unit": unit,
        "frac": round(max(t_fp32, t_lds) / t, 4), "traffic": traffic,
        "kernel": f"bm_das_beamform ({eng.plan.kernel_for(n_s, interp)})",
        "kernel_ms_per_launch": round(das_ms, 4),
        "algorithmic": f"{contrib} contributions per launch x {per}",
        "peak_source": ("measured per-SM rates (profiles/r02_microbench.json: LDS 128 B/clk/SM, "
                        "FADD2/FFMA2 128 and DADD/DMUL 64 lane-ops/clk/SM) x %d SMs x %.0f MHz "
                        "sampled during the run" % (n_sm, sm_mhz)),
        "launch_shape": shape,
        "t_smem_gather_roof_ms": round(t_lds * 1000, 4),
        "t_fp_pipe_roof_ms": round(t_fp32 * 1000, 4),
        "fp_lane_ops_per_contribution": round(ops, 4),
        "hbm": {"achieved": round(hbm_bytes / t / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(hbm_bytes / t / 1e9 / hbm_peak, 4),
                "algorithmic_bytes_per_launch": hbm_bytes,
                "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else
                "fallback"},
    }


def time_engine(eng, rf, out, steps, warmup, barrier, max_over_ranks):
    """Device-resident steps of eng.reconstruct: (ms total, mean DAS ms per
    launch, launches).  DAS is bracketed by events on its own stream."""
    import torch

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        eng.reconstruct(rf, out=out)
    torch.cuda.synchronize()
    eng.check()
    das_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
    launches0 = eng.launches
    barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record()
    for k in range(steps):
        eng.reconstruct(rf, out=out, stream=stream, das_events=das_ev[k])
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    eng.check()
    ms_total = max_over_ranks(t_start.elapsed_time(t_end))
    das_ms = statistics.mean(a.elapsed_time(b) for a, b in das_ev)
    return ms_total, das_ms, eng.launches - launches0


def stai_block(name, B, args, dev, clocks_fn, n_sm, peaks, barrier, max_over_ranks):
    """A STAI pipeline measured in the same run as the headline (BASELINE's
    metric names both the STAI and the PWI pipelines)."""
    import torch

    import paper_1811_01566_b200 as bm
    from paper_1811_01566_b200 import environment as ME

    ctx, grid, n_s = ME.config_geometry(name)
    distinct = min(B, 4)
    host = synth_frames(ctx, n_s, distinct, 0)
    rf = torch.from_numpy(host).to(dev)
    if distinct < B:  # inputs still exceed L2 (B x 33.5 / 268 MB)
        rf = rf.repeat((B + distinct - 1) // distinct, 1, 1, 1)[:B].contiguous()
    eng = bm.BmodeEngine(ctx, grid, interp=args.interp)
    out = torch.empty((B, grid.n_z, grid.n_x), dtype=torch.float32, device=dev)
    steps = max(5, args.steps // 2) if name != "cfg1" else args.steps
    ms, das_ms, launches = time_engine(eng, rf, out, steps, args.warmup, barrier, max_over_ranks)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    clk = clocks_fn()
    rl = das_roofline(eng, ctx, grid, n_s, B, das_ms, args.interp, clk, n_sm, peaks,
                      WORKLOADS[name])
    del rf, out
    torch.cuda.empty_cache()
    return {"workload": WORKLOADS[name].replace("linear", args.interp), "value": round(
        world * B * steps / (ms / 1000.0), 2), "unit": "frames/s",
        "frames_per_gpu_per_step": B, "steps": steps, "ms_per_step": round(ms / steps, 4),
        "das_ms_per_frame": round(das_ms / B, 5),
        "envelope_display_ms_per_frame": round((ms / steps - das_ms) / B, 5),
        "binding": {k: rl[k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                       "launch_shape", "kernel_ms_per_launch")},
        "gpu_launches": launches}


def reference_arm(args, ctx, grid, n_s, world):
    """--impl reference: echopipe itself (baseline/_ref, its own
    pipeline.benchmark on its own SimulatorSource, numba threads = all host
    cores), the C port of the same algorithm timed beside it."""
    frames = synth_frames(ctx, n_s, 2, 0).astype(np.float32 if args.dtype == "f32" else np.float64)
    port = []
    for i in range(args.warmup + args.steps):
        fps, cores, n, el = cpu_reference(ctx, grid, frames, 0.0, args.interp, max_frames=1)
        if i >= args.warmup:
            port.append(el / n)
    port_ms = statistics.median(port) * 1000.0
    ref = None
    try:
        ref = echopipe_benchmark(args, grid, n_s, args.steps, args.warmup)
    except Exception as exc:  # pragma: no cover - reported, not hidden
        ref = {"error": f"{type(exc).__name__}: {exc}"}
    sample = f"1 {args.config} frame per step"
    if ref is not None and "ms" in ref:
        ms, kind, cores = ref["ms"], "reference", ref["threads"]
        what = (f"{sample}: echopipe {ref['version']} pipeline.benchmark (numba _das_kernel on "
                f"{ref['threads']} threads, effective parallelism {ref['effective']} pixel blocks "
                f"of 16384; scipy.fft; numpy), median of {args.steps} frames after "
                f"{args.warmup} warm-up, plan cached")
    else:
        ms, kind, cores = port_ms, "port", cores
        what = f"{sample}: oracle/ C DAS (pthreads, all cores) + scipy.fft analytic + numpy dB"
    val = 1000.0 / ms
    line = {
        "impl": "reference", "metric": "B-mode frames/sec", "value": round(val, 4),
        "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic wire phantom + N(0,0.01)",
        "config": {"workload": WORKLOAD + (", f64" if args.dtype == "f64" else ""),
                   "frames_per_step": 1},
        "cpu_baseline": {"value": round(val, 4), "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": what},
        "e2e": {"value": round(val, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "port": {"value": round(1000.0 / port_ms, 4), "unit": "frames/s", "cores": cores,
                 "kind": "port", "ms_per_frame": round(port_ms, 3),
                 "sample": "oracle/ C DAS (pthreads, all cores) + scipy.fft + numpy dB, same "
                           "frames, plan prebuilt"},
    }
    if ref is not None and "stages_ms" in ref:
        line["reference_stages_ms"] = ref["stages_ms"]
    if ref is not None and "error" in ref:
        line["reference_error"] = ref["error"]
    print(json.dumps(line), flush=True)


def echopipe_benchmark(args, grid_m, n_s, steps, warmup):
    """echopipe's own benchmark (pipeline.py:398-437) of its bmode_chain on
    its own seeded simulator (environment.py:181-221), imported from the
    vendored install baseline/_ref."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "echopipe")):
        raise FileNotFoundError("baseline/_ref/echopipe not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_echopipe")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import numba
    from echopipe import __version__ as ver  # noqa: F401
    from echopipe import environment as EE
    from echopipe import pipeline as EPL
    from echopipe import presets as EPR
    from echopipe import types as ET

    from paper_1811_01566_b200 import environment as ME

    ctx_m, _, _ = ME.config_geometry(args.config)
    if ctx_m.is_pw:
        scheme = ET.PwScheme(ctx_m.tx_scheme.angles_rad)
    else:
        scheme = ET.StaScheme(ctx_m.tx_scheme.tx_elements)
    ctx = ET.AcquisitionContext(ctx_m.speed_of_sound, ctx_m.sampling_frequency,
                                ctx_m.n_elements, ctx_m.pitch, scheme,
                                rx_channel_map=ctx_m.rx_channel_map)
    threads = os.cpu_count() or 1
    numba.set_num_threads(min(threads, numba.config.NUMBA_NUM_THREADS))
    spec = EPL.bmode_chain(interpolation=args.interp,
                           grid={"x_positions": grid_m.x_positions.tolist(),
                                 "z_positions": grid_m.z_positions.tolist()})
    graph = EPL.build_graph(spec)
    env = EE.open_simulator(EPR.wire_phantom(), ctx, n_s,
                            dtype=np.float32 if args.dtype == "f32" else np.float64, seed=0,
                            noise_std=0.01)
    res = EPL.benchmark(graph, env, n_frames=steps, warmup=max(1, warmup))
    n_px = grid_m.n_z * grid_m.n_x
    return {"ms": res.timing.total_ms, "threads": numba.get_num_threads(),
            "effective": min(numba.get_num_threads(), -(-n_px // 16384)),
            "version": getattr(sys.modules["echopipe"], "__version__", "?"),
            "stages_ms": {k: round(v, 3) for k, v in res.timing.stages}}


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
        if rank == 0:
            reference_arm(args, ctx, grid, n_s, world)
        return

    import torch

    from paper_1811_01566_b200 import _native as N

    for kv in args.debug:
        k, v = kv.split("=")
        N.load().bm_debug_set(N.DEBUG_KEYS[k], int(v))
    if world > 1 or (args.config == "cfg5" and args.transport == "peer"):
        import torch.distributed as dist

        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    if args.config == "cfg5":
        return run_cfg5(args, ctx, grid, n_s, rank, world, local, dev)

    B = args.frames
    fdt = np.float32 if args.dtype == "f32" else np.float64
    host = synth_frames(ctx, n_s, B, seed0=rank * B).astype(fdt)
    apod = bm.ApodizationSpec(args.window, args.f_number)
    eng = bm.engine.BmodeEngine(ctx, grid, apod=apod, interp=args.interp, dtype=fdt)
    if not eng.plan.uniform:
        WORKLOAD = WORKLOAD + f", {args.window} F={args.f_number:g}"
    if args.dtype == "f64":
        WORKLOAD = WORKLOAD + ", f64"
        frame_bytes, img_bytes = 2 * frame_bytes, 2 * img_bytes
    rf = torch.from_numpy(host).to(dev)
    out = torch.empty((B, grid.n_z, grid.n_x), dtype=eng.tdtype, device=dev)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass

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
    clocks.mark()  # keep only samples taken from here on
    ms_total, das_ms, launches = time_engine(eng, rf, out, args.steps, 0, barrier, max_over_ranks)
    clk = clocks.stop()
    ms_step = ms_total / args.steps
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
        # every step: H2D of its B RF frames from pinned host memory, the
        # chain, D2H of its B displays; steps are pipelined back to back and
        # the clock stops when the last display is on the host
        eng.reconstruct_host_stream([(rf_h, disp_h)] * e2e_steps)
        el = max_over_ranks(time.perf_counter() - t0)
        eng.check()
        e2e = {"value": round(world * B * e2e_steps / el, 2), "unit": "frames/s",
               "h2d_bytes_per_step": B * frame_bytes, "d2h_bytes_per_step": B * img_bytes,
               "ms_per_step": round(el / e2e_steps * 1000.0, 3)}
        del rf_h, disp_h

    # one frame per call through the reference-facing chain (measured before
    # the STAI blocks, whose large allocations left it ~6 % slower)
    if e2e is not None and world == 1 and args.dtype == "f32":
        e2e["dropin_per_frame_fps"] = round(dropin_fps(ctx, grid, host, args.interp), 1)
        e2e["dropin_note"] = ("one frame per call through the reference-facing operator chain "
                              "(numpy in, numpy display out, pageable copies), median of 3 runs "
                              "of 100 calls; value above is the batched engine from pinned "
                              "memory")

    roofline = das_roofline(eng, ctx, grid, n_s, B, das_ms, args.interp, clk, n_sm, peaks,
                            WORKLOAD)

    stai = None
    if not args.no_stai and args.config == "cfg2" and args.dtype == "f32":
        del rf
        torch.cuda.empty_cache()
        clocks2 = ClockSampler(local)
        clocks2.start()
        clocks2.mark()
        stai = {}
        for name, nb in (("cfg1", 32), ("cfg3", 8)):
            stai[name] = stai_block(name, nb, args, dev, lambda: dict(clk), n_sm, peaks, barrier,
                                    max_over_ranks)
        clk2 = clocks2.stop()
        stai["clocks"] = clk2

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu and args.cpu_seconds > 0 and world == 1 and args.dtype == "f32":
        fps, cores, n, el = cpu_reference(ctx, grid, host[:4], args.cpu_seconds, args.interp)
        cpu = {"value": round(fps, 4), "unit": "frames/s", "cores": cores, "kind": "port",
               "sample": f"{n} {args.config} frames in {el:.1f}s: oracle/ C DAS (pthreads) + "
                         f"scipy.fft + numpy dB, plan prebuilt"}

    line = {
        "metric": "B-mode frames/sec", "value": round(value, 2), "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic wire phantom + N(0,0.01)",
        "config": {"workload": WORKLOAD, "frames_per_gpu_per_step": B,
                   "global_frames_per_step": B * world, "parallelism": f"frames over {world} GPU",
                   "l2": f"inputs {B * frame_bytes / 1e6:.0f} MB per GPU > 126 MB L2, no flush"},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roofline,
        "cpu_baseline": cpu,
        "stages_ms_per_frame": {"das": round(das_ms / B, 5),
                                "envelope+dB (fused)": round((ms_step - das_ms) / B, 5)},
        "stai": stai,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
