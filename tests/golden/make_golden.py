"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
(echopipe, /root/reference/pkg/src) in this container.

    NUMBA_CACHE_DIR=/tmp/nb PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py

/root/reference does not exist on the GPU box; the fixtures written here are
what travels.  Inputs are NOT stored: every instance is rebuilt from a seed by
tests/cases.py, whose draw order matches the reference's own tests.

Outputs:
  das_small.npz   criterion-4 instances (test_acceptance.py:124-177): sha256 of
                  das_beamform output bytes for {f64, f32} x {nearest, linear},
                  plus the full arrays of the first 12 cases.
  chain.npz       Fig-2 chain (beamform -> analytic -> envelope -> dB, f32) on
                  six mid-size instances: rf, envelope, display arrays and the
                  complex analytic signal of two of them.
  sigproc.npz     analytic_signal / dynamic_adjustment on seeded arrays.
  fir.npz         fir_filter (lfilter) on seeded f32/f64 traces, taps 1..64,
                  along the sample axis and along axis 0 (inputs stored).
  qus.npz         sliding_moments / estimate_hk_map on seeded Rayleigh
                  envelopes with a seeded relu/softplus/identity model.
  ref_small.wfrf, ref_pw.wfrf
                  WFRF files written by the reference (STA f32 with t0; PW f64
                  with an rx map); pgm.npz: write_pgm bytes of seeded displays.
  sim.npz         simulate_rf (noise-free): f64 STA (t0, rx map) and PW frames,
                  sha256 of the cfg2 wire-phantom f32 frame.
  engine.npz      the benchmarked batched path: per frame of the bench's own
                  cine generator (cfg2 wire phantom + N(0, 0.01), seed = frame
                  index; cfg1 and cfg3 likewise), the sha256 of the f32 input
                  RF, the sha256 of the reference's das_beamform output, and
                  the full f32 display of the reference chain for some frames.
  sigproc_long.npz  analytic_signal at n = 2048 / 4096 (f32: 37 / 9 lanes,
                  f64: 5 / 3 lanes; inputs from cases.long_lanes).
  configs.json    sha256 of das_beamform f32 output at full BASELINE sizes
                  (cfg1/cfg2 linear+nearest, cfg3 linear, cfg1 f64) on seeded
                  N(0,1) RF, and of simulate_rf for the cfg2 wire phantom.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root

import echopipe.types as ET  # noqa: E402
from echopipe import beamform as EB  # noqa: E402
from echopipe import environment as EE  # noqa: E402
from echopipe import presets as EP  # noqa: E402
from echopipe import sigproc as ES  # noqa: E402

import cases  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def das_small():
    hashes = {}
    arrays = {}
    for i, (ctx, data, grid, apod) in enumerate(cases.criterion4_cases(ET)):
        for dt in ("f64", "f32"):
            frame = ET.RfFrame(data if dt == "f64" else data.astype(np.float32))
            for interp in ("nearest", "linear"):
                img = EB.das_beamform(frame, ctx, grid, apod, interp=interp).data
                hashes[f"{i}_{dt}_{interp}"] = sha(img)
                if i < 12:
                    arrays[f"{i}_{dt}_{interp}"] = img
        if i < 12:
            oracle = EB.das_beamform_oracle(ET.RfFrame(data), ctx, grid, apod, interp="linear")
            arrays[f"{i}_f64_linear_oracle"] = oracle.data
    keys = sorted(hashes)
    np.savez_compressed(os.path.join(HERE, "das_small.npz"),
                        hash_keys=np.array(keys), hash_vals=np.array([hashes[k] for k in keys]),
                        **arrays)


def chain():
    arrays = {}
    for name, ctx, data, grid, apod, interp in cases.chain_cases(ET):
        frame = ET.RfFrame(data)
        rf = EB.das_beamform(frame, ctx, grid, apod, interp=interp).data
        z = ES.analytic_signal(rf, axis=0)
        env = ES.envelope(z)
        disp = ES.dynamic_adjustment(env, 30.0).astype(rf.dtype, copy=False)
        arrays[f"{name}_rf"] = rf
        arrays[f"{name}_env"] = env
        arrays[f"{name}_disp"] = disp
        if name in ("sta_rect_linear", "pw_t0_oddN_linear"):
            arrays[f"{name}_z"] = z
        # f64 chain on the same instance for the f64 GPU path
        rf64 = EB.das_beamform(ET.RfFrame(data.astype(np.float64)), ctx, grid, apod,
                               interp=interp).data
        env64 = ES.envelope(ES.analytic_signal(rf64, axis=0))
        arrays[f"{name}_rf64"] = rf64
        arrays[f"{name}_disp64"] = ES.dynamic_adjustment(env64, 30.0)
    np.savez_compressed(os.path.join(HERE, "chain.npz"), **arrays)


def fir():
    """fir.npz: the reference's fir_filter (scipy lfilter) on seeded traces,
    f32 and f64 frames, taps of 1..64, along the sample axis and axis 0."""
    rng = np.random.default_rng(91)
    out = {}
    for nt in (1, 2, 7, 33, 64):
        h = rng.normal(size=nt)
        x32 = rng.normal(size=(3, 5, 300)).astype(np.float32)
        x64 = rng.normal(size=(2, 4, 257))
        out[f"h_{nt}"] = h
        out[f"x32_{nt}"] = x32
        out[f"y32_{nt}"] = ES.fir_filter(x32, ES.FirSpec(h))
        out[f"x64_{nt}"] = x64
        out[f"y64_{nt}"] = ES.fir_filter(x64, ES.FirSpec(h))
        xa = rng.normal(size=(90, 6))
        out[f"xa_{nt}"] = xa
        out[f"ya_{nt}"] = ES.fir_filter(xa, ES.FirSpec(h), axis=0)
    np.savez_compressed(os.path.join(HERE, "fir.npz"), **out)


def qus():
    """qus.npz: the reference's sliding_moments / estimate_hk_map on seeded
    Rayleigh envelopes with a seeded 3-layer model (inputs stored)."""
    from echopipe import qus as EQ

    rng = np.random.default_rng(303)
    out = {}
    cases = [((64, 48), (8, 4), (4, 2)), ((97, 31), (5, 5), (1, 1)),
             ((512, 40), (64, 4), (32, 2)), ((33, 33), (33, 33), (1, 1))]
    layers = [(rng.normal(size=(8, 3)), rng.normal(size=8), "relu"),
              (rng.normal(size=(6, 8)), rng.normal(size=6), "softplus"),
              (rng.normal(size=(2, 6)), rng.normal(size=2), "identity")]
    model = EQ.DenseModel(tuple(EQ.DenseLayer(w, b, a) for w, b, a in layers))
    for i, (shape, win, st) in enumerate(cases):
        img = rng.rayleigh(1.0, size=shape).astype(np.float32 if i % 2 else np.float64)
        m = EQ.sliding_moments(img, win, st)
        hk = EQ.estimate_hk_map(img, win, st, model)
        out[f"img_{i}"] = img
        out[f"win_{i}"], out[f"stride_{i}"] = np.array(win), np.array(st)
        out[f"m1_{i}"], out[f"m2_{i}"], out[f"m3_{i}"] = m.m1, m.m2, m.m3
        out[f"u_{i}"], out[f"k_{i}"] = hk.u, hk.k
    for j, (w, b, a) in enumerate(layers):
        out[f"W_{j}"], out[f"b_{j}"] = w, b
    out["acts"] = np.array([a for _, _, a in layers])
    np.savez_compressed(os.path.join(HERE, "qus.npz"), **out)


def formats():
    """ref_small.wfrf / ref_pw.wfrf written by the reference's write_wfrf, and
    pgm.npz: write_pgm bytes of seeded display images (f32 and f64)."""
    from echopipe import formats as EF
    from echopipe.types import (AcquisitionContext, BmodeImage, ImageGrid, PwScheme, RfFrame,
                                StaScheme)

    rng = np.random.default_rng(404)
    ctx = AcquisitionContext(1540.0, 20e6, 4, 3e-4, StaScheme((0, 1, 2, 3)),
                             time_zero_offset=np.linspace(0, 1e-6, 4))
    frames = [RfFrame(rng.normal(size=(4, 4, 32)).astype(np.float32)) for _ in range(3)]
    EF.write_wfrf(os.path.join(HERE, "ref_small.wfrf"), frames, ctx)
    ctx = AcquisitionContext(1540.0, 40e6, 6, 2e-4, PwScheme((-0.1, 0.0, 0.1)),
                             rx_channel_map=np.array([[0, 2, 4], [1, 3, 5], [5, 4, 3]]))
    frames = [RfFrame(rng.normal(size=(3, 3, 16))) for _ in range(2)]
    EF.write_wfrf(os.path.join(HERE, "ref_pw.wfrf"), frames, ctx)
    out = {}
    for name, dt in (("f32", np.float32), ("f64", np.float64)):
        d = rng.random((37, 29)).astype(dt)
        d[0, :6] = np.array([0.0, 1.0, 0.5, 0.5 / 255, 1.5 / 255, 254.5 / 255], dtype=dt)
        img = BmodeImage(d, stage="display", grid=ImageGrid(np.arange(29) * 1e-4,
                                                             np.arange(37) * 1e-4))
        path = os.path.join("/tmp", f"golden_{name}.pgm")
        EF.write_pgm(img, path)
        out[f"disp_{name}"] = d
        out[f"pgm_{name}"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "pgm.npz"), **out)


def sim():
    """sim.npz: the reference's simulate_rf (noise-free) -- f64 frames of a
    small STA case (t0 offsets, rx map) and a small PW case, and the sha256 of
    the cfg2 wire-phantom frame in f32 (the benchmark cine's clean signal)."""
    from echopipe.types import AcquisitionContext as AC, PwScheme as PS, StaScheme as SS

    from paper_1811_01566_b200 import environment as ME

    ph = EE.Phantom(((0.4e-3, 4.9e-3, 1.0), (-1.1e-3, 7.3e-3, 0.6), (2.0e-3, 3.1e-3, -0.8)),
                    center_frequency=5e6, n_cycles=2)
    out = {}
    ctx = AC(1540.0, 40e6, 16, 2e-4, SS((0, 5, 11, 15)),
             rx_channel_map=np.array([[i, (i + 3) % 16, 15 - i] for i in (0, 5, 11, 15)]),
             time_zero_offset=np.array([0.0, 1e-7, -2e-7, 3.3e-7]))
    out["sta_f64"] = EE.simulate_rf(ph, ctx, 600, dtype=np.float64).data
    ctx = AC(1480.0, 31.25e6, 24, 3e-4, PS((-0.2, 0.05, 0.17)))
    out["pw_f64"] = EE.simulate_rf(ph, ctx, 500, dtype=np.float64).data
    ctx_m, grid_m, n_s = ME.config_geometry("cfg2")
    ctx = AC(ctx_m.speed_of_sound, ctx_m.sampling_frequency, ctx_m.n_elements, ctx_m.pitch,
             PS(ctx_m.tx_scheme.angles_rad))
    clean = EE.simulate_rf(EP.wire_phantom(), ctx, n_s, dtype=np.float32).data
    out["cfg2_wire_f32_sha256"] = np.array(hashlib.sha256(clean.tobytes()).hexdigest())
    np.savez_compressed(os.path.join(HERE, "sim.npz"), **out)


def sigproc():
    rng = np.random.default_rng(77)
    out = {}
    for n in (2, 3, 8, 9, 33, 64, 100, 256, 1000, 1024):
        x32 = rng.normal(size=(n, 5)).astype(np.float32)
        x64 = rng.normal(size=(n, 3))
        out[f"x32_{n}"] = x32
        out[f"z32_{n}"] = ES.analytic_signal(x32, axis=0)
        out[f"x64_{n}"] = x64
        out[f"z64_{n}"] = ES.analytic_signal(x64, axis=0)
    # wide images (37 lanes: a partial 8-lane CTA) at the register-FFT sizes
    rng_w = np.random.default_rng(78)
    for n in (256, 512, 1024):
        xw = rng_w.normal(size=(n, 37)).astype(np.float32)
        out[f"x32w_{n}"] = xw
        out[f"z32w_{n}"] = ES.analytic_signal(xw, axis=0)
    e = np.abs(rng.normal(size=(64, 48))).astype(np.float32)
    e[3, 4] = 0.0
    out["dyn_in32"] = e
    out["dyn_out32_30"] = ES.dynamic_adjustment(e, 30.0)
    out["dyn_out32_45"] = ES.dynamic_adjustment(e, 45.0)
    out["dyn_in64"] = e.astype(np.float64) * 3.0
    out["dyn_out64_30"] = ES.dynamic_adjustment(out["dyn_in64"], 30.0)
    np.savez_compressed(os.path.join(HERE, "sigproc.npz"), **out)


def configs():
    from paper_1811_01566_b200 import environment as ME

    res = {}
    specs = [("cfg1", "f32", "linear", 0), ("cfg1", "f32", "nearest", 0),
             ("cfg1", "f64", "linear", 0), ("cfg2", "f32", "linear", 1),
             ("cfg2", "f32", "nearest", 1), ("cfg3", "f32", "linear", 2)]
    for name, dt, interp, seed in specs:
        ctx_m, grid_m, n_s = ME.config_geometry(name)
        ctx = ET.AcquisitionContext(ctx_m.speed_of_sound, ctx_m.sampling_frequency,
                                    ctx_m.n_elements, ctx_m.pitch,
                                    ET.PwScheme(ctx_m.tx_scheme.angles_rad) if ctx_m.is_pw
                                    else ET.StaScheme(ctx_m.tx_scheme.tx_elements))
        grid = ET.ImageGrid(grid_m.x_positions, grid_m.z_positions)
        data = cases.config_rf((ctx.n_tx, ctx.n_elements, n_s), seed)
        if dt == "f64":
            data = data.astype(np.float64)
        t = time.time()
        img = EB.das_beamform(ET.RfFrame(data), ctx, grid, interp=interp).data
        res[f"{name}_{dt}_{interp}_seed{seed}"] = sha(img)
        print(name, dt, interp, f"{time.time() - t:.1f}s", flush=True)
    # simulator pin: cfg2 wire phantom, f32, noise 0.01 seed 0
    ctx_m, grid_m, n_s = ME.config_geometry("cfg2")
    ctx = ET.AcquisitionContext(ctx_m.speed_of_sound, ctx_m.sampling_frequency,
                                ctx_m.n_elements, ctx_m.pitch,
                                ET.PwScheme(ctx_m.tx_scheme.angles_rad))
    env = EE.open_simulator(EP.wire_phantom(), ctx, n_s, dtype=np.float32, seed=0,
                            noise_std=0.01)
    frame, _ = env.next_observation()
    res["sim_cfg2_wire_f32_seed0_noise0.01"] = sha(frame.data)
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


def _ref_ctx(ctx_m):
    return ET.AcquisitionContext(ctx_m.speed_of_sound, ctx_m.sampling_frequency,
                                 ctx_m.n_elements, ctx_m.pitch,
                                 ET.PwScheme(ctx_m.tx_scheme.angles_rad) if ctx_m.is_pw
                                 else ET.StaScheme(ctx_m.tx_scheme.tx_elements))


# frames of each config's bench cine that get golden outputs: (rf sha seeds,
# display seeds).  cfg2 batches are 32 frames (FP = 2 x FT = 4 passes), so the
# seeds hit several pass / thread slots; cfg3 batches are 8 frames.
ENGINE_FRAMES = {"cfg2": ((0, 1, 2, 3, 13, 31), (0, 13, 31)),
                 "cfg1": ((0, 5, 31), (0,)),
                 "cfg3": ((0, 7), (0,))}


def engine():
    """engine.npz: reference outputs for frames of bench.synth_frames' cine
    (the clean wire-phantom frame from the reference's own simulate_rf in f64,
    plus N(0, 0.01) drawn from default_rng(seed), cast to f32)."""
    from paper_1811_01566_b200 import environment as ME

    out = {}
    for name, (rf_seeds, disp_seeds) in ENGINE_FRAMES.items():
        ctx_m, grid_m, n_s = ME.config_geometry(name)
        ctx = _ref_ctx(ctx_m)
        grid = ET.ImageGrid(grid_m.x_positions, grid_m.z_positions)
        clean = EE.simulate_rf(EP.wire_phantom(), ctx, n_s, dtype=np.float64).data
        plan = None
        for seed in rf_seeds:
            rng = np.random.default_rng(seed)
            data = (clean + rng.normal(0.0, 0.01, clean.shape)).astype(np.float32)
            frame = ET.RfFrame(data)
            if plan is None:
                plan = EB.DasPlan(ctx, grid, ET.ApodizationSpec(), np.float32, ctx.n_elements)
            rf = EB.das_beamform(frame, ctx, grid, plan=plan).data
            out[f"{name}_in_sha_{seed}"] = np.array(sha(data))
            out[f"{name}_rf_sha_{seed}"] = np.array(sha(rf))
            if seed in disp_seeds:
                env = ES.envelope(ES.analytic_signal(rf, axis=0))
                out[f"{name}_disp_{seed}"] = ES.dynamic_adjustment(env, 30.0).astype(np.float32)
            print(name, seed, flush=True)
    np.savez_compressed(os.path.join(HERE, "engine.npz"), **out)


def sigproc_long():
    """sigproc_long.npz: scipy.fft analytic signals of long axes (2048: cfg5
    and sta-paper n_z; 4096) -- outputs only, the inputs are rebuilt from
    cases.long_lanes(n, lanes, dtype) (general N is checked against the
    oracle, scipy itself, at test time)."""
    out = {}
    for n, l32, l64 in cases.LONG_AXES:
        out[f"z32_{n}"] = ES.analytic_signal(cases.long_lanes(n, l32, np.float32), axis=0)
        out[f"z64_{n}"] = ES.analytic_signal(cases.long_lanes(n, l64, np.float64), axis=0)
    np.savez_compressed(os.path.join(HERE, "sigproc_long.npz"), **out)


ALL = ("das_small", "chain", "sigproc", "fir", "qus", "formats", "sim", "configs", "engine",
       "sigproc_long")

if __name__ == "__main__":
    names = sys.argv[1:] or ALL
    for fn in (globals()[n] for n in names):
        t = time.time()
        fn()
        print(fn.__name__, f"{time.time() - t:.1f}s", flush=True)
