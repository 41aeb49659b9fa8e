"""``python -m paper_1811_01566_b200.cli`` -- the reference's benchmark and
reconstruct commands (cli.py:85-167) on the B200 path.

* ``benchmark``: per-stage GPU times (CUDA events) of a pipeline over the
  paper presets (``--synthetic sta-paper|pwi-paper``, presets.py:53-100)
  and/or a WFRF dataset (``--in``), grouped into the paper's Table 1 rows by
  :mod:`.report` -- the same text / JSON-records output and CSV file as the
  reference, so its tooling reads the GPU rows unchanged.  RF is staged to
  the device before each frame's clock starts (the table's "pure compute per
  stage"); ``--host-input`` keeps the host->device copy inside the beamform
  row instead.
* ``reconstruct``: a WFRF file to one 8-bit PGM per frame through the batched
  engine (BmodeEngine.reconstruct_file: pinned staging, copy/compute overlap;
  bm_quantize_u8 + write_pgm).
* ``simulate``: seeded wire-phantom / JSON-phantom RF frames to a WFRF file.

Diagnostics go to stderr, tables/records to stdout; exit 0 success, 1
processing failure, 2 usage error (cli.py:217-231).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

PRESET_NAMES = ("sta-paper", "pwi-paper")
_DTYPES = {"f32": np.float32, "f64": np.float64}


def _json(path, what):
    from .errors import EchopipeError

    try:
        with open(path, encoding="utf-8") as fh:
            return json.load(fh)
    except FileNotFoundError:
        raise EchopipeError(f"{what} file not found: {path}")
    except json.JSONDecodeError as exc:
        raise EchopipeError(f"{what} file {path} is not valid JSON: {exc}")


def preset_environment(name: str, dtype=np.float32, seed: int = 0, max_frames=None):
    """Simulator stream of a paper preset (presets.py:87-94)."""
    from . import environment as E

    if name not in E.PRESETS:
        raise KeyError(f"unknown preset {name!r}; choose from {PRESET_NAMES}")
    return E.open_simulator(E.wire_phantom(), E.PRESETS[name](), E.N_SAMPLES, dtype=dtype,
                            seed=seed, max_frames=max_frames)


def preset_pipeline(name: str) -> dict:
    """The preset's chain: 30 dB, nearest interpolation (presets.py:97-100)."""
    from .pipeline import bmode_chain

    if name not in PRESET_NAMES:
        raise KeyError(f"unknown preset {name!r}; choose from {PRESET_NAMES}")
    return bmode_chain(range_db=30.0, interpolation="nearest")


def mode_label(ctx) -> str:
    return "PWI" if ctx.is_pw else "STAI"


def _cmd_benchmark(args) -> int:
    from . import report as R
    from .environment import open_dataset
    from .errors import EchopipeError
    from .pipeline import benchmark, bmode_chain, build_graph

    runs = []
    for preset in args.synthetic:
        env = preset_environment(preset, _DTYPES[args.dtype], args.seed)
        spec = _json(args.pipeline, "pipeline spec") if args.pipeline else preset_pipeline(preset)
        runs.append((mode_label(env._source.ctx), build_graph(spec), env))
    if args.input:
        env = open_dataset(args.input)
        spec = _json(args.pipeline, "pipeline spec") if args.pipeline else bmode_chain()
        runs.append((mode_label(env._source._reader.context), build_graph(spec), env))
    if not runs:
        raise EchopipeError("benchmark needs --synthetic <preset> and/or --in <wfrf>")
    results = []
    for label, graph, env in runs:
        res = benchmark(graph, env, n_frames=args.frames, warmup=args.warmup,
                        device_resident=not args.host_input)
        results.append((label, graph, res))
        print(f"{label}: {res.n_frames} frame(s) measured, {res.timing.total_ms:.3f} ms/frame "
              f"median (B200, CUDA-event stage times)", file=sys.stderr)
    rep = R.make_report(results)
    print(R.format_table(rep) if args.format == "table" else R.format_records(rep))
    if args.report_dir:
        out = Path(args.report_dir)
        out.mkdir(parents=True, exist_ok=True)
        R.write_csv(rep, out / "benchmark.csv")
        wrote = ["benchmark.csv"]
        try:
            R.save_timing_figure(rep, out / "benchmark.png")
            wrote.append("benchmark.png")
        except ImportError:
            print("matplotlib absent: no benchmark.png", file=sys.stderr)
        print(f"wrote {' and '.join(wrote)} to {out}", file=sys.stderr)
    return 0


def _cmd_reconstruct(args) -> int:
    from .engine import BmodeEngine
    from .errors import EchopipeError
    from .formats import WfrfReader, write_pgm
    from .types import BmodeImage, default_grid

    with WfrfReader(args.input) as rd:
        ctx, n = rd.context, rd.frame_count
        shape, dtype = tuple(rd.frame_shape), np.dtype(rd.dtype.newbyteorder("="))
    if n == 0:
        raise EchopipeError(f"no frames in {args.input}")
    grid = default_grid(ctx, shape[2], "pw" if ctx.is_pw else "sta")
    eng = BmodeEngine(ctx, grid, interp=args.interpolation, range_db=args.range_db, dtype=dtype,
                      n_rx=shape[1])
    disp, _ = eng.reconstruct_file(args.input)
    eng.check()
    out = Path(args.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    for i in range(n):
        write_pgm(BmodeImage(disp[i].numpy(), stage="display", grid=grid),
                  out / f"frame_{i:04d}.pgm")
    print(f"wrote {n} image(s) to {out}", file=sys.stderr)
    return 0


def _cmd_simulate(args) -> int:
    from .environment import Environment, Phantom, SimulatorSource, wire_phantom
    from .formats import context_from_dict, write_wfrf

    if args.phantom:
        raw = _json(args.phantom, "phantom spec")
        pulse = raw.get("pulse", {})
        phantom = Phantom(tuple(tuple(s) for s in raw["scatterers"]),
                          center_frequency=float(pulse.get("center_frequency", 5e6)),
                          n_cycles=float(pulse.get("n_cycles", 2.0)))
    else:
        phantom = wire_phantom()
    ctx = context_from_dict(_json(args.ctx, "context spec"))
    src = SimulatorSource(phantom, ctx, args.n_samples, dtype=_DTYPES[args.dtype], seed=args.seed,
                          noise_std=args.noise_std, max_frames=args.frames)
    frames = [f for f, _ in Environment(src)]
    write_wfrf(args.out, frames, ctx)
    print(f"wrote {len(frames)} frame(s) to {args.out}", file=sys.stderr)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1811_01566_b200.cli",
                                 description="B-mode reconstruction on the B200")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("benchmark", help="per-stage GPU timing (Table 1 rows)")
    b.add_argument("--synthetic", action="append", choices=PRESET_NAMES, default=[])
    b.add_argument("--in", dest="input")
    b.add_argument("--pipeline")
    b.add_argument("--frames", type=int, default=1)
    b.add_argument("--warmup", type=int, default=1)
    b.add_argument("--format", choices=("table", "records"), default="table")
    b.add_argument("--dtype", choices=sorted(_DTYPES), default="f32")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--report-dir")
    b.add_argument("--host-input", action="store_true",
                   help="keep each frame's host->device copy inside the beamform row")
    b.set_defaults(func=_cmd_benchmark)
    r = sub.add_parser("reconstruct", help="WFRF file -> PGM images (batched engine)")
    r.add_argument("--in", dest="input", required=True)
    r.add_argument("--out-dir", required=True)
    r.add_argument("--interpolation", choices=("nearest", "linear"), default="linear")
    r.add_argument("--range-db", type=float, default=30.0)
    r.set_defaults(func=_cmd_reconstruct)
    s = sub.add_parser("simulate", help="synthesize RF frames into a WFRF file")
    s.add_argument("--phantom", help="phantom spec JSON (default: the paper's wire phantom)")
    s.add_argument("--ctx", required=True, help="acquisition context JSON")
    s.add_argument("--out", required=True)
    s.add_argument("--frames", type=int, default=1)
    s.add_argument("--n-samples", type=int, default=2048)
    s.add_argument("--dtype", choices=sorted(_DTYPES), default="f64")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--noise-std", type=float, default=0.0)
    s.set_defaults(func=_cmd_simulate)
    return ap


def cli_main(argv=None) -> int:
    from .errors import EchopipeError

    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except (EchopipeError, OSError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(cli_main())
