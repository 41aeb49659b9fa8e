"""GPU: the reference's benchmark / reconstruct commands on the B200 path
(cli.py:85-167): Table 1 rows from CUDA-event stage times for the paper
presets, and a WFRF dataset reconstructed to PGM files by the batched
engine, equal to the per-frame drop-in chain."""

import json
import os

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import cli

pytestmark = pytest.mark.gpu


def test_benchmark_table1_rows_for_both_presets(capsys, tmp_path):
    rc = cli.cli_main(["benchmark", "--synthetic", "sta-paper", "--synthetic", "pwi-paper",
                       "--frames", "3", "--warmup", "1", "--format", "records",
                       "--report-dir", str(tmp_path)])
    assert rc == 0
    recs = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    for mode in ("STAI", "PWI"):
        steps = {r["step"]: r for r in recs if r["mode"] == mode}
        assert set(steps) == {"Beamforming", "Envelope Detection", "Dynamic Adjustment", "Total",
                              "FPS"}
        assert steps["Beamforming"]["ms_per_frame"] > steps["Dynamic Adjustment"]["ms_per_frame"]
        assert steps["FPS"]["value"] > 50.0  # the paper's Titan X: 55 STAI / 17 PWI fps
    assert os.path.exists(tmp_path / "benchmark.csv")


def test_reconstruct_wfrf_to_pgm_equals_drop_in_chain(golden_dir, tmp_path):
    path = os.path.join(golden_dir, "ref_small.wfrf")
    assert cli.cli_main(["reconstruct", "--in", path, "--out-dir", str(tmp_path)]) == 0
    frames, ctx = bm.read_wfrf(path)
    grid = bm.default_grid(ctx, frames[0].n_samples, "sta")
    graph = bm.build_graph(bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                                                "z_positions": grid.z_positions.tolist()}))
    for i, fr in enumerate(frames):
        disp = bm.execute(graph, (fr, ctx))[0]["dynamic_adjustment"]
        ref = tmp_path / "ref.pgm"
        bm.write_pgm(bm.BmodeImage(disp.numpy(), stage="display", grid=grid), ref)
        assert open(tmp_path / f"frame_{i:04d}.pgm", "rb").read() == open(ref, "rb").read()
