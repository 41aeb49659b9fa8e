"""CPU: the Table-1 report surface (report.py mirror of the reference's
report.py:28-148) on synthetic stage timings -- row grouping (analytic +
envelope summed per frame before the median), table / records / CSV output,
and the CLI's argument handling."""

import csv
import json

import pytest

from paper_1811_01566_b200 import cli
from paper_1811_01566_b200 import report as R
from paper_1811_01566_b200.pipeline import BenchmarkResult, StageTiming, bmode_chain, build_graph


def _result(per_frame):
    frames = [StageTiming(tuple(st), total) for st, total in per_frame]
    stages = tuple((n, sorted(t.stage_ms(n) for t in frames)[len(frames) // 2])
                   for n, _ in frames[0].stages)
    return BenchmarkResult(StageTiming(stages, sorted(t.total_ms for t in frames)[len(frames) // 2]),
                           frames, len(frames), 0)


def test_stage_rows_sum_grouped_stages_per_frame_before_the_median():
    graph = build_graph(bmode_chain())
    res = _result([
        ([("beamform", 1.0), ("analytic_signal", 0.1), ("envelope", 0.5),
          ("dynamic_adjustment", 0.2)], 1.9),
        ([("beamform", 2.0), ("analytic_signal", 0.4), ("envelope", 0.1),
          ("dynamic_adjustment", 0.3)], 2.9),
        ([("beamform", 3.0), ("analytic_signal", 0.2), ("envelope", 0.2),
          ("dynamic_adjustment", 0.1)], 3.6),
    ])
    rows = R.stage_rows(graph, res)
    assert [r for r, _ in rows] == ["Beamforming", "Envelope Detection", "Dynamic Adjustment"]
    # per-frame sums 0.6, 0.5, 0.4 -> median 0.5 (the medians of the parts would give 0.4)
    assert dict(rows)["Envelope Detection"] == pytest.approx(0.5)
    assert dict(rows)["Beamforming"] == 2.0


def test_report_table_records_and_csv(tmp_path):
    graph = build_graph(bmode_chain())
    st = [("beamform", 0.09), ("analytic_signal", 0.001), ("envelope", 0.002),
          ("dynamic_adjustment", 0.003)]
    rep = R.make_report([("STAI", graph, _result([(st, 0.5)])),
                         ("PWI", graph, _result([(st, 0.25)]))])
    assert rep.columns == ["STAI [ms/frame]", "PWI [ms/frame]"]
    assert rep.fps == [2000.0, 4000.0]
    text = R.format_table(rep).splitlines()
    assert text[0].split() == ["Step", "STAI", "[ms/frame]", "PWI", "[ms/frame]"]
    assert text[2].startswith("Beamforming") and text[2].split()[-2:] == ["0.090", "0.090"]
    assert text[-1].split()[-2:] == ["2000.00", "4000.00"]
    recs = [json.loads(l) for l in R.format_records(rep).splitlines()]
    assert {"mode": "PWI", "step": "FPS", "value": 4000.0} in recs
    assert {"mode": "STAI", "step": "Envelope Detection", "ms_per_frame": 0.003} in recs
    R.write_csv(rep, tmp_path / "b.csv")
    rows = list(csv.reader(open(tmp_path / "b.csv")))
    assert rows[0] == ["step", "STAI [ms/frame]", "PWI [ms/frame]"]
    assert rows[-1][0] == "FPS" and float(rows[-1][2]) == 4000.0


def test_cli_usage_errors_exit_2_and_missing_inputs_exit_1(capsys):
    assert cli.cli_main(["benchmark", "--synthetic", "nope"]) == 2
    assert cli.cli_main(["benchmark"]) == 1
    assert "needs --synthetic" in capsys.readouterr().err
    assert cli.cli_main(["reconstruct", "--in", "/nonexistent.wfrf", "--out-dir", "/tmp/x"]) == 1
