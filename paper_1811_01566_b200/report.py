"""Table-1 benchmark report for GPU stage timings.

Same surface as the reference's report module (report.py:28-148) so a user's
benchmark scripts keep working: ``stage_rows``, ``BenchmarkReport``,
``make_report``, ``format_table``, ``report_records``, ``format_records``,
``write_csv``.  It accepts this package's ``BenchmarkResult`` (CUDA-event
stage times, pipeline.benchmark) and the reference's own (echopipe's
host-clock benchmark running the B200 kinds, which synchronise per node), as
both carry ``per_frame`` StageTimings and a ``timing.total_ms``.

Row grouping follows the paper's table: analytic signal and envelope form
"Envelope Detection"; per frame the grouped stage times are added before the
median over frames (report.py:36-57).  Figures need matplotlib, which this
image does not ship, so ``save_timing_figure`` raises ImportError cleanly
instead of failing at import time as the reference module does.
"""

from __future__ import annotations

import csv
import json
import statistics
from dataclasses import dataclass, field

TABLE1_ROWS = {
    "beamform": "Beamforming",
    "analytic_signal": "Envelope Detection",
    "envelope": "Envelope Detection",
    "dynamic_adjustment": "Dynamic Adjustment",
}


def _row_of(graph, node: str) -> str:
    kind = graph.node_kind(node) if hasattr(graph, "node_kind") else graph.nodes[node].kind.name
    return TABLE1_ROWS.get(kind, node)


def stage_rows(graph, result) -> list[tuple[str, float]]:
    """(row label, median ms/frame) in graph order; unknown kinds keep one
    row per node."""
    members: dict[str, list[str]] = {}
    for node in graph.order:
        members.setdefault(_row_of(graph, node), []).append(node)
    out = []
    for label, nodes in members.items():
        per_frame = [sum(t.stage_ms(n) for n in nodes) for t in result.per_frame]
        out.append((label, statistics.median(per_frame)))
    return out


@dataclass
class BenchmarkReport:
    """Runs as columns ("<mode> [ms/frame]"), grouped stages as rows."""

    columns: list = field(default_factory=list)
    row_labels: list = field(default_factory=list)
    cells: list = field(default_factory=list)  # [row][column], None where absent
    totals: list = field(default_factory=list)
    fps: list = field(default_factory=list)


def make_report(runs) -> BenchmarkReport:
    """``runs``: iterable of (mode label, graph, BenchmarkResult)."""
    runs = list(runs)
    per_run = [dict(stage_rows(g, r)) for _, g, r in runs]
    labels: list[str] = []
    for rows in per_run:
        labels.extend(k for k in rows if k not in labels)
    rep = BenchmarkReport(row_labels=labels)
    rep.cells = [[rows.get(label) for rows in per_run] for label in labels]
    for mode, _, res in runs:
        total = res.timing.total_ms
        rep.columns.append(f"{mode} [ms/frame]")
        rep.totals.append(total)
        rep.fps.append(1000.0 / total if total > 0 else float("inf"))
    return rep


def format_table(report: BenchmarkReport) -> str:
    """Aligned text: a header, one line per row, then Total and FPS."""
    first = max(len(s) for s in ["Step", "Total [ms/frame]", "FPS", *report.row_labels])
    widths = [max(12, len(c)) for c in report.columns]

    def line(label, values, spec):
        cells = []
        for v, w in zip(values, widths):
            cells.append(("-" if v is None else format(v, spec)).rjust(w))
        return f"{label:<{first}}  " + "  ".join(cells)

    head = f"{'Step':<{first}}  " + "  ".join(c.rjust(w) for c, w in zip(report.columns, widths))
    rule = "-" * len(head)
    body = [line(label, row, ".3f") for label, row in zip(report.row_labels, report.cells)]
    return "\n".join([head, rule, *body, rule, line("Total [ms/frame]", report.totals, ".3f"),
                      line("FPS", report.fps, ".2f")])


def report_records(report: BenchmarkReport) -> list[dict]:
    """One dict per cell, then a Total and an FPS record per run."""
    recs = []
    for j, col in enumerate(report.columns):
        mode = col.split(" ", 1)[0]
        recs += [{"mode": mode, "step": label, "ms_per_frame": row[j]}
                 for label, row in zip(report.row_labels, report.cells) if row[j] is not None]
        recs.append({"mode": mode, "step": "Total", "ms_per_frame": report.totals[j]})
        recs.append({"mode": mode, "step": "FPS", "value": report.fps[j]})
    return recs


def format_records(report: BenchmarkReport) -> str:
    return "\n".join(json.dumps(r) for r in report_records(report))


def write_csv(report: BenchmarkReport, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["step", *report.columns])
        for label, row in zip(report.row_labels, report.cells):
            w.writerow([label, *("" if v is None else repr(v) for v in row)])
        w.writerow(["Total [ms/frame]", *map(repr, report.totals)])
        w.writerow(["FPS", *map(repr, report.fps)])


def save_timing_figure(report: BenchmarkReport, path) -> None:
    """Bar chart of the table (needs matplotlib)."""
    import matplotlib

    matplotlib.use("Agg")
    import matplotlib.pyplot as plt

    fig, ax = plt.subplots(figsize=(6, 3.5))
    n = len(report.columns)
    for j, col in enumerate(report.columns):
        vals = [row[j] or 0.0 for row in report.cells]
        ax.bar([i + j / (n + 1) for i in range(len(vals))], vals, width=1 / (n + 1), label=col)
    ax.set_xticks(range(len(report.row_labels)), report.row_labels)
    ax.set_ylabel("ms / frame")
    ax.legend()
    fig.tight_layout()
    fig.savefig(path)
    plt.close(fig)
