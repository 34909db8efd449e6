"""Command line: generation, solve, bench, plot and the
exit codes 0 / 1 / 2."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2305_07030_b200 import cli
from paper_2305_07030_b200.benchmark import SpeedupRow

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gen_is_deterministic(tmp_path):
    a, b = tmp_path / "a.net", tmp_path / "b.net"
    assert cli.main(["gen", "--lattice", "2,2,2", "--seed", "0", "-o", str(a)]) == 0
    assert cli.main(["gen", "--lattice", "2,2,2", "--seed", "0", "-o", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()


def test_gen_grid_counts(tmp_path):
    out = tmp_path / "c.net"
    assert cli.main(["gen", "--lattice", "3,3,3", "--jitter", "0", "--seed", "0", "-o", str(out)]) == 0
    text = out.read_text()
    assert "nodes 27" in text and "elements 54" in text


def test_usage_errors_exit_1(tmp_path, capsys):
    assert cli.main(["gen", "--lattice", "1,2,2", "-o", str(tmp_path / "x")]) == 1
    assert cli.main(["gen", "--bogus"]) == 1
    assert cli.main(["solve", "--network", str(tmp_path / "missing.net"), "--deform"] + ["1"] * 9) == 1
    assert "error" in capsys.readouterr().err


def test_plot_is_deterministic_and_counts_polylines(tmp_path):
    rows = [SpeedupRow("team", d, n, 1.0, float(n) / 2, None) for d in (300, 3000) for n in (1, 4, 16)]
    from paper_2305_07030_b200.benchmark import SUMMARY_HEADER, emit_csv
    csv_path = tmp_path / "s.csv"
    csv_path.write_text(emit_csv(rows, SUMMARY_HEADER))
    a, b = tmp_path / "a.svg", tmp_path / "b.svg"
    assert cli.main(["plot", "--input", str(csv_path), "-o", str(a)]) == 0
    assert cli.main(["plot", "--input", str(csv_path), "-o", str(b)]) == 0
    svg = a.read_text()
    assert a.read_bytes() == b.read_bytes()
    assert svg.count("<polyline") == 2 and all(line.count(",") == 3 for line in svg.splitlines()
                                                if line.startswith("<polyline"))
    empty = tmp_path / "e.csv"
    empty.write_text(emit_csv([], SUMMARY_HEADER))
    assert cli.main(["plot", "--input", str(empty), "-o", str(a)]) == 0
    assert "<svg" in a.read_text() and "<polyline" not in a.read_text()


def test_module_entry_point_runs(tmp_path):
    out = tmp_path / "m.net"
    proc = subprocess.run([sys.executable, "-m", "paper_2305_07030_b200", "gen", "--lattice", "2,2,3", "-o", str(out)],
                          cwd=ROOT, capture_output=True, text=True)
    assert proc.returncode == 0 and out.read_text().startswith("nodes 12")


@pytest.mark.gpu
def test_solve_exit_codes_and_bar(cuda_device, tmp_path):
    bar = tmp_path / "bar.net"
    bar.write_text("nodes 3\n0 0 0\n0.5 0 0\n1 0 0\nelements 2\n0 1 0\n1 2 0\nmaterials 1\n1 1 1\nboundary 2\n0\n2\n")
    res = tmp_path / "r.json"
    F = ["1.1", "0", "0", "0", "1", "0", "0", "0", "1"]
    assert cli.main(["solve", "--network", str(bar), "--deform", *F, "-o", str(res)]) == 0
    doc = json.loads(res.read_text())
    assert abs(doc["u"][3] - 0.05) < 1e-6 and doc["converged"]
    ident = ["1", "0", "0", "0", "1", "0", "0", "0", "1"]
    assert cli.main(["solve", "--network", str(bar), "--deform", *ident, "-o", str(res)]) == 0
    assert not np.any(json.loads(res.read_text())["u"])
    assert cli.main(["solve", "--network", str(bar), "--deform", *F, "--max-iters", "2", "-o", str(res)]) == 2
    assert cli.main(["solve", "--network", str(bar), "--deform", *F, "--strategy", "naive", "-o", str(res)]) == 0


@pytest.mark.gpu
def test_bench_one_cell(cuda_device, tmp_path):
    out = tmp_path / "raw.csv"
    assert cli.main(["bench", "--sizes", "3,3,3", "--counts", "1", "--reps", "1", "--strategies", "serial",
                     "-o", str(out)]) == 0
    assert len(out.read_text().strip().splitlines()) == 2
    summ = (tmp_path / "raw.summary.csv").read_text().strip().splitlines()
    assert summ[1].split(",")[4] == "1.0"
