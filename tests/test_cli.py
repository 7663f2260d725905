"""The sweep CLI (mirrors the reference's tests/test_cli.py:304-359)."""

from __future__ import annotations

import subprocess
import sys

import pytest

from paper_2201_02789_b200.bench import CSV_COLUMNS
from paper_2201_02789_b200.cli import build_parser, main

from conftest import ROOT


def test_flags_parse_like_the_reference():
    a = build_parser().parse_args(
        ["sweep", "--bench", "bfs", "--dataset", "hand", "--thresholds",
         "0,32,inf", "--aggs", "none,block,warp", "--cfactors", "1,8"])
    assert a.thresholds == [0, 32, 2147483647]
    assert a.aggs == [None, "block", "warp"]
    assert a.cfactors == [1, 8]


def test_bad_flag_values_exit_nonzero(capsys):
    assert main(["sweep", "--bench", "bfs", "--dataset", "hand",
                 "--aggs", "tile"]) != 0
    assert main(["sweep", "--bench", "bfs", "--dataset", "hand",
                 "--thresholds", "x"]) != 0


def test_failing_rows_give_exit_code_1_without_device(capsys):
    rc = main(["sweep", "--bench", "manylaunch", "--dataset",
               "sizes:40:seed3", "--aggs", "multiblock", "--agg-threshold",
               "4", "--no-verify"])
    out = capsys.readouterr()
    assert rc == 1
    assert out.out.splitlines()[0] == ",".join(CSV_COLUMNS)
    assert "aggregation threshold requires block granularity" in out.err


def test_unknown_benchmark_is_an_error(capsys):
    assert main(["sweep", "--bench", "mst", "--dataset", "hand"]) == 1
    assert "unknown benchmark" in capsys.readouterr().err


@pytest.mark.gpu
def test_sweep_subprocess_default_grid(tmp_path):
    out = tmp_path / "rows.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2201_02789_b200",
                        "sweep", "--bench", "bfs", "--dataset", "hand",
                        "--report", str(out)], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert len(lines) == 13 and lines[0] == ",".join(CSV_COLUMNS)
    # deterministic columns (everything but timings) repeat exactly
    r2 = subprocess.run([sys.executable, "-m", "paper_2201_02789_b200",
                         "sweep", "--bench", "bfs", "--dataset", "hand"],
                        cwd=ROOT, capture_output=True, text=True, timeout=300)
    keep = CSV_COLUMNS.index("instructions")
    assert [ln.split(",")[:keep] for ln in lines] == \
        [ln.split(",")[:keep] for ln in r2.stdout.splitlines()]
