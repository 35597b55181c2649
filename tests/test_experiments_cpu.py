"""Experiment output formats (reference experiments.py:23-124) on CPU: CSV
header and value formatting, the truncation row, the manifest sidecar, and
the flop model against the numbers the reference publishes (BASELINE.md:
K = 30, T = 5 -> Jac-PCG 46,530 vs direct 108,029 flops, flops.py:35-69)."""
import csv
import json

import numpy as np
import pytest

from paper_2305_13925_b200 import experiments as E
from paper_2305_13925_b200.errors import ConfigurationError


def test_columns_and_fmt():
    assert E.CSV_COLUMNS["se_vs_m"] == ["M", "method", "mean_sum_se", "sem", "trials"]
    assert E._fmt(0.1 + 0.2) == "0.3"
    assert E._fmt(np.float64(1.0) / 3) == "0.333333333333"
    assert E._fmt(1e-20) == "1e-20"
    assert E._fmt(7) == "7" and E._fmt("cg") == "cg"


def test_flop_model_published_numbers():
    assert E.flop_model("jacpcg", 30, 5)[2] == 46530
    assert E.flop_model("direct", 30, 5)[2] == 108029
    rows = list(E.rows_flops([30], ["jacpcg", "cg", "gs", "jor", "direct"], 5))
    assert rows[0] == ["jacpcg", 30, 5, 4 * 900 + 60, 8 * 900 + 46 * 30 - 6, 46530]
    with pytest.raises(ConfigurationError):
        E.flop_model("qr", 4, 1)


def test_write_experiment_csv_and_manifest(tmp_path):
    out = tmp_path / "se.csv"
    rows = [[256, "jacpcg", 35.123456789012345, 0.25, 100], [256, "direct", 36.0, 0.5, 100]]
    E.write_experiment("se_vs_m", iter(rows), str(out), {"m_grid": [256]}, 7)
    with open(out, encoding="utf-8", newline="") as fh:
        got = list(csv.reader(fh))
    assert got[0] == E.CSV_COLUMNS["se_vs_m"]
    assert got[1] == ["256", "jacpcg", "35.123456789", "0.25", "100"]
    man = json.load(open(str(out) + ".manifest.json"))
    assert set(man) == {"config", "seed", "version", "timestamp", "wall_seconds", "output"}
    assert man["seed"] == 7 and man["config"] == {"m_grid": [256]} and man["output"] == str(out)


def test_write_experiment_truncation_row(tmp_path):
    out = tmp_path / "bad.csv"

    def gen():
        yield [1, "cg", 0.5, 0.1, 3]
        raise RuntimeError("boom")
    with pytest.raises(RuntimeError):
        E.write_experiment("se_vs_m", gen(), str(out), {}, 0)
    got = list(csv.reader(open(out, encoding="utf-8", newline="")))
    assert got[-1] == [E.TRUNCATION_MARKER, "RuntimeError", "", "", ""]
    with pytest.raises(ConfigurationError):
        E.write_experiment("nope", iter([]), str(out), {}, 0)
