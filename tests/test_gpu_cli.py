"""The reference's command-line protocol on the B200 backend (reference: cli.py)."""

import csv
import io
import json

import numpy as np
import pytest

from oracle import parcube_oracle as po
from paper_2302_05730_b200 import harness

pytestmark = pytest.mark.gpu


def test_integrate_pagani_json(capsys):
    rc = harness.main(["integrate", "--integrator", "pagani", "--integrand", "f4", "-d", "5", "--format", "json"])
    row = json.loads(capsys.readouterr().out)[0]
    assert rc == 0 and row["converged"] is True and row["reason"] == "tolerance met"
    assert (row["iterations"], row["regions_processed"]) == (10, 3328)            # BASELINE config 1
    assert abs(row["estimate"] - 1.791581473187015e-06) <= 1e-10 * 1.8e-06
    assert row["abs_deviation"] == abs(row["estimate"] - row["reference"])


def test_integrate_exit_code_one_when_not_converged(capsys):
    rc = harness.main(["integrate", "--integrator", "pagani", "--integrand", "f6", "-d", "5", "--max-iterations", "2"])
    out = capsys.readouterr().out
    assert rc == 1 and "reason: max iterations reached" in out


def test_integrate_mcubes_csv(capsys):
    rc = harness.main(["integrate", "--integrator", "mcubes", "--integrand", "f5", "-d", "5", "--samples", "1e5",
                       "--iterations", "4", "--seed", "3", "--format", "csv"])
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    want = po.mcubes_run("f5", 100000, 5, 4, seed=3)
    assert rc == 0 and abs(float(rows[0]["estimate"]) - want["estimate"]) <= 1e-9 * abs(want["estimate"])
    assert int(rows[0]["samples_per_iteration"]) == want["plan"]["m"] * want["plan"]["p"]


def test_compare_csv_schema(capsys, tmp_path):
    out = tmp_path / "cmp.csv"
    rc = harness.main(["compare", "--config-a", "workers=1", "--config-b", "workers=8", "--format", "csv", "--out", str(out),
                       "--scenario", "pagani:f4:d=5:g=4:reps=3", "--scenario", "mcubes:f5:d=5:n=1e5:reps=3"])
    lines = out.read_text().strip().splitlines()
    assert rc == 0 and lines[0] == harness.COMPARE_HEADER and len(lines) == 3
    assert lines[1].startswith("mcubes:f5") and lines[2].startswith("pagani:f4")      # sorted by id
    assert all(float(v) > 0 for v in lines[1].split(",")[1:3])


def test_bench_invoke_accumulator_matches_serial_sum(capsys):
    rc = harness.main(["bench-invoke", "--integrand", "f2", "-d", "6", "--points", "2000", "--repetitions", "3",
                       "--seed", "5", "--format", "json"])
    row = json.loads(capsys.readouterr().out)[0]
    pts = np.random.default_rng(5).random((2000, 6))
    acc = 0.0
    for v in po.genz_eval("f2", 6, pts):      # the reference's serial accumulation (cli.py:138-141)
        acc += float(v)
    assert rc == 0 and row["accumulator"] == acc and len(row["samples_ms"]) == 3 and row["invocations"] == 2000
