"""GPU runs of the precision suite (vs the reference's own digits-lost
table, tests/golden/precision_ref.csv) and the CLI compute command."""
from __future__ import annotations

import csv
import io

import pytest

from conftest import GOLDEN
from paper_2510_03421_b200 import cli, precision as PR

pytestmark = pytest.mark.gpu


def _rows(text):
    return {(r["family"], r["algorithm"], int(r["m"]), int(r["n"]), r["kind"]): r
            for r in csv.DictReader(io.StringIO(text))}


def test_precision_suite_vs_reference():
    """Same grid as `permanent precision --max-n 16 --attempts 200`: the same
    overflow flags; per (family, algorithm, kind) the mean digits lost is no
    worse than the reference's and the maximum within 1.2 digits of it
    (single cells of the ill-conditioned Ryser/Cauchy family vary by about a
    digit either way with the rounding order); cell by cell within 1.5."""
    ref = _rows((GOLDEN / "precision_ref.csv").read_text())
    ours = _rows(PR.precision_csv(PR.run_precision_suite(n_range=range(2, 17), seed=0, cauchy_attempts=200)))
    assert set(ours) == set(ref)
    worst_ref, worst_ours, diff = {}, {}, {}
    for key, r in ref.items():
        o = ours[key]
        assert o["overflow"] == r["overflow"], key
        if r["overflow"] == "true":
            continue
        dr, do = float(r["digits_lost"]), float(o["digits_lost"])
        assert do <= max(dr, 0.0) + 1.5, (key, do, dr)
        g = key[:2] + (key[4],)
        worst_ref[g] = max(worst_ref.get(g, -9), dr)
        worst_ours[g] = max(worst_ours.get(g, -9), do)
        diff.setdefault(g, []).append(do - max(dr, 0.0))
    for g in worst_ref:
        assert worst_ours[g] <= max(worst_ref[g], 0.0) + 1.2, (g, worst_ours[g], worst_ref[g])
        assert sum(diff[g]) / len(diff[g]) <= 0.05, (g, sum(diff[g]) / len(diff[g]))


def test_cli_compute(capsys):
    assert cli.main(["compute", "1 2 3; 4 5 6; 7 8 9"]) == 0
    assert capsys.readouterr().out.strip() == "450"
    assert cli.main(["compute", "--algorithm", "ryser_rectangular", "1 1 1 1; 1 1 1 1"]) == 0
    assert capsys.readouterr().out.strip() == "12"
    assert cli.main(["compute", "--algorithm", "glynn", "0.5 0.25; 1 2"]) == 0
    assert float(capsys.readouterr().out) == pytest.approx(1.25)
    assert cli.main(["compute", "--verbose", "1+1i 0; 0 1"]) == 0
    out = capsys.readouterr()
    assert "algorithm:" in out.err and out.out.strip().endswith("i")
    assert cli.main(["compute", "4611686018427387904 3; 5 4611686018427387904"]) == 3


def test_bench_engine_line_contract():
    """`bench.py` on the GPU (a short n = 30 run): one JSON line carrying
    the driver's keys, the self-check against the committed double-double
    value, the roofline / cpu_baseline / e2e objects, the launch count and
    the clock samples."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--n", "30", "--no-configs",
           "--cpu-seconds", "1"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, check=True).stdout.strip().splitlines()
    assert len(out) == 1
    line = json.loads(out[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in line, key
    assert line["unit"] == "steps/s" and line["n_gpus"] == 1 and line["steps"] == 3 and line["dtype"] == "f64"
    assert line["vs_baseline"] is None and line["gpu_launches"] >= 3
    assert line["config"]["value_check"]["checked"] is True and line["config"]["value_check"]["rel_err"] <= 1e-10
    assert abs(line["value"] - (1 << 29) / (line["ms_per_step"] * 1e-3)) <= 1e-6 * line["value"]
    rf = line["roofline"]
    assert 0.5 < rf["frac"] <= 1.02 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] == 1 and cb["value"] > 0
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] == 30 * 30 * 8 and e2e["d2h_bytes_per_step"] > 0
    assert 0 < e2e["value"] <= line["value"] * 1.01
    clocks = line["clocks"]  # a run this short may end before the first nvidia-smi sample
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(clocks)
    assert clocks["sm_mhz"] is None or clocks["sm_mhz"] > 0
    assert not any("slowdown" in r for r in clocks["reasons"])
