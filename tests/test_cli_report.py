"""Front end and reports: report round-trips on CPU,
usage/runtime exit codes, and -- on a GPU -- end-to-end CLI solves."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_1301_5914_b200 import _native as N
from paper_1301_5914_b200.cli import main
from paper_1301_5914_b200.report import (REPORT_COLUMNS, RunReport, ScalingRow, reports_from_csv,
                                         reports_from_json, reports_to_csv, reports_to_json,
                                         scaling_to_csv, scaling_to_json, strip_timings)


def _report(**kw):
    base = dict(mesh_source="icosphere level=3 radius=2.0", n_vertices=642, n_faces=1280, eps1=1.0,
                eps2=80.0, kappa=0.1257, n_charges=1, scheme="hobi", workers=1, rule_id="conical-radau-4",
                rule_degree=3, energy_kcal=-82.18921350940137, phi_error=3.2e-5, observed_order=None,
                iterations=6, residual=2.87e-8, time_discretize_s=0.1, time_solve_s=0.002,
                time_energy_s=0.001, memory_lower_bound_mb=1.5, gpus=1, matvecs=8, pairs_per_s=1.2e10)
    base.update(kw)
    return RunReport(**base)


def test_report_round_trips():
    reps = [_report(), _report(phi_error=None, observed_order=1.5, scheme="lobi")]
    assert reports_from_json(reports_to_json(reps)) == reps
    assert reports_from_csv(reports_to_csv(reps)) == reps
    assert reports_to_csv(reps).splitlines()[0].split(",") == list(REPORT_COLUMNS)
    assert strip_timings(reps[0]).time_solve_s == 0.0 and strip_timings(reps[0]).pairs_per_s == 0.0
    with pytest.raises(ValueError, match="not finite"):
        _report(residual=float("nan"))
    with pytest.raises(ValueError, match="header"):
        reports_from_csv("a,b\n1,2\n")
    rows = [ScalingRow(1, 1.0, 1.0, 0.0), ScalingRow(2, 0.51, 0.98, 0.0)]
    assert json.loads(scaling_to_json(rows, {"n_faces": 1280}))["scaling"][1]["workers"] == 2
    assert scaling_to_csv(rows).splitlines()[0] == "workers,time_solve_s,efficiency,max_solution_diff"


def test_usage_errors_exit_2(capsys):
    for argv in (["solve"], ["solve", "--sphere", "3"], ["scaling", "--workers-list", "x"],
                 ["convergence", "--charge-position", "1,2"]):
        with pytest.raises(SystemExit) as info:
            main(argv)
        assert info.value.code == 2


def test_runtime_error_exit_1(tmp_path, capsys):
    bad = tmp_path / "q.txt"
    bad.write_text("1 2 3\n")
    assert main(["solve", "--sphere", "1,2.0", "--charges", str(bad)]) == 1
    assert capsys.readouterr().err.startswith("error: MeshFormatError: charge line 1")


@pytest.mark.gpu
def test_cli_solve_and_convergence(tmp_path, capsys):
    q = tmp_path / "q.txt"
    q.write_text("0 0 0 1.0\n")
    out = tmp_path / "r.json"
    assert main(["solve", "--sphere", "3,2.0", "--charges", str(q), "--kappa", "0.1257", "--restart",
                 "10", "--out", str(out)]) == 0
    rep = reports_from_json(out.read_text())[0]
    assert rep.energy_kcal == pytest.approx(-82.18921350940137, rel=1e-8)
    assert rep.iterations == 6 and rep.matvecs == 8 and rep.phi_error < 1e-4
    assert "E_sol = -82.1892" in capsys.readouterr().out  # summary line when --out is given
    assert main(["convergence", "--levels", "2,3", "--kappa", "0.1257", "--format", "csv"]) == 0
    reps = reports_from_csv(capsys.readouterr().out)
    assert len(reps) == 2 and reps[1].phi_error < reps[0].phi_error and reps[1].observed_order > 0


@pytest.mark.gpu
def test_cli_scaling_one_gpu(tmp_path):
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "paper_1301_5914_b200", "scaling", "--sphere", "2,2.0",
                        "--kappa", "0.1257", "--workers-list", "1,2"], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = json.loads(r.stdout)["scaling"]
    assert rows[0]["workers"] == 1 and rows[0]["max_solution_diff"] == 0.0
    if N.device_count() >= 2:
        assert rows[1]["max_solution_diff"] == 0.0
