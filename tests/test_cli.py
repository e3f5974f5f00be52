"""The remat-compatible CLI (paper_1905_11722_b200.cli) against the reference
CLI's own outputs (tests/golden/cli.json, made by running reference cli.py):
exit codes, plan JSON bytes, stderr messages, simulate summary / trace /
schedule files, report table and CSV.  ``gen`` and the input-error paths run
on CPU; everything that plans runs on the GPU."""

from __future__ import annotations

import contextlib
import io
import json
import subprocess
import sys
from pathlib import Path

import pytest

from _util import golden
from paper_1905_11722_b200.cli import main

ROOT = Path(__file__).resolve().parents[1]


def _run(argv):
    so, se = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
        code = main(argv)
    return code, so.getvalue(), se.getvalue()


def _replay(rec, tmp_path, want_kind):
    graphs = {}
    for name, text in rec["graphs"].items():
        p = tmp_path / f"{name}.json"
        p.write_text(text)
        graphs[name] = str(p)
    n = 0
    for run in rec["runs"]:
        if run["argv"][0] != want_kind:
            continue
        files = {"plan": tmp_path / "plan.json", "trace": tmp_path / "trace.json",
                 "schedule": tmp_path / "sched.txt", "csv": tmp_path / "rows.csv",
                 "out": tmp_path / "out.json"}
        if "plan" in run:
            files["plan"].write_text(run["plan"])
        argv = []
        for a in run["argv"]:
            if a.startswith("@"):
                key = a[1:]
                argv.append(graphs[key] if key in graphs else str(files[key]))
            else:
                argv.append(a)
        if want_kind == "gen":
            argv += ["--out", str(files["out"])]
        code, so, se = _run(argv)
        assert code == run["code"], (run["argv"], se)
        if "stdout" in run:
            assert so == run["stdout"], run["argv"]
            assert se == run["stderr"], run["argv"]
        for k, text in run.get("files", {}).items():
            assert files[k].read_text() == text, (run["argv"], k)
        n += 1
    return n


def test_gen_matches_reference_bytes(tmp_path):
    assert _replay(golden("cli.json")[0], tmp_path, "gen") == 5


def test_help_exits_zero():
    assert _run(["--help"])[0] == 0


def test_bad_flags_are_input_errors():
    assert _run(["plan", "--graph", "x.json", "--budget", "4", "--algo", "magic"])[0] == 1
    assert _run(["frobnicate"])[0] == 1


def test_missing_file_is_input_error():
    assert _run(["plan", "--graph", "/nonexistent.json", "--budget", "4"])[0] == 1


def test_cyclic_graph_is_input_error(tmp_path):
    bad = tmp_path / "cyclic.json"
    bad.write_text(json.dumps({
        "nodes": [{"id": "a", "memory_cost": 1}, {"id": "b", "memory_cost": 1}],
        "edges": [["a", "b"], ["b", "a"]],
    }))
    code, _, err = _run(["plan", "--graph", str(bad), "--budget", "4"])
    assert code == 1 and "cycle detected" in err


def test_bad_budget_is_input_error(tmp_path):
    g = tmp_path / "c.json"
    assert _run(["gen", "--family", "chain", "--depth", "3", "--out", str(g)])[0] == 0
    code, _, err = _run(["plan", "--graph", str(g), "--budget", "lots"])
    assert code == 1 and "budget must be an integer or 'min'" in err


@pytest.mark.gpu
def test_plan_runs_match_reference(tmp_path):
    assert _replay(golden("cli.json")[0], tmp_path, "plan") > 100


@pytest.mark.gpu
def test_simulate_runs_match_reference(tmp_path):
    assert _replay(golden("cli.json")[0], tmp_path, "simulate") == 10


@pytest.mark.gpu
def test_report_runs_match_reference(tmp_path):
    assert _replay(golden("cli.json")[0], tmp_path, "report") == 5


@pytest.mark.gpu
def test_simulate_fault_exit_codes(tmp_path):
    g = tmp_path / "c.json"
    _run(["gen", "--family", "chain", "--depth", "3", "--out", str(g)])
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"segments": [["zzz"], ["v0", "v1", "v2"]]}))
    code, _, err = _run(["simulate", "--graph", str(g), "--plan", str(bad)])
    assert code == 3 and "zzz" in err
    bad.write_text(json.dumps({"segments": [["v1"], ["v0", "v2"]]}))
    code, _, err = _run(["simulate", "--graph", str(g), "--plan", str(bad)])
    assert code == 3 and "not a lower set" in err


@pytest.mark.gpu
def test_lattice_cap_env_override(tmp_path, monkeypatch):
    g = tmp_path / "wide.json"
    _run(["gen", "--family", "random-dag", "--depth", "5", "--edge-prob", "0.0", "--out", str(g)])
    monkeypatch.setenv("REMAT_LATTICE_CAP", "8")
    code, _, err = _run(["plan", "--graph", str(g), "--budget", "10"])
    assert code == 1 and "lattice too large" in err
    monkeypatch.delenv("REMAT_LATTICE_CAP")
    assert _run(["plan", "--graph", str(g), "--budget", "10"])[0] == 0


@pytest.mark.gpu
def test_module_entry_point(tmp_path):
    g = tmp_path / "c.json"
    _run(["gen", "--family", "chain", "--depth", "3", "--out", str(g)])
    proc = subprocess.run([sys.executable, "-m", "paper_1905_11722_b200.cli", "plan", "--graph",
                           str(g), "--budget", "min"], capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr
    assert json.loads(proc.stdout)["feasible"] is True
