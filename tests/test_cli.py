"""Ports of the reference's test_cli.cpp (/root/reference/proj/tests) against
`python -m paper_2207_06374_b200.cli` (exit codes, CSV/JSON outputs and the
solve -> certify consistency contract)."""
import json
import math
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2207_06374_b200.cli", *args], cwd=ROOT,
                       capture_output=True, text=True)
    return r.returncode, r.stdout + r.stderr


def test_bounds_prints_exact_closed_forms():  # test_cli.cpp:50-56
    code, out = run_cli("bounds", "--d", "3", "--N", "9")
    assert code == 0
    assert "N,welch,orthoplex,levenshtein,gerzon_max" in out
    assert "9,0.5,,,9" in out


def test_bounds_range_populates_orthoplex_only_past_d_squared():  # test_cli.cpp:58-79
    code, out = run_cli("bounds", "--d", "2", "--N-range", "3:7")
    assert code == 0
    rows = [l.split(",") for l in out.strip().splitlines()[1:]]
    assert len(rows) == 5
    for cells in rows:
        n = int(cells[0])
        assert (cells[2] == "") == (n <= 4)


def test_usage_errors_exit_with_code_2():  # test_cli.cpp:81-89
    assert run_cli("solve", "--N", "4")[0] == 2            # missing --d
    assert run_cli("solve", "--d", "3", "--N", "2")[0] == 2  # N < d
    assert run_cli("bounds", "--d", "2")[0] == 2             # no N or range
    assert run_cli("bounds", "--d", "2", "--N-range", "9:3")[0] == 2
    assert run_cli("certify", "--in", "/no/such/file.json")[0] == 2
    assert run_cli("distortion", "--in", "/no/such/file.json")[0] == 2
    assert run_cli("distortion", "--in", "/no/such/file.json", "--samples", "0")[0] == 2
    assert run_cli("nonsense")[0] == 2


def test_help_exits_cleanly():  # test_cli.cpp:91-96
    code, out = run_cli("--help")
    assert code == 0 and "solve" in out


@pytest.mark.gpu
def test_solve_writes_a_record_that_certify_reproduces_exactly():  # test_cli.cpp:125-160
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "run.json")
        code, out = run_cli("solve", "--d", "2", "--N", "4", "--restarts", "4", "--seed", "7", "--out", path)
        assert code == 0 and "d=2 N=4" in out
        record = json.load(open(path))
        best = record["best_coherence"]
        assert best <= 0.5774 + 1e-3
        frame_path = os.path.join(tmp, "frame.json")
        json.dump(record["best_frame"], open(frame_path, "w"))
        code, out = run_cli("certify", "--in", frame_path, "--tol", "1e-6")
        assert code == 0
        report = json.loads(out)
        assert report["coherence"] == best
        assert any(c["kind"] == "etf" for c in report["certificates"])
        assert abs(report["targets"]["conjecture1"] - 1.0 / math.sqrt(3.0)) <= 1e-15


@pytest.mark.gpu
def test_sweep_writes_records_and_monotone_csv():  # main.cpp:198-267
    with tempfile.TemporaryDirectory() as tmp:
        code, out = run_cli("sweep", "--d", "2", "--N-range", "3:5", "--restarts", "2", "--out", tmp)
        assert code == 0
        lines = open(os.path.join(tmp, "sweep_d2.csv")).read().strip().splitlines()
        assert lines[0] == "N,coherence,coherence_monotone,welch,orthoplex,levenshtein" and len(lines) == 4
        mono = [float(l.split(",")[2]) for l in lines[1:]]
        assert mono == sorted(mono)
        for n in (3, 4, 5):
            assert json.load(open(os.path.join(tmp, "run_d2_N%d.json" % n)))["schema_version"] == 1


@pytest.mark.gpu
def test_distortion_is_deterministic_for_a_fixed_seed():  # test_cli.cpp:107-123
    from tests.test_records import sic_2_4
    from paper_2207_06374_b200 import records as rec
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "sic.json")
        rec.save_frame(path, sic_2_4(), 2, 4)
        a = run_cli("distortion", "--in", path, "--samples", "20000", "--seed", "5")
        b = run_cli("distortion", "--in", path, "--samples", "20000", "--seed", "5")
        assert a[0] == 0 and a == b
        report = json.loads(a[1])
        assert report["samples"] == 20000 and 0.0 <= report["estimate"] <= 1.0
        assert abs(report["coherence_of_codebook"] - 1.0 / math.sqrt(3.0)) <= 1e-12
