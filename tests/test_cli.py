"""Command line (cli.py): argument errors, report schema, artifacts.

CPU part: usage/data errors and exit codes, the analytic flop estimate.
GPU part: ``fit-srm`` on the reference-written golden manifest writes the
reference's artifact set and a schema-1 report, with the same numbers as
``srm.fit`` on the same subjects.
"""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1608_04647_b200 import cli, data_io

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "sfab"


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_1608_04647_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_flop_estimate_is_the_reference_formula():
    # cli.py:66-75: 2(2VTK) + 2VK^2 + (2VK^2 - 2/3 K^3) per subject-iteration
    v, t, k = 30000, 1000, 50
    per = 4.0 * v * t * k + 4.0 * v * k * k - 2.0 / 3.0 * k ** 3
    assert cli.srm_flops_per_subject_iteration(v, t, k) == pytest.approx(per, rel=1e-15)
    assert cli.srm_flop_estimate([v, v], t, k, 3) == pytest.approx(6 * per, rel=1e-15)


def test_usage_and_data_errors(tmp_path):
    r = _run("fit-srm", "--manifest", str(GOLD / "manifest.json"), "--k", "0", "--out", str(tmp_path))
    assert r.returncode == 2 and json.loads(r.stderr.strip().splitlines()[-1])["error"] == "UsageError"
    r = _run("fit-srm", "--manifest", str(GOLD / "manifest.json"), "--k", "2", "--iters", "0", "--out", str(tmp_path))
    assert r.returncode == 2
    r = _run("fit-srm", "--k", "2", "--out", str(tmp_path))  # argparse: missing --manifest
    assert r.returncode == 2
    r = _run("bench", "--manifest", str(tmp_path / "missing.json"), "--k", "2")
    assert r.returncode == 1 and json.loads(r.stderr.strip().splitlines()[-1])["error"] == "FileNotFoundError"
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"subjects": [{"id": "a", "data_path": str(GOLD / "malformed" / "bad_magic.sfab")}]}))
    r = _run("bench", "--manifest", str(bad), "--k", "2")
    err = json.loads(r.stderr.strip().splitlines()[-1])
    assert r.returncode == 1 and err["error"] == "FormatError" and err["field"] == "magic" and err["offset"] == 0


def test_report_schema_keys():
    rep = cli.make_report("bench", "serial", 1, {"load": 1.0, "compute": 2.0, "communicate": 0.0}, [1.5], 4e9, {})
    assert set(rep) == {"schema", "command", "backend", "workers", "timings", "objective", "flops",
                        "gflops_per_s", "outputs"}
    assert rep["schema"] == 1 and rep["gflops_per_s"] == pytest.approx(2.0)


@pytest.mark.gpu
def test_fit_srm_artifacts(tmp_path):
    from paper_1608_04647_b200 import srm

    out = tmp_path / "out"
    r = _run("fit-srm", "--manifest", str(GOLD / "manifest.json"), "--k", "3", "--iters", "4", "--seed", "5",
             "--out", str(out))
    assert r.returncode == 0, r.stderr
    rep = json.loads((out / "report.json").read_text())
    assert rep["schema"] == 1 and rep["command"] == "fit-srm" and rep["workers"] == 1
    assert len(rep["objective"]) == 4 and rep["flops"] > 0 and rep["device"]["em_iterations"] == 4
    man = data_io.load_manifest(GOLD / "manifest.json", model="srm")
    subs = [data_io.load_subject(e.data_path, None, e.subject_id) for e in man.subjects]
    m = srm.fit([srm.SubjectData(s.subject_id, s.X) for s in subs], srm.SrmConfig(k=3, iterations=4, seed=5))
    assert np.array_equal(data_io.load_matrix(out / "shared_response.sfab"), m.S)
    assert np.array_equal(data_io.load_matrix(out / "shared_covariance.sfab"), m.sigma_s)
    assert np.array_equal(data_io.load_matrix(out / "noise_variance.sfab")[:, 0], m.rho2_all)
    for sid, w, mu in zip(m.subject_ids, m.W, m.mu):
        assert np.array_equal(data_io.load_matrix(out / "subjects" / f"{sid}_mapping.sfab"), w)
        assert np.array_equal(data_io.load_matrix(out / "subjects" / f"{sid}_mean.sfab")[:, 0], mu)
    assert rep["objective"] == pytest.approx(m.objective_trace, rel=0, abs=0)
