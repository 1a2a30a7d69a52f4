"""The command-line drivers end to end on the GPU (commands.cpp eigs /
cluster / bench): the report agrees with the library API on the same input,
the dense-reference metrics come from the Direct backend, numerical failures
write a report and exit 1 (commands.cpp:258-277)."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1808_04580_b200 as fgs
from test_cli import EXE, check_report, run, write_spiral_csv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spiral(tmp_path_factory):
    from paper_1808_04580_b200 import build
    build.build()
    d = tmp_path_factory.mktemp("cli")
    out = d / "spiral.csv"
    write_spiral_csv(out, per_class=400, seed=4)
    return out


def test_eigs_report_matches_api(spiral, tmp_path):
    rep_path = tmp_path / "eigs.json"
    r = run(EXE, "eigs", "--in", spiral, "--out", rep_path, "--sigma", 3.5, "--k", 6, "--with-reference")
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    check_report(rep)
    assert rep["command"] == "eigs" and rep["method"] == "nfft-lanczos" and rep["status"] == "ok"
    m = rep["metrics"]
    assert m["lanczos_converged"]["value"] == 1.0
    assert m["max_residual_operator"]["value"] <= 1e-9
    assert m["max_eigenvalue_error"]["value"] <= 1e-5  # setup 2 (N=32, m=4) vs the exact operator
    assert m["max_residual"]["value"] <= 1e-4
    assert set(rep["timings_seconds"]) >= {"setup", "solve", "reference"}
    # the same solve through the library API: bitwise the same eigenvalues
    X = np.loadtxt(spiral, delimiter=",", skiprows=1)[:, :3]
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(3.5), fgs.FastsumParams.preset(2))
    pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-12, seed=1))
    assert np.array_equal(np.array(rep["eigenvalues"]), pairs.values)
    # and against the CPU oracle's lanczos_largest on the same file
    # (spectral.cpp:141-256 on the reference's fast operator): A-space values
    from oracle import oracle as orc
    ref = orc.AdjacencyOperator(X, 0, 3.5, N=32, m=4, p=4)  # preset 2 (fastsum.cpp:9-23)
    vals, _, _, conv = ref.lanczos_largest(6, max_iter=1000, tol=1e-12, seed=1)
    assert conv
    assert np.max(np.abs(np.asarray(rep["eigenvalues"]) - np.asarray(vals))) <= 1e-8


def test_eigs_direct_method(spiral, tmp_path):
    rep_path = tmp_path / "direct.json"
    r = run(EXE, "eigs", "--in", spiral, "--out", rep_path, "--sigma", 3.5, "--k", 4, "--method", "direct",
            "--with-reference")
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    assert rep["metrics"]["max_eigenvalue_error"]["value"] <= 1e-10


def test_cluster_writes_labels_and_rate(spiral, tmp_path):
    rep_path = tmp_path / "cl.json"
    r = run(EXE, "cluster", "--in", spiral, "--out", rep_path, "--sigma", 3.5, "--k", 5)
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    check_report(rep)
    labels = np.loadtxt(str(rep_path) + ".labels.csv", skiprows=1, dtype=int)
    assert labels.shape == (2000,) and labels.min() >= 0 and labels.max() < 5
    rate = rep["metrics"]["misclassification_rate_permuted"]["value"]
    truth = np.loadtxt(spiral, delimiter=",", skiprows=1)[:, 3].astype(int)
    assert rate == fgs.misclassification_rate_permuted(labels, truth)


def test_bench_sweep_report(tmp_path):
    rep_path = tmp_path / "bench.json"
    r = run(EXE, "bench", "--out", rep_path, "--sizes", "1000,2000", "--k", 4, "--with-reference", "--applies", 3)
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    check_report(rep)
    cells = rep["extra"]["cells"]
    assert [c["n"] for c in cells] == [1000, 2000]
    for c in cells:
        assert c["matvec_seconds"] > 0 and c["solve_seconds"] > 0
        assert c["eigenvalue_error"]["max"] <= 1e-5 and c["residual"]["max"] <= 1e-4
    assert "matvec_time_ratio" in rep["metrics"]


def test_numerical_failure_writes_report(tmp_path):
    p = tmp_path / "far.csv"
    p.write_text("x0\n0\n1000\n1000.5\n")
    rep_path = tmp_path / "fail.json"
    r = run(EXE, "eigs", "--in", p, "--out", rep_path, "--sigma", 0.01, "--k", 1, "--method", "direct")
    assert r.returncode == 1
    rep = json.loads(rep_path.read_text())
    assert rep["status"] == "numerical-failure" and "node 0" in rep["diagnostic"]
