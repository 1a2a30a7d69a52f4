"""GPU nystrom_gaussian (nystrom.cu) against the oracle restatement
(spectral.cpp:384-444) on the same operator and seed: same probes (same
mt19937_64 stream), same 2L applies (ours as block applies), Householder QR
(cuSOLVER vs the oracle's), symmetric eigensolves (Jacobi vs tridiagonal QL).
Agreement is to rounding of well-separated pairs."""
import json

import numpy as np
import pytest

import paper_1808_04580_b200 as fgs
from test_cli import EXE, check_report, run, write_spiral_csv

pytestmark = pytest.mark.gpu


def _case(orc, n=2500, d=3, sigma=0.12, seed=7):
    X = orc.random_cloud(n, d, 0.25, seed)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(sigma), fgs.FastsumParams(32, 4, 4, 0.0))
    ref = orc.AdjacencyOperator(X, 0, sigma, N=32, m=4, p=4)
    return X, op, ref


def test_nystrom_matches_oracle(orc):
    X, op, ref = _case(orc)
    opts = fgs.NystromOptions(k=4, L=30, M=8, seed=3)
    got = fgs.nystrom_gaussian(op, opts)
    vals, vecs = orc.nystrom_adjacency(ref, X.shape[0], 4, 30, 8, seed=3)
    assert np.max(np.abs(got.values - vals) / np.abs(vals)) <= 1e-9
    gaps = np.abs(np.diff(vals))
    for j in range(4):
        sep = min(gaps[j - 1] if j > 0 else np.inf, gaps[j] if j < 3 else np.inf)
        if sep > 1e-3 * abs(vals[0]):
            assert np.linalg.norm(got.vectors[:, j] - vecs[:, j]) <= 1e-7
    assert np.max(np.abs(got.vectors.T @ got.vectors - np.eye(4))) <= 1e-10
    for j in range(4):
        col = got.vectors[:, j]
        assert col[np.argmax(np.abs(col))] > 0


def test_nystrom_deterministic_and_errors(orc):
    X, op, _ = _case(orc, n=1200, seed=9)
    opts = fgs.NystromOptions(k=3, L=20, M=5, seed=17)
    a, b = fgs.nystrom_gaussian(op, opts), fgs.nystrom_gaussian(op, opts)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.vectors, b.vectors)
    for k, L, M in ((0, 6, 3), (4, 6, 3), (2, 6, 7), (2, 5000, 3)):
        with pytest.raises(fgs.ParameterError):
            fgs.nystrom_gaussian(op, fgs.NystromOptions(k=k, L=L, M=M))


def test_nystrom_top_pair_close_to_lanczos():
    X = fgs.workload_nodes(2, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.05), fgs.FastsumParams(64, 6, 6, 0.0))
    ny = fgs.nystrom_gaussian(op, fgs.NystromOptions(k=4, L=100, M=10, seed=1))
    lz = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-10))
    assert abs(ny.values[0] - lz.values[0]) <= 1e-4  # approximation quality of the sketch (M = 10)
    assert np.all(np.isfinite(ny.vectors))


def test_cli_nystrom_method(tmp_path):
    out = tmp_path / "s.csv"
    write_spiral_csv(out, per_class=200, seed=2)
    rep_path = tmp_path / "ny.json"
    r = run(EXE, "eigs", "--in", out, "--out", rep_path, "--sigma", 3.5, "--k", 4, "--method", "nystrom-gauss-nfft",
            "--L", 40, "--M", 8)
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    check_report(rep)
    assert rep["method"] == "nystrom-gauss-nfft" and len(rep["eigenvalues"]) == 4
    assert set(rep["timings_seconds"]) >= {"setup", "solve"}
