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
from test_cli import EXE, check_report, run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spiral(tmp_path_factory):
    from paper_1808_04580_b200 import build
    build.build()
    d = tmp_path_factory.mktemp("cli")
    out = d / "spiral.csv"
    r = run(EXE, "gen", "--spiral", "--per-class", 400, "--out", out, "--seed", 4)
    assert r.returncode == 0, r.stderr
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


def test_ssl_kernel_cg_and_truncated(tmp_path):
    # commands.cpp:531-652: CG on (I + beta L_s) per one-vs-rest channel, or
    # the truncated-eigenbasis closed form
    pts = tmp_path / "cm.csv"
    assert run(EXE, "gen", "--crescent-fullmoon", "--n", 2000, "--out", pts, "--seed", 3).returncode == 0
    rates = {}
    for extra, method in (((), "cg"), (("--k", 16), "truncated-eig")):
        rep_path = tmp_path / f"ssl_{method}.json"
        r = run(EXE, "ssl-kernel", "--in", pts, "--out", rep_path, "--sigma", 2.0, "--beta", 10,
                "--samples-per-class", 10, "--tol", 1e-8, *extra)
        assert r.returncode == 0, r.stderr
        rep = json.loads(rep_path.read_text())
        check_report(rep)
        assert rep["method"] == method and rep["status"] == "ok"
        rates[method] = rep["metrics"]["misclassification_rate"]["value"]
        labels = np.loadtxt(str(rep_path) + ".labels.csv", skiprows=1, dtype=int)
        assert labels.shape == (2000,) and set(labels.tolist()) <= {0, 1}
    assert rates["cg"] <= 0.05
    cg = json.loads((tmp_path / "ssl_cg.json").read_text())
    assert cg["metrics"]["cg_converged"]["value"] == 1.0
    # too narrow a kernel for setup 2: the reference's nonpositive-degree
    # failure, reported with status numerical-failure and exit 1
    r = run(EXE, "ssl-kernel", "--in", pts, "--out", tmp_path / "bad.json", "--sigma", 0.5, "--beta", 10)
    assert r.returncode == 1
    assert json.loads((tmp_path / "bad.json").read_text())["status"] == "numerical-failure"


def test_krr_command(tmp_path):
    pts = tmp_path / "cm.csv"
    assert run(EXE, "gen", "--crescent-fullmoon", "--n", 800, "--out", pts, "--seed", 3).returncode == 0
    rep_path = tmp_path / "krr.json"
    r = run(EXE, "krr", "--in", pts, "--out", rep_path, "--sigma", 1.0, "--beta", 1e-2, "--setup", 3)
    assert r.returncode == 0, r.stderr
    rep = json.loads(rep_path.read_text())
    check_report(rep)
    assert rep["metrics"]["train_accuracy"]["value"] >= 0.95
    # unlabeled input is a usage error (commands.cpp:279-285)
    bare = tmp_path / "bare.csv"
    bare.write_text("x0,x1\n0.1,0.2\n0.3,0.1\n0.5,0.5\n")
    assert run(EXE, "krr", "--in", bare, "--out", tmp_path / "x.json").returncode == 2


def _voronoi_image(w, h, sites, seed):
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0, 1, (sites, 2)) * [w, h]
    cols = rng.uniform(0, 255, (sites, 3))
    yy, xx = np.mgrid[0:h, 0:w]
    d = (xx[..., None] - pts[:, 0]) ** 2 + (yy[..., None] - pts[:, 1]) ** 2
    img = cols[np.argmin(d, axis=-1)] + rng.normal(0, 5, (h, w, 3))
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def test_segment_small_image_with_reference(tmp_path):
    from test_cli import write_ppm
    img = _voronoi_image(80, 60, 4, 2)
    src = tmp_path / "img.ppm"
    write_ppm(src, img)
    out = tmp_path / "seg.ppm"
    r = run(EXE, "segment", "--in", src, "--out", out, "--with-reference")
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "seg.ppm.report.json").read_text())
    check_report(rep)
    assert rep["command"] == "segment" and rep["parameters"]["sigma"] == 90.0 and rep["parameters"]["k"] == 4
    assert rep["metrics"]["label_difference_fraction"]["value"] <= 0.01
    data = out.read_bytes()
    assert data.startswith(b"P6\n80 60\n255\n") and len(data) == len(b"P6\n80 60\n255\n") + 80 * 60 * 3
    assert (tmp_path / "seg.diff.ppm").exists()


def test_segment_config3_image_matches_api(tmp_path):
    # BASELINE config 3: the 800 x 600 synthetic image, k = 4, then k-means
    from test_cli import write_ppm
    X = fgs.workload_nodes(3, 2024)
    assert X.shape == (480000, 3)
    src = tmp_path / "c3.ppm"
    write_ppm(src, X.reshape(600, 800, 3))
    out = tmp_path / "c3_seg.ppm"
    r = run(EXE, "segment", "--in", src, "--out", out, "--N", 32, "--m", 4, "--p", 4)
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "c3_seg.ppm.report.json").read_text())
    assert rep["metrics"]["lanczos_converged"]["value"] == 1.0
    # the same pipeline through the library: identical labels
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(90.0), fgs.FastsumParams(32, 4, 4, 0.0))
    pairs = fgs.lanczos_largest(op, 4, fgs.LanczosOptions(tol=1e-12, seed=1))
    assert np.array_equal(np.array(rep["eigenvalues"]), pairs.values)
    labels = fgs.spectral_cluster(pairs, 4, fgs.KMeansOptions(seed=1))
    pal = np.array([[31, 119, 180], [255, 127, 14], [44, 160, 44], [214, 39, 40]], dtype=np.uint8)
    raw = out.read_bytes()
    pix = np.frombuffer(raw[len(b"P6\n800 600\n255\n"):], dtype=np.uint8).reshape(-1, 3)
    assert np.array_equal(pix, pal[labels])
