"""The command-line drivers (paper_1808_04580_b200/cli, tools/commands.cpp
analogue): exit codes, the fgs-report-v1 report, CSV handling and the
generators.  CPU only: nothing here touches the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
EXE = os.path.join(os.path.dirname(HERE), "paper_1808_04580_b200", "fgs-b200")


@pytest.fixture(scope="module")
def exe():
    from paper_1808_04580_b200 import build
    build.build()
    assert os.path.exists(EXE)
    return EXE


def run(exe, *args):
    return subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=120)


def check_report(rep):
    """schema/report.schema.json constraints, restated."""
    for key in ("schema", "command", "parameters", "seed", "metrics", "timings_seconds", "status"):
        assert key in rep, key
    assert rep["schema"] == "fgs-report-v1"
    assert isinstance(rep["command"], str) and isinstance(rep["parameters"], dict)
    assert isinstance(rep["seed"], int) and rep["seed"] >= 0
    assert all(isinstance(v, (int, float)) for v in rep.get("eigenvalues", []))
    for name, m in rep["metrics"].items():
        assert set(m) >= {"value", "definition"} and isinstance(m["definition"], str), name
        assert isinstance(m["value"], (int, float, list))
    assert all(isinstance(v, (int, float)) and v >= 0 for v in rep["timings_seconds"].values())
    assert rep["status"] in ("ok", "numerical-failure")
    assert isinstance(rep.get("diagnostic", ""), str)
    if "extra" in rep:
        assert isinstance(rep["extra"], dict)


def test_gen_spiral_and_crescent(exe, tmp_path):
    out = tmp_path / "s.csv"
    r = run(exe, "gen", "--spiral", "--classes", 3, "--per-class", 40, "--out", out, "--seed", 9)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "x0,x1,x2,label" and len(lines) == 121
    data = np.array([[float(v) for v in l.split(",")] for l in lines[1:]])
    assert np.array_equal(data[:, 3], np.repeat([0, 1, 2], 40))
    rep = json.loads((tmp_path / "s.csv.report.json").read_text())
    check_report(rep)
    assert rep["command"] == "gen" and rep["method"] == "spiral" and rep["metrics"]["n"]["value"] == 120
    # deterministic in the seed
    run(exe, "gen", "--spiral", "--classes", 3, "--per-class", 40, "--out", tmp_path / "t.csv", "--seed", 9)
    assert (tmp_path / "t.csv").read_text() == out.read_text()
    r = run(exe, "gen", "--crescent-fullmoon", "--n", 200, "--out", tmp_path / "c.csv")
    assert r.returncode == 0, r.stderr
    pts = np.loadtxt(tmp_path / "c.csv", delimiter=",", skiprows=1)
    assert pts.shape == (200, 3) and np.sum(pts[:, 2] == 0) == 50
    moon, cres = pts[pts[:, 2] == 0, :2], pts[pts[:, 2] == 1, :2]
    assert np.all(np.hypot(moon[:, 0], moon[:, 1]) <= 5.0)  # dataset.cpp:227-234
    rr = np.hypot(cres[:, 0], cres[:, 1])
    assert np.all((rr > 5.0) & (rr <= 8.0)) and np.all(cres[:, 1] <= 0.0)


def test_usage_errors_exit_2(exe, tmp_path):
    assert run(exe).returncode == 2
    assert run(exe, "gen", "--out", tmp_path / "x.csv").returncode == 2  # neither generator
    assert run(exe, "gen", "--spiral", "--crescent-fullmoon", "--out", tmp_path / "x.csv").returncode == 2
    assert run(exe, "eigs", "--out", tmp_path / "r.json").returncode == 2  # --in required
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--bogus", 1).returncode == 2
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--setup", 4).returncode == 2
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--kernel", "cosine").returncode == 2
    assert run(exe, "segment", "--in", "a.png", "--out", "r.json").returncode == 2
    assert run(exe, "bench", "--out", "r.json", "--methods", "magic").returncode == 2
    assert run(exe, "--help").returncode == 0


def test_csv_input_errors_exit_2(exe, tmp_path):
    cases = {"empty.csv": "", "noheader.csv": "\n1,2\n", "ragged.csv": "x0,x1\n1,2\n3\n",
             "nonnum.csv": "x0,x1\n1,abc\n", "inf.csv": "x0,x1\n1,inf\n", "norows.csv": "x0,x1\n",
             "badlabel.csv": "x0,label\n1,2.5\n"}
    for name, text in cases.items():
        p = tmp_path / name
        p.write_text(text)
        r = run(exe, "eigs", "--in", p, "--out", tmp_path / "r.json")
        assert r.returncode == 2 and "input error" in r.stderr, (name, r.stderr)
    r = run(exe, "eigs", "--in", tmp_path / "missing.csv", "--out", tmp_path / "r.json")
    assert r.returncode == 2 and "cannot open" in r.stderr


def write_ppm(path, rgb):
    h, w, _ = rgb.shape
    with open(path, "wb") as f:
        f.write(b"P6\n%d %d\n255\n" % (w, h))
        f.write(np.ascontiguousarray(rgb, dtype=np.uint8).tobytes())


def test_segment_image_input_errors(exe, tmp_path):
    png = tmp_path / "a.png"
    png.write_bytes(b"\x89PNG\r\n\x1a\n" + b"\0" * 32)
    r = run(exe, "segment", "--in", png, "--out", tmp_path / "o.ppm")
    assert r.returncode == 2 and "libpng" in r.stderr
    bad = tmp_path / "b.ppm"
    bad.write_bytes(b"P3\n2 2\n255\n")
    assert run(exe, "segment", "--in", bad, "--out", tmp_path / "o.ppm").returncode == 2
    trunc = tmp_path / "t.ppm"
    trunc.write_bytes(b"P6\n4 4\n255\n" + b"\0" * 10)
    r = run(exe, "segment", "--in", trunc, "--out", tmp_path / "o.ppm")
    assert r.returncode == 2 and "truncated" in r.stderr
    deep = tmp_path / "d.ppm"
    deep.write_bytes(b"P6\n1 1\n65535\n" + b"\0" * 6)
    assert run(exe, "segment", "--in", deep, "--out", tmp_path / "o.ppm").returncode == 2
